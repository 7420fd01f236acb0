# round-2 GPU check 3: new tests first, then the whole suite, latency, 2-rank bench under gloo
timeout 1500 python -m pytest tests/test_gpu_direct.py tests/test_gpu_concurrency.py tests/test_gpu_degenerate.py tests/test_gpu_shim.py tests/test_gpu_benchscale.py -q -x -s -p no:cacheprovider --durations=10 > gpurun_out/r2_new.log 2>&1; echo "rc=$?" >> gpurun_out/r2_new.log
tail -25 gpurun_out/r2_new.log
timeout 600 python scripts/latency_probe.py > gpurun_out/r2_latency.jsonl 2>&1; cat gpurun_out/r2_latency.jsonl
TDB_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_gloo2.out 2> gpurun_out/r2_gloo2.err; echo "gloo2 rc=$?"; tail -2 gpurun_out/r2_gloo2.out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/r2_gputest3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest3.log
tail -32 gpurun_out/r2_gputest3.log
