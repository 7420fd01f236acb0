set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2_gputest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest1.log
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err
timeout 600 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
timeout 900 python bench.py --config c3s --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r2_bench_c3s.json 2> gpurun_out/r2_bench_c3s.err
tail -3 gpurun_out/r2_gputest1.log; cat gpurun_out/r2_bench_*.json
