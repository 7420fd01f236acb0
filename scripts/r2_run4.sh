# round-2 (re-entry) GPU check: whole GPU suite, latency, default bench, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/r2_gputest4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest4.log
tail -40 gpurun_out/r2_gputest4.log
timeout 600 python scripts/latency_probe.py > gpurun_out/r2_latency.jsonl 2>&1; cat gpurun_out/r2_latency.jsonl
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo "bench rc=$?"; cat gpurun_out/r2_bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc=$?"; cat gpurun_out/r2_bench_ref.json
