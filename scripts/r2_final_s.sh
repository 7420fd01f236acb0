# round-2 closing evidence (sphere skip build): GPU suite, sweep, default bench + reference arm,
# launch list, smoke (the kernels changed since r2n are captured in r2r)
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/r2s_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s_gputest.log
tail -3 gpurun_out/r2s_gputest.log
bash scripts/sweep.sh; python scripts/hit_probe.py > gpurun_out/r2s_hit_probe.txt 2>&1; cat gpurun_out/r2s_hit_probe.txt
cp gpurun_out/sweep.jsonl gpurun_out/r2s_sweep.jsonl
timeout 900 python bench.py > gpurun_out/r2s_bench_default.json 2> gpurun_out/r2s_bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2s_bench_reference.json 2> gpurun_out/r2s_bench_reference.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_bench_default.csv python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2s_launches.log 2>&1; echo "launches rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo "smoke rc=$?"
