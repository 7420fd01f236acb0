# round-2 closing check on the shipped build: GPU suite, small-call latency, paper intersects and
# default C2 bench lines
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/r2p_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2p_gputest.log
tail -3 gpurun_out/r2p_gputest.log
timeout 600 python scripts/latency_probe.py > gpurun_out/r2p_latency.jsonl 2> gpurun_out/r2p_latency.err; echo "latency rc=$?"; cat gpurun_out/r2p_latency.jsonl
timeout 900 python bench.py --config paper --op intersects --steps 8 > gpurun_out/r2p_bench_paper_hit.json 2> gpurun_out/r2p_bench_paper_hit.err; echo "paper rc=$?"; cut -c1-200 gpurun_out/r2p_bench_paper_hit.json
timeout 900 python bench.py > gpurun_out/r2p_bench_default.json 2> gpurun_out/r2p_bench_default.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/r2p_bench_default.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2p_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2p_smoke.log
