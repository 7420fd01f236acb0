# small-call changes: the whole GPU suite, then both latency probes
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/r2_gputest6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest6.log
tail -10 gpurun_out/r2_gputest6.log
timeout 600 python scripts/latency_probe.py > gpurun_out/r2_latency3.jsonl 2>&1; cat gpurun_out/r2_latency3.jsonl
gcc -O2 -Iinclude scripts/latency_c.c -Lpaper_1808_09571_b200 -ltindb_b200 -Wl,-rpath,$PWD/paper_1808_09571_b200 -o /tmp/latency_c && /tmp/latency_c > gpurun_out/r2_latency3_c.jsonl 2>&1; cat gpurun_out/r2_latency3_c.jsonl
