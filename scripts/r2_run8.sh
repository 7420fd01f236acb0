# small-call path: parity (direct vs pipeline), concurrency, shim; latency probe
timeout 1200 python -m pytest tests/test_gpu_direct.py tests/test_gpu_concurrency.py tests/test_gpu_degenerate.py tests/test_gpu_shim.py tests/test_gpu_queries.py tests/test_gpu_literal.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2_small.log 2>&1; echo "rc=$?" >> gpurun_out/r2_small.log
tail -5 gpurun_out/r2_small.log
timeout 600 python scripts/latency_probe.py > gpurun_out/r2_latency2.jsonl 2>&1; cat gpurun_out/r2_latency2.jsonl
gcc -O2 -Iinclude scripts/latency_c.c -Lpaper_1808_09571_b200 -ltindb_b200 -Wl,-rpath,$PWD/paper_1808_09571_b200 -o /tmp/latency_c && /tmp/latency_c > gpurun_out/r2_latency_c.jsonl 2>&1; cat gpurun_out/r2_latency_c.jsonl
