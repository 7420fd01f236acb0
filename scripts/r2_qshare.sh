# shared-edge fused query kernel: query parity (fused / chunked / flag / bounds / shim), then the paper bench
timeout 1500 python -m pytest tests/test_gpu_degenerate.py tests/test_gpu_queries.py tests/test_gpu_bounds.py tests/test_gpu_shim.py tests/test_gpu_parity.py -q -x -p no:cacheprovider --durations=5 > gpurun_out/r2_qshare_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_qshare_tests.log
tail -9 gpurun_out/r2_qshare_tests.log
timeout 900 python bench.py --config paper --steps 8 --no-cpu 2>/dev/null | tail -1 | cut -c1-300
