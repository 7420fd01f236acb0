timeout 1500 python -m pytest tests/test_gpu_queries.py tests/test_gpu_bounds.py tests/test_gpu_literal.py tests/test_gpu_degenerate.py tests/test_gpu_direct.py tests/test_gpu_shim.py -q -x -p no:cacheprovider > gpurun_out/r2_qhit_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_qhit_tests.log
tail -3 gpurun_out/r2_qhit_tests.log
timeout 900 python bench.py --config paper --op intersects --steps 8 --no-cpu 2>/dev/null | tail -1 | cut -c1-260
