# FP32 edge/edge lists: parity (features, parity, fullsize C2), the FP32 bound test, a default bench
timeout 1500 python -m pytest tests/test_gpu_features.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_bounds.py -q -p no:cacheprovider -x -s --durations=5 > gpurun_out/r2k_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2k_tests.log
tail -25 gpurun_out/r2k_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo "bench rc=$?"
cat gpurun_out/r2k_bench.json; tail -5 gpurun_out/r2k_bench.err
