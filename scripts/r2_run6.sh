# split filter (faces/vertices kernel + A-edge x B-edge kernel): parity, bounds, bench
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py tests/test_gpu_group.py tests/test_gpu_bounds.py tests/test_gpu_shim.py -x -q -p no:cacheprovider --durations=8 > gpurun_out/r2_split5_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_split5_tests.log
tail -15 gpurun_out/r2_split5_tests.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/r2_split5_bench.json 2> gpurun_out/r2_split5_bench.err; echo "bench rc=$?"; cat gpurun_out/r2_split5_bench.json; tail -5 gpurun_out/r2_split5_bench.err
