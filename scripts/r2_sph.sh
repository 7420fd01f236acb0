# filter_kernel<false>: A-face sphere vs B-block sphere skip of the straddle loop. Distance GPU tests,
# default bench, ncu of the filter kernel
make -s lib >/dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_features.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_bounds.py tests/test_gpu_fuzz.py tests/test_gpu_benchscale.py -q -p no:cacheprovider -x > gpurun_out/r2r_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2r_tests.log
tail -3 gpurun_out/r2r_tests.log
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu --e2e-steps 4 > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/r2r_bench.json
ncu --set full --clock-control none --import-source on -k regex:"^filter_kernel" -c 1 -o gpurun_out/r2r_c2_filter_kernel -f python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2r_prof_filter.log 2>&1; echo "ncu rc=$?"
