# super-tile A lists: feature tests (incl. the numpy restatement of the counts), parity, memcheck, bench
timeout 900 python -m pytest tests/test_gpu_features.py -x -q -p no:cacheprovider > gpurun_out/r2_hd_features.log 2>&1; echo "rc=$?" >> gpurun_out/r2_hd_features.log
tail -6 gpurun_out/r2_hd_features.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py tests/test_gpu_group.py tests/test_gpu_bounds.py tests/test_gpu_shim.py -x -q -p no:cacheprovider > gpurun_out/r2_hd_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_hd_tests.log
tail -4 gpurun_out/r2_hd_tests.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_features.py -q -p no:cacheprovider -x > gpurun_out/r2_hd_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2_hd_memcheck.log
tail -3 gpurun_out/r2_hd_memcheck.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/r2_hd_bench.json 2> gpurun_out/r2_hd_bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/r2_hd_bench.json; python -c "
import json; d=json.load(open('gpurun_out/r2_hd_bench.json')); r=d['roofline']; print(d['e2e']['value'], r['features_per_face'], r['fp64_instr_per_pair'], r['fp64_pipe_frac'])"
