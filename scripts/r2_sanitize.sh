# compute-sanitizer over the round-2 kernels: memcheck (feature lists, split
# filter, direct path, concurrency) and racecheck (split filter SMEM/TMA
# stages; concurrent callers)
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_features.py tests/test_gpu_direct.py tests/test_gpu_concurrency.py -q -p no:cacheprovider -x > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2_memcheck.log
tail -4 gpurun_out/r2_memcheck.log
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_features.py tests/test_gpu_concurrency.py -q -p no:cacheprovider -x -k "not table_records" > gpurun_out/r2_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r2_racecheck.log
tail -4 gpurun_out/r2_racecheck.log
