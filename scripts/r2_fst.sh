# filter_kernel<false> stage pipeline (per-warp release, TDB_FSTAGES blocks in flight) and the packed
# FP32 edge/edge loop (TDB_E32_PACKED): variants on a 65,536-row C2 call, then parity / feature /
# bound tests and a short bench on the default build, and ncu of both kernels
make -s lib >/dev/null 2>&1
bash scripts/variants_dist.sh 65536 "-DTDB_FSTAGES=2 -DTDB_E32_PACKED=0" "-DTDB_FSTAGES=4 -DTDB_E32_PACKED=0" \
  "-DTDB_FSTAGES=3" "-DTDB_FSTAGES=4" "-DTDB_FSTAGES=6" "-DTDB_FSTAGES=4 -DTDB_E32_MINB=5" \
  "-DTDB_FSTAGES=4 -DTDB_E32_APT=2 -DTDB_E32_MINB=8" "-DTDB_FSTAGES=4 -DTDB_UE32=4" 2>&1 | tee gpurun_out/r2l_variants.txt
timeout 1500 python -m pytest tests/test_gpu_features.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_bounds.py -q -p no:cacheprovider -x > gpurun_out/r2l_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2l_tests.log
tail -4 gpurun_out/r2l_tests.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/r2l_bench.json
for k in edge32_kernel filter_kernel; do
ncu --set full --clock-control none --import-source on -k regex:"^$k" -c 1 -o gpurun_out/r2l_c2_$k -f python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2l_prof_$k.log 2>&1; echo "ncu $k rc=$?"
done
