# chunk-major CTA order for filter_kernel<false> / vertex_kernel, stage count, edge32 occupancy:
# bench variants, then tests + bench + ncu of the default build
make -s lib >/dev/null 2>&1
bash scripts/variants_bench.sh "-DTDB_FCHUNK_MAJOR=0 -DTDB_FSTAGES=2" "-DTDB_FCHUNK_MAJOR=0 -DTDB_FSTAGES=4" \
  "-DTDB_FCHUNK_MAJOR=1 -DTDB_FSTAGES=2" "-DTDB_FCHUNK_MAJOR=1 -DTDB_FSTAGES=3" "-DTDB_FCHUNK_MAJOR=1 -DTDB_FSTAGES=4" \
  "-DTDB_FCHUNK_MAJOR=1 -DTDB_FSTAGES=4 -DTDB_E32_MINB=5" "-DTDB_FCHUNK_MAJOR=1 -DTDB_FSTAGES=4 -DTDB_E32_PACKED=1" \
  "-DTDB_FCHUNK_MAJOR=1 -DTDB_FSTAGES=3 -DTDB_FACE_MINB=5" 2>&1 | tee gpurun_out/r2m_variants.txt
timeout 1500 python -m pytest tests/test_gpu_features.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/r2m_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2m_tests.log
tail -3 gpurun_out/r2m_tests.log
for k in filter_kernel vertex_kernel; do
ncu --set full --clock-control none --import-source on -k regex:"^$k" -c 1 -o gpurun_out/r2m_c2_$k -f python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2m_prof_$k.log 2>&1; echo "ncu $k rc=$?"
done
