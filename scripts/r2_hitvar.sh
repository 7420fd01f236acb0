# hit_kernel block cull: parity / bounds tests, then occupancy variants on C3 and C3 stress
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py tests/test_gpu_fullsize.py tests/test_gpu_group.py -q -x -p no:cacheprovider -k "intersect or hit or cull or c3" > gpurun_out/r2_hit_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_hit_tests.log
tail -3 gpurun_out/r2_hit_tests.log
for v in "-DTDB_HIT_MINB=4" "-DTDB_HIT_MINB=3"; do
  touch paper_1808_09571_b200/csrc/intersects.cu; make -s lib EXTRA="$v" >/dev/null 2>&1 || echo "build failed $v"
  echo "== $v"; python scripts/hit_probe.py 2>&1 | tail -2
done
touch paper_1808_09571_b200/csrc/intersects.cu; make -s lib >/dev/null 2>&1
