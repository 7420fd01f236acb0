# q_hit_kernel with NS staged sub-tiles released per warp (Stream<.., NS>): variants on the paper
# intersects workload, then the query / literal / fuzz GPU tests and ncu on the default build
make -s lib >/dev/null 2>&1
for v in 2 4 6 8; do
  touch paper_1808_09571_b200/csrc/queries.cu
  make -s lib EXTRA="-DTDB_QHIT_STAGES=$v" >/dev/null 2>&1 || { echo "build failed $v"; continue; }
  timeout 600 python bench.py --config paper --op intersects --steps 8 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('TDB_QHIT_STAGES=$v %.4g pairs/s  %.2f ms/step' % (d['value'], d['ms_per_step']))"
done 2>&1 | tee gpurun_out/r2o_qhit_variants.txt
touch paper_1808_09571_b200/csrc/queries.cu; make -s lib >/dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_queries.py tests/test_gpu_literal.py tests/test_gpu_fuzz.py tests/test_gpu_bounds.py -q -p no:cacheprovider -x > gpurun_out/r2o_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2o_tests.log
tail -3 gpurun_out/r2o_tests.log
ncu --set full --clock-control none --import-source on -k regex:"^q_hit_kernel" -c 1 -o gpurun_out/r2o_paper_q_hit_kernel -f python bench.py --config paper --op intersects --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2o_prof_q_hit_kernel.log 2>&1; echo "q_hit_kernel rc=$?"
