# hit_kernel with NS staged sub-tiles released per warp (TDB_HIT_STAGES) of TDB_HIT_SB faces:
# variants on the C3 / C3-stress probe, then the full GPU suite and ncu on the default build
make -s lib >/dev/null 2>&1
for v in "-DTDB_HIT_STAGES=2 -DTDB_HIT_SB=128" "-DTDB_HIT_STAGES=2 -DTDB_HIT_SB=64" "-DTDB_HIT_STAGES=4 -DTDB_HIT_SB=64" "-DTDB_HIT_STAGES=8 -DTDB_HIT_SB=32"; do
  touch paper_1808_09571_b200/csrc/intersects.cu
  make -s lib EXTRA="$v" >/dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"; timeout 600 python scripts/hit_probe.py 2>&1 | tail -2
done 2>&1 | tee gpurun_out/r2q_hit_variants.txt
touch paper_1808_09571_b200/csrc/intersects.cu; make -s lib >/dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=3 > gpurun_out/r2q_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2q_gputest.log
tail -3 gpurun_out/r2q_gputest.log
timeout 900 python bench.py --config c3 --steps 4 > gpurun_out/r2q_bench_c3.json 2> gpurun_out/r2q_bench_c3.err; echo "c3 rc=$?"; cut -c1-200 gpurun_out/r2q_bench_c3.json
ncu --set full --clock-control none --import-source on -k regex:"^hit_kernel" -c 1 -o gpurun_out/r2q_c3_hit_kernel -f python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2q_prof_hit_kernel.log 2>&1; echo "hit_kernel rc=$?"
