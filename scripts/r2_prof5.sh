# round-2 evidence with the shipped build: default bench (+ reference arm),
# launch list, --set full of each distance kernel and of hit_kernel at the
# bench launch sizes
timeout 900 python bench.py > gpurun_out/r2e_bench_default.json 2> gpurun_out/r2e_bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2e_bench_reference.json 2> gpurun_out/r2e_bench_reference.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launches_bench_default.csv python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2e_launches.log 2>&1; echo "launches rc=$?"
for k in edge_kernel vertex_kernel filter_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" -c 1 -o gpurun_out/r2e_c2_$k -f python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2e_prof_$k.log 2>&1; echo "$k rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:"^hit_kernel" -c 1 -o gpurun_out/r2e_c3_hit_kernel -f python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2e_prof_hit.log 2>&1; echo "hit rc=$?"
