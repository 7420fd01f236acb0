# round-2 captures of each FULL-mode distance kernel at the bench launch size (65,536 x 1,310,720)
for k in edge_kernel vertex_kernel filter_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" -c 1 -o gpurun_out/r2_c2_$k -f python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2_prof4_$k.log 2>&1
  tail -1 gpurun_out/r2_prof4_$k.log
done
