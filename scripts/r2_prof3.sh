# round-2 captures of the FULL-mode distance kernels at the bench's launch size
# (65,536 terrain rows x 1,310,720 ore faces = one C2 step) + the bench launch list
ncu --set full --clock-control none --import-source on -k regex:"^(filter_kernel|edge_kernel|vertex_kernel)" -c 3 -o gpurun_out/r2_c2_kernels -f python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2_prof3a.log 2>&1
tail -2 gpurun_out/r2_prof3a.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench_default.csv python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2_prof3b.log 2>&1
tail -2 gpurun_out/r2_prof3b.log
