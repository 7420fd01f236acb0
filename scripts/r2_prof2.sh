# ncu --set full of the split filter's two kernels (8,192 terrain rows x 1.31M ore faces)
ncu --set full --clock-control none --import-source on -k regex:"^(filter_kernel|edge_kernel)" -c 2 -o gpurun_out/r2_split -f python scripts/one_call.py distance 8192 > gpurun_out/r2_prof2.log 2>&1
tail -3 gpurun_out/r2_prof2.log
