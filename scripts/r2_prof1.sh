# ncu --set full of the feature-block filter (8,192 terrain rows x 1.31M ore faces)
ncu --set full --clock-control none --import-source on -k regex:filter_kernel -c 1 -o gpurun_out/r2_filter_fb -f python scripts/one_call.py distance 8192 > gpurun_out/r2_prof1.log 2>&1
tail -3 gpurun_out/r2_prof1.log
