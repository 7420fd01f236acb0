bash scripts/variants_dist.sh 32768 "" "-DTDB_EDGE_APT=2" "-DTDB_EDGE_APT=2 -DTDB_UEE=2" "-DTDB_EDGE_APT=2 -DTDB_EDGE_MINB=3" > gpurun_out/r2_var4.txt 2>&1
cat gpurun_out/r2_var4.txt
