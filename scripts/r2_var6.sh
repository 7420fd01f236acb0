bash scripts/variants_dist.sh 65536 "" "-DTDB_EDGE_APT=3 -DTDB_EDGE_MINB=3" "-DTDB_EDGE_APT=4 -DTDB_EDGE_MINB=3" "-DTDB_EDGE_APT=1 -DTDB_EDGE_MINB=4 -DTDB_UEE=8" > gpurun_out/r2_var6.txt 2>&1
cat gpurun_out/r2_var6.txt
