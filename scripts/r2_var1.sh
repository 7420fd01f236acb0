# filter variants: occupancy (MINB) x feature block size (KFB); one C2 call of 65,536 rows each
bash scripts/variants.sh 65536 "-DTDB_FILTER_MINB=3" "-DTDB_FILTER_MINB=4" "-DTDB_KFB=128" "-DTDB_KFB=128 -DTDB_FILTER_MINB=4" "-DTDB_KFB=32 -DTDB_FILTER_MINB=4" > gpurun_out/r2_var1.txt 2>&1
cat gpurun_out/r2_var1.txt
