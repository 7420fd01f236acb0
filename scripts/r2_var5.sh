# sharing granularity: A super-tile size (tiles) x B edge group (faces); one C2 call of 65,536 rows
bash scripts/variants.sh 65536 "" "-DTDB_BSUPER=4096" "-DTDB_BSUPER=8192" "-DTDB_SUPERTILE=256" "-DTDB_SUPERTILE=256 -DTDB_BSUPER=8192" > gpurun_out/r2_var5.txt 2>&1
cat gpurun_out/r2_var5.txt
