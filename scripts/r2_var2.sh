bash scripts/variants_dist.sh 32768 "-DTDB_UF=1" "-DTDB_UF=2" "-DTDB_UE=2" "-DTDB_UV=2 -DTDB_UF=2 -DTDB_UE=2" "-DTDB_UF=2 -DTDB_UV=4 -DTDB_UE=2" > gpurun_out/r2_var2.txt 2>&1
cat gpurun_out/r2_var2.txt
