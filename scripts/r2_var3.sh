bash scripts/variants_dist.sh 32768 "" "-DTDB_FACE_MINB=4" "-DTDB_EDGE_MINB=5" "-DTDB_FACE_MINB=4 -DTDB_EDGE_MINB=5" "-DTDB_UEE=2 -DTDB_EDGE_MINB=6" "-DTDB_UEE=8" "-DTDB_FACE_MINB=4 -DTDB_UEE=2 -DTDB_EDGE_MINB=5" > gpurun_out/r2_var3.txt 2>&1
cat gpurun_out/r2_var3.txt
