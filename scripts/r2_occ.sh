# occupancy variants of filter_kernel<false> / vertex_kernel after the sphere skip (bench C2)
make -s lib >/dev/null 2>&1
bash scripts/variants_bench.sh "-DTDB_FSTAGES=4" "-DTDB_FACE_MINB=5" "-DTDB_FACE_MINB=5 -DTDB_UV=2" "-DTDB_VERT_MINB=5" "-DTDB_FACE_MINB=5 -DTDB_VERT_MINB=5" "-DTDB_FSTAGES=2" 2>&1 | tee gpurun_out/r2t_occ_variants.txt
