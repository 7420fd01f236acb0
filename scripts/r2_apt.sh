# edge32_kernel A edges per thread (packed pairs) x CTAs/SM, bench C2
make -s lib >/dev/null 2>&1
bash scripts/variants_bench.sh "-DTDB_E32_APT=4 -DTDB_E32_MINB=5" "-DTDB_E32_APT=6 -DTDB_E32_MINB=4" "-DTDB_E32_APT=8 -DTDB_E32_MINB=3" "-DTDB_E32_APT=4 -DTDB_E32_MINB=5 -DTDB_UE32=4" 2>&1 | tee gpurun_out/r2u_apt_variants.txt
