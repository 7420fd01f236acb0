# round-2 final evidence (4-stage chunk-major filter, packed FP32 edges): GPU suite, sweep, default bench + reference arm,
# launch list, ncu --set full of each FULL-mode distance kernel (bench launch)
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/r2n_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2n_gputest.log
tail -3 gpurun_out/r2n_gputest.log
bash scripts/sweep.sh; python scripts/hit_probe.py > gpurun_out/r2n_hit_probe.txt 2>&1; cat gpurun_out/r2n_hit_probe.txt
cp gpurun_out/sweep.jsonl gpurun_out/r2n_sweep.jsonl
timeout 900 python bench.py > gpurun_out/r2n_bench_default.json 2> gpurun_out/r2n_bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2n_bench_reference.json 2> gpurun_out/r2n_bench_reference.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n_launches_bench_default.csv python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2n_launches.log 2>&1; echo "launches rc=$?"
for k in edge32_kernel vertex_kernel filter_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" -c 1 -o gpurun_out/r2n_c2_$k -f python bench.py --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2n_prof_$k.log 2>&1; echo "$k rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:"^hit_kernel" -c 1 -o gpurun_out/r2n_c3_hit_kernel -f python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2n_prof_hit_kernel.log 2>&1; echo "hit_kernel rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"^q_hit_kernel" -c 1 -o gpurun_out/r2n_paper_q_hit_kernel -f python bench.py --config paper --op intersects --steps 1 --warmup 0 --no-cpu --e2e-steps 0 > gpurun_out/r2n_prof_q_hit_kernel.log 2>&1; echo "q_hit_kernel rc=$?"
