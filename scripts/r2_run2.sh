# round-2 GPU check: full GPU suite
timeout 3300 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/r2_gputest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest2.log
tail -40 gpurun_out/r2_gputest2.log
