# feature-sharing parity + the whole GPU suite
timeout 900 python -m pytest tests/test_gpu_features.py -x -q -p no:cacheprovider --durations=8 > gpurun_out/r2_features.log 2>&1; echo "rc=$?" >> gpurun_out/r2_features.log
tail -15 gpurun_out/r2_features.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2_gputest5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest5.log
tail -16 gpurun_out/r2_gputest5.log
