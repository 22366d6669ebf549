mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -q -k warps_per_matrix > gpurun_out/wpm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wpm_tests.log
