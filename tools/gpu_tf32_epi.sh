mkdir -p gpurun_out
(TD=4096 timeout 60 ./tools/tf32_timing_; TIME_D=4096 timeout 120 python tools/time_f32_gemm.py; NSERIES_LIB=tools/variants/orig.so TIME_D=4096 timeout 120 python tools/time_f32_gemm.py) > gpurun_out/tf32_epi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "f32 or tf32 or fp32 or sym" > gpurun_out/tf32_epi_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tf32_epi_tests.log
