mkdir -p gpurun_out
(for i in 1 2 3; do for lead in 0 1; do echo -n "lead=$lead "; NSERIES_TF32_LEAD=$lead TIME_D=4096 timeout 120 python tools/time_f32_gemm.py; done; done
for lead in 0 1; do echo -n "lead=$lead d=8192 "; NSERIES_TF32_LEAD=$lead TIME_D=8192 timeout 200 python tools/time_f32_gemm.py; done) > gpurun_out/tf32_lead.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "f32 or tf32 or fp32 or sym or splitk" > gpurun_out/tf32_lead_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tf32_lead_tests.log
