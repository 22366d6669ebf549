mkdir -p gpurun_out
TIME_D=4096 timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -s 5 -c 1 -o gpurun_out/tf32_full -f python tools/time_f32_gemm.py > gpurun_out/tf32_ncu.log 2>&1
