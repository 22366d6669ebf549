mkdir -p gpurun_out
(TD=4096 timeout 60 ./tools/tf32_timing_ | grep -E "variant|phases"
for i in 1 2; do for lib in tools/variants/ru4.so paper_2602_11843_b200/libnseries.so; do echo -n "$lib "; NSERIES_LIB=$lib TIME_D=4096 timeout 120 python tools/time_f32_gemm.py; done; done) > gpurun_out/tf32_na.txt 2>&1
