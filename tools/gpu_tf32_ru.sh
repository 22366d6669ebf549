mkdir -p gpurun_out
(for b in tools/tf32_timing_ tools/tf32_timing_ru4 tools/tf32_timing_ru8; do echo "== $b"; TD=4096 timeout 60 ./$b | grep -E "variant|phases"; done
for i in 1 2; do for lib in paper_2602_11843_b200/libnseries.so tools/variants/ru4.so tools/variants/ru8.so; do echo -n "$lib "; NSERIES_LIB=$lib TIME_D=4096 timeout 120 python tools/time_f32_gemm.py; done; done) > gpurun_out/tf32_ru.txt 2>&1
