mkdir -p gpurun_out
(for i in 1 2; do for lib in paper_2602_11843_b200/libnseries.so tools/variants/kc16.so; do NSERIES_LIB=$lib ALL=1 timeout 200 python tools/time_batched.py; done; done) > gpurun_out/bw_kc.txt 2>&1
