mkdir -p gpurun_out
(for i in 1 2; do for lib in paper_2602_11843_b200/libnseries.so tools/variants/c2test.so tools/variants/c2hint20.so tools/variants/c2hint1000.so; do echo "== $lib"; NSERIES_LIB=$lib timeout 120 python tools/time_small.py 2>&1 | head -4; done; done) > gpurun_out/small_ab2.txt 2>&1
