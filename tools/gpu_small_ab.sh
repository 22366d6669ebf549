mkdir -p gpurun_out
(for i in 1 2 3; do for lib in tools/variants/orig.so paper_2602_11843_b200/libnseries.so; do echo "== $lib"; NSERIES_LIB=$lib timeout 120 python tools/time_small.py 2>&1 | head -4; done; done) > gpurun_out/small_ab.txt 2>&1
