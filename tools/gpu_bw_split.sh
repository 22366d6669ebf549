# batched config-4 kernel: tf32 split via cvt.rn (F2FP) vs the bit-pattern rna split; WPM sweep
mkdir -p gpurun_out
O=gpurun_out/bw_split.txt
: > $O
(nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/f2fp tools/f2fp_split.cu && timeout 120 /tmp/f2fp) >> $O 2>&1
for i in 1 2; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/bw_bits.so; do
    NSERIES_LIB=$lib ALL=1 timeout 200 python tools/time_batched.py >> $O 2>&1
  done
done
for w in 1 4; do NSERIES_BATCHED_WPM=$w timeout 200 python tools/time_batched.py >> $O 2>&1; done
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q >> $O 2>&1
echo done >> $O
