# batched config-4 kernel A/B: current tree vs tools/variants/bw_head.so (previous commit), alternating
mkdir -p gpurun_out
O=gpurun_out/bw_ab.txt
: > $O
for i in 1 2; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/bw_head.so; do
    NSERIES_LIB=$lib ALL=1 timeout 200 python tools/time_batched.py 2>&1 | grep -v "^worst" >> $O
  done
done
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_stats.py -x -q >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or f32 or batched" >> $O 2>&1
echo done >> $O
