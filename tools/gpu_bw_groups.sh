# batched kernel: 6 / 7 / 8 (default) matrices per SM (register budget 170 / 146 / 128 per thread)
mkdir -p gpurun_out
O=gpurun_out/bw_groups.txt
: > $O
for i in 1 2; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/bw_g7.so tools/variants/bw_g6.so; do
    NSERIES_LIB=$lib ALL=1 timeout 200 python tools/time_batched.py 2>&1 | grep -v "^worst" >> $O
  done
done
