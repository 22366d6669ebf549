# batched kernel: hi*hi IEEE add lagged one k-step (bw_lag.so) vs immediate (current)
mkdir -p gpurun_out
O=gpurun_out/bw_lag.txt
: > $O
for i in 1 2 3; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/bw_lag.so; do
    NSERIES_LIB=$lib ALL=1 timeout 200 python tools/time_batched.py 2>&1 | grep -v "^worst" >> $O
  done
done
