# batched SIMT control with one warp per matrix (4 rows x 4 column pairs per lane, 171 FMAs per
# shared-memory wavefront) vs 2 warps per matrix and the 3xTF32 kernel
mkdir -p gpurun_out
O=gpurun_out/bw_ffma4.txt
: > $O
for i in 1 2; do
  NSERIES_LIB=paper_2602_11843_b200/libnseries.so ALL=1 timeout 200 python tools/time_batched.py 2>&1 | grep -v "^worst" >> $O
  for w in 1 2; do NSERIES_BATCHED_WPM=$w NSERIES_LIB=tools/variants/bw_ffma_o8.so ALL=1 timeout 200 python tools/time_batched.py 2>&1 | grep -v "^worst" >> $O; done
done
