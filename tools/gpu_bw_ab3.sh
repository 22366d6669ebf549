# batched kernel: natural row order + run-time diagonal predicate (current) vs row-swapped
# order (previous commit, bw_head.so); instruction counts from one ncu capture of each
mkdir -p gpurun_out
O=gpurun_out/bw_ab3.txt
: > $O
for i in 1 2 3; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/bw_head.so; do
    NSERIES_LIB=$lib ALL=1 timeout 200 python tools/time_batched.py 2>&1 | grep -v "^worst" >> $O
  done
done
for lib in paper_2602_11843_b200/libnseries.so tools/variants/bw_head.so; do
  NSERIES_LIB=$lib timeout 300 ncu --metrics smsp__inst_executed.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:batched_warp -s 3 -c 1 python tools/time_batched.py 2>&1 | grep -E "smsp__inst|hmma|bank" >> $O
done
timeout 600 python -m pytest tests/test_gpu_batched.py tests/test_gpu_stats.py -x -q >> $O 2>&1
echo done >> $O
