# batched config-4 control: SIMT FFMA2 products (tools/variants/bw_ffma.so) vs 3xTF32 mma.sync
mkdir -p gpurun_out
O=gpurun_out/bw_ffma.txt
: > $O
for i in 1 2; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/bw_ffma.so; do
    NSERIES_LIB=$lib ALL=1 timeout 200 python tools/time_batched.py >> $O 2>&1
  done
done
NSERIES_LIB=tools/variants/bw_ffma.so timeout 300 ncu --metrics smsp__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:batched_warp -s 3 -c 1 python tools/time_batched.py 2>&1 | grep -E "smsp__|sm__|l1tex" >> $O
