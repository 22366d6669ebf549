# batched config-4 SIMT control: original swizzle, fully unrolled k loop (bw_ffma_o8) vs quad swizzle (bw_ffma_q8)
mkdir -p gpurun_out
O=gpurun_out/bw_ffma3.txt
: > $O
for i in 1 2; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/bw_ffma_o8.so tools/variants/bw_ffma_q8.so; do
    NSERIES_LIB=$lib ALL=1 timeout 200 python tools/time_batched.py 2>&1 | grep -v "^worst" >> $O
  done
done
NSERIES_LIB=tools/variants/bw_ffma_o8.so timeout 300 ncu --metrics smsp__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:batched_warp -s 3 -c 1 python tools/time_batched.py 2>&1 | grep -E "smsp__|sm__|l1tex" >> $O
