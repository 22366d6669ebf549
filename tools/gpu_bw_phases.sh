# batched kernel phase timing (clock64 per warp-op) and mainloop experiments (timing only)
mkdir -p gpurun_out
O=gpurun_out/bw_phases.txt
: > $O
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/bw_probe.cu paper_2602_11843_b200/csrc/plan.cc paper_2602_11843_b200/csrc/compile.cc"
for v in "-DNSERIES_BW_PROBE=0 -DNSERIES_BW_TIMING" "-DNSERIES_BW_PROBE=1 -DNSERIES_BW_TIMING" \
         "-DNSERIES_BW_PROBE=0" "-DNSERIES_BW_PROBE=0 -DNSERIES_BW_CHAIN_BIG" "-DNSERIES_BW_PROBE=0 -DNSERIES_BW_NOSPLIT" \
         "-DNSERIES_BW_PROBE=1 -DNSERIES_BW_NOSPLIT" "-DNSERIES_BW_PROBE=1 -DNSERIES_BW_CHAIN_BIG -DNSERIES_BW_NOSPLIT"; do
  echo "=== $v" >> $O
  $B $v -o /tmp/bwx >> $O 2>&1 && timeout 100 /tmp/bwx 2>&1 | grep -v "delay [248]00" >> $O
done
