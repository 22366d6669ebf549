# ncu source-level capture of the batched config-4 kernel (per-instruction executed counts + stalls)
mkdir -p gpurun_out
timeout 200 python tools/time_batched.py > gpurun_out/bw_time.txt 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:batched_warp -s 3 -c 1 -o gpurun_out/bw_src -f python tools/time_batched.py > gpurun_out/bw_src_ncu.log 2>&1
