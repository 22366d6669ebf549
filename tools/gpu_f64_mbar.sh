# fp64 engine: mbarrier k-tile pipeline (current tree) vs the per-k-tile __syncthreads pipeline
# (tools/variants/f64_nombar.so), alternating; then the full GPU suite; batched probe
mkdir -p gpurun_out
O=gpurun_out/f64_mbar.txt
: > $O
for i in 1 2; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/f64_nombar.so; do
    echo "== $lib" >> $O
    NSERIES_LIB=$lib timeout 200 python tools/time_plans_f64.py >> $O 2>&1
    NSERIES_LIB=$lib TILE_D=1024,2048,4096,8192 timeout 200 python tools/time_f64_sk.py >> $O 2>&1
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f64_mbar_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/f64_mbar_tests.log
(nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DNSERIES_BW_PROBE=0 -Iinclude -o /tmp/bwp0 tools/bw_probe.cu paper_2602_11843_b200/csrc/plan.cc paper_2602_11843_b200/csrc/compile.cc && \
 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DNSERIES_BW_PROBE=1 -Iinclude -o /tmp/bwp1 tools/bw_probe.cu paper_2602_11843_b200/csrc/plan.cc paper_2602_11843_b200/csrc/compile.cc && \
 timeout 100 /tmp/bwp0 && timeout 100 /tmp/bwp1) > gpurun_out/bw_probe.txt 2>&1
