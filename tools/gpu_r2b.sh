# Harness: tcgen05 drain microbenchmark + ncu of the fp64 32x32-tile kernel at d = 1024
mkdir -p gpurun_out
timeout 120 ./tools/drain_rate > gpurun_out/drain_rate.txt 2>&1; echo "rc=$?" >> gpurun_out/drain_rate.txt
cat > /tmp/one1024.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2602_11843_b200 as P
h = P.nseries_create(0)
d = 1024
X = torch.randn(d, d, device="cuda", dtype=torch.float64) / 32
Y = torch.randn(d, d, device="cuda", dtype=torch.float64) / 32
C = torch.empty_like(X)
for _ in range(6):
    P.nseries_matmul(h, X, Y, C, d, dtype=P.NSERIES_F64)
torch.cuda.synchronize()
PY
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 3 -c 1 -o gpurun_out/f64_d1024 -f python /tmp/one1024.py > gpurun_out/ncu_f64_1024.log 2>&1
for t in 3 4; do NSERIES_F64_TILE=$t timeout 300 ncu --set full --clock-control none -k regex:gemm_f64 -s 3 -c 1 -o gpurun_out/f64_d1024_t$t -f python /tmp/one1024.py >> gpurun_out/ncu_f64_1024.log 2>&1; done
