"""Harness-only: a few fp64 d=4096 products through nseries_matmul (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_11843_b200 as P
h = P.nseries_create(0)
d = 4096
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(d, d, device="cuda", dtype=torch.float64, generator=g) / 64
Y = torch.randn(d, d, device="cuda", dtype=torch.float64, generator=g) / 64
C = torch.empty_like(X)
for _ in range(3):
    P.nseries_matmul(h, X, Y, C, d, dtype=P.NSERIES_F64)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10):
    P.nseries_matmul(h, X, Y, C, d, dtype=P.NSERIES_F64)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"fp64 matmul d=4096: {ms:.3f} ms = {2*d**3/ms/1e9:.1f} TFLOP/s")
