"""Harness: fp64 GEMM (nseries_matmul) per tile configuration NSERIES_F64_TILE (0 = library
choice, 1 = 128x128, 3 = 64x64, 4 = 32x32, 8 = stream-K 128x128, 9 = stream-K 64x64): fraction
of the DMMA peak, error vs torch (cuBLAS) and bit-identity of repeated products."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402

h = P.nseries_create(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {"tile": os.environ.get("NSERIES_F64_TILE", "0")}
g = torch.Generator(device="cuda").manual_seed(0)
for d in [int(x) for x in os.environ.get("TILE_D", "768,1024,1536,2048,3072,4096").split(",")]:
    X = torch.randn(d, d, device="cuda", dtype=torch.float64, generator=g)
    Y = torch.randn(d, d, device="cuda", dtype=torch.float64, generator=g)
    C = torch.empty_like(X)
    for _ in range(3):
        P.nseries_matmul(h, X, Y, C, d)
    torch.cuda.synchronize()
    C0 = C.clone()
    n = max(5, int(1e11 / (2 * d ** 3)))
    e0.record()
    for _ in range(n):
        P.nseries_matmul(h, X, Y, C, d)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    ref = X @ Y
    err = float((C - ref).norm() / ref.norm())
    same = bool(torch.equal(C, C0))
    out[str(d)] = [round(2.0 * d ** 3 / (ms * 1e-3) / 1e12 / 37.161, 3), f"{err:.1e}", same]
print(json.dumps(out), flush=True)
