"""Harness: fp64 GEMM (nseries_matmul) per tile configuration: NSERIES_F64_TILE = 1 (128x128),
3 (64x64), 0 (the library's choice); prints TFLOP/s and the fraction of the DMMA peak."""
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
    n = max(5, int(1e11 / (2 * d ** 3)))
    e0.record()
    for _ in range(n):
        P.nseries_matmul(h, X, Y, C, d)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    out[str(d)] = round(2.0 * d ** 3 / (ms * 1e-3) / 1e12 / 37.161, 3)
print(json.dumps(out))
