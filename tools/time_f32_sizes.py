"""Harness: fp32 engine (nseries_matmul, incl. the two plane-split launches) across d:
fraction of the TF32 peak of the 3xTF32 tensor rate (3 x 2 d^3 per product)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402

TF32_PEAK = 1631.8 * 1.1 / 2.25
h = P.nseries_create(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {}
g = torch.Generator(device="cuda").manual_seed(0)
for d in [int(x) for x in os.environ.get("F32_D", "512,768,1024,1280,1536,1664,2048,4096").split(",")]:
    X = torch.randn(d, d, device="cuda", generator=g)
    Y = torch.randn(d, d, device="cuda", generator=g)
    C = torch.empty_like(X)
    for _ in range(3):
        P.nseries_matmul(h, X, Y, C, d)
    torch.cuda.synchronize()
    n = max(5, int(3e11 / (2 * d ** 3)))
    e0.record()
    for _ in range(n):
        P.nseries_matmul(h, X, Y, C, d)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    out[str(d)] = {"ms": round(ms, 4), "tf32_frac": round(3 * 2.0 * d ** 3 / (ms * 1e-3) / 1e12 / TF32_PEAK, 3)}
print(json.dumps(out))
