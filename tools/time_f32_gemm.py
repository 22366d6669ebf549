"""Harness: fp32 (3xTF32) engine timing through nseries_matmul and an x15^3 eval at d (env
TIME_D, default 4096); NSERIES_TF32_SPLITK=0 disables the split-K tail for comparison."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_11843_b200 import _binding as P, inputs  # noqa: E402

d = int(os.environ.get("TIME_D", "4096"))
h = P.nseries_create(0)
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(d, d, device="cuda", generator=g)
Y = torch.randn(d, d, device="cuda", generator=g)
C = torch.empty_like(X)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    P.nseries_matmul(h, X, Y, C, d)
torch.cuda.synchronize()
n = 20
e0.record()
for _ in range(n):
    P.nseries_matmul(h, X, Y, C, d)
e1.record()
torch.cuda.synchronize()
mm = e0.elapsed_time(e1) / n
A = (0.9 * X / d ** 0.5).contiguous()
plan = P.nseries_plan_finalize([15, 15, 15], 3375, P.NSERIES_ALLOW_APPROX)
S = torch.empty_like(A)
for _ in range(3):
    P.nseries_eval(h, A, d, 3375, plan=plan, S=S, flags=P.NSERIES_ALLOW_APPROX)
torch.cuda.synchronize()
n = 5
e0.record()
for _ in range(n):
    P.nseries_eval(h, A, d, 3375, plan=plan, S=S, flags=P.NSERIES_ALLOW_APPROX)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"d": d, "splitk": os.environ.get("NSERIES_TF32_SPLITK", "1"), "matmul_ms": round(mm, 4),
                  "x15^3_ms": round(e0.elapsed_time(e1) / n, 3)}))
