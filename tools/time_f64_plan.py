"""Harness: fp64 x15^3 at d = 4096 (config-3 plan) ms per eval and one plain product."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402

d = 4096
h = P.nseries_create(0)
g = torch.Generator(device="cuda").manual_seed(0)
A = (0.9 * torch.randn(d, d, device="cuda", dtype=torch.float64, generator=g) / d ** 0.5).contiguous()
S = torch.empty_like(A)
plan = P.nseries_plan_finalize([15, 15, 15], 3375, P.NSERIES_ALLOW_APPROX)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    P.nseries_eval(h, A, d, 3375, plan=plan, S=S, flags=P.NSERIES_ALLOW_APPROX)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    P.nseries_eval(h, A, d, 3375, plan=plan, S=S, flags=P.NSERIES_ALLOW_APPROX)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"lib": os.environ.get("NSERIES_LIB", "default"), "x15^3_ms": round(e0.elapsed_time(e1) / 5, 3)}))
