"""Harness: ms per eval of fp64 plans at several d (config 1/2/3 plans, Table-3 d = 500),
graph-replayed, 20 timed evals after 3 warm-ups.  NSERIES_PDL=0 / NSERIES_LIB for A/B."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402

h = P.nseries_create(0)
cases = [(64, [9, 9]), (500, [9, 9]), (500, [2] * 7), (1024, [9, 9, 9]), (1024, [5] * 4), (1024, [2] * 9),
         (1024, [2] * 10), (2048, [9, 9, 9]), (4096, [15, 15, 15])]
only = os.environ.get("ONLY_D")
out = []
for d, steps in cases:
    if only and str(d) not in only.split(","):
        continue
    g = torch.Generator(device="cuda").manual_seed(d)
    A = (0.9 * torch.randn(d, d, device="cuda", dtype=torch.float64, generator=g) / d ** 0.5).contiguous()
    S = torch.empty_like(A)
    k = 1
    for m in steps:
        k *= m
    fl = P.NSERIES_ALLOW_APPROX if 15 in steps else 0
    plan = P.nseries_plan_finalize(steps, k, fl)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20 if d <= 2048 else 5
    for _ in range(3):
        P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    tf = plan.products * 2 * d ** 3 / ms / 1e9
    out.append({"d": d, "steps": steps, "ms": round(ms, 4), "tflops": round(tf, 2), "frac_dmma": round(tf / 37.16, 3)})
print(json.dumps({"pdl": os.environ.get("NSERIES_PDL", "1"), "lib": os.environ.get("NSERIES_LIB", "default"), "runs": out}))
