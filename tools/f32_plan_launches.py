"""Harness-only: one fp32 eval per plan at d=4096 (config-3 matrix) for an ncu launch list
(per-op kernel durations show how the epilogue cost scales with outputs / planes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_11843_b200 as P
d = 4096
h = P.nseries_create(0)
g = torch.Generator(device="cuda").manual_seed(2)
A = (torch.randn(d, d, device="cuda", generator=g) * (0.5 / d ** 0.5)).float()
S = torch.empty_like(A)
for steps, k in (([2] * 12, 4096), ([15, 15, 15], 3375), ([9] * 4, 6561)):
    flags = P.NSERIES_ALLOW_APPROX if 15 in steps else 0
    plan = P.nseries_plan_finalize(steps, k, flags)
    P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=flags | P.NSERIES_NO_GRAPH)
    torch.cuda.synchronize()
    print("plan", steps, flush=True)
