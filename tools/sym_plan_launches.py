"""Harness-only: one fp64 and one fp32 x15^3 eval with NSERIES_SYMMETRIC at d=4096 on config 3
(for ncu launch lists / full captures of the symmetric-mode kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_11843_b200 as P
from paper_2602_11843_b200 import inputs
h = P.nseries_create(0)
A, _, _ = inputs.cfg3(device="cuda")
for dt in (torch.float64, torch.float32):
    Ad = A.to(dt).contiguous()
    S = torch.empty_like(Ad)
    fl = P.NSERIES_ALLOW_APPROX | P.NSERIES_SYMMETRIC | P.NSERIES_NO_GRAPH
    plan = P.nseries_plan_finalize([15, 15, 15], 3375, fl)
    P.nseries_eval(h, Ad, 4096, 3375, plan=plan, S=S, flags=fl)
    torch.cuda.synchronize()
    print(dt, "ok", flush=True)
