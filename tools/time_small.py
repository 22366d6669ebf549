"""Latency of small evaluations (config 1, d=64 fp64; config 2, d=1024) through the C ABI.
NSERIES_SMALL_WARPS selects the warps of the shared-memory small kernel (library knob)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_11843_b200 as P
from paper_2602_11843_b200 import inputs
h = P.nseries_create(0)
dims = [int(x) for x in os.environ.get("TIME_SMALL_D", "64,1024").split(",")]
for d, mk in ((64, lambda: torch.from_numpy(inputs.cfg1()).cuda()), (1024, lambda: torch.from_numpy(inputs.cfg2()).cuda())):
    if d not in dims:
        continue
    A = mk(); S = torch.empty_like(A)
    for steps, k in (([9, 9], 81), ([2] * 6, 64), ([5, 5, 5], 125), ([15, 15], 225)) if d == 64 else (([9, 9, 9], 729), ([5] * 4, 625), ([2] * 9, 512), ([2] * 10, 1024)):
        fl = P.NSERIES_ALLOW_APPROX if 15 in steps else 0
        plan = P.nseries_plan_finalize(steps, k, fl)
        for _ in range(5): P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        n = 200 if d == 64 else 20
        e0.record()
        for _ in range(n): P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        print(json.dumps({"d": d, "plan": steps, "warps": os.environ.get("NSERIES_SMALL_WARPS", "default"),
                          "us_per_eval": round(us, 1), "products": plan.products}), flush=True)
