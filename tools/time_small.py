"""Latency of small evaluations (config 1, d=64 fp64) with and without CUDA-graph replay."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_11843_b200 as P
from paper_2602_11843_b200 import inputs
h = P.nseries_create(0)
for d, mk in ((64, lambda: torch.from_numpy(inputs.cfg1()).cuda()), (1024, lambda: torch.from_numpy(inputs.cfg2()).cuda())):
    A = mk(); S = torch.empty_like(A)
    for steps, k in (([9, 9], 81), ([2] * 6, 64), ([5, 5, 5], 125)) if d == 64 else (([9, 9, 9], 729), ([5] * 4, 625), ([2] * 9, 512), ([2] * 10, 1024)):
        plan = P.nseries_plan_finalize(steps, k, 0)
        for fl in (P.NSERIES_NO_GRAPH, 0):
            for _ in range(5): P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            n = 200 if d == 64 else 20
            e0.record()
            for _ in range(n): P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
            e1.record(); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / n * 1e3
            print(json.dumps({"d": d, "plan": steps, "graph": fl == 0, "us_per_eval": round(us, 1),
                              "products": plan.products, "stats": P.nseries_last_stats(h)}), flush=True)
