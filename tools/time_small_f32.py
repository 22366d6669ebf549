"""Harness: small fp32 single-matrix evaluation (d <= 64): nseries_eval (tiled engine) vs the
batched kernels with batch = 1, us per eval."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

h = P.nseries_create(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for d in (16, 32, 48, 64):
    A = torch.from_numpy(inputs.random_matrix(d, 5, 0.7)).float().cuda()
    S = torch.empty_like(A)
    plan = P.nseries_plan_finalize([9, 9], 81, 0)
    t_eval = timed(lambda: P.nseries_eval(h, A, d, 81, plan=plan, S=S))
    t_b = timed(lambda: P.nseries_eval_batched_strided(h, A, d * d, 1, d, 81, plan=plan, S=S))
    print(json.dumps({"d": d, "eval_us": round(t_eval, 1), "batched1_us": round(t_b, 1)}))
