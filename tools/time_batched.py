"""Config 4 timing (harness-only): 16384 x 32x32 fp32 batched, one launch per eval.
NSERIES_BATCHED_WPM selects warps per matrix (library tuning knob)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_11843_b200 as P
from paper_2602_11843_b200 import inputs
h = P.nseries_create(0)
Ab = torch.from_numpy(inputs.cfg4()).cuda()
S = torch.empty_like(Ab)
B, d = Ab.shape[0], Ab.shape[1]
for steps, k in (([9, 9], 81), ([5, 5], 25)):
    plan = P.nseries_plan_finalize(steps, k, 0)
    for _ in range(3): P.nseries_eval_batched_strided(h, Ab, d * d, B, d, k, plan=plan, S=S)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 20
    e0.record()
    for _ in range(n): P.nseries_eval_batched_strided(h, Ab, d * d, B, d, k, plan=plan, S=S)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    print(json.dumps({"wpm": os.environ.get("NSERIES_BATCHED_WPM", "default"), "plan": steps, "k": k,
                      "us": round(us, 1), "matrices_per_s": B / us * 1e6,
                      "hbm_gbs": 2 * B * d * d * 4 / us / 1e3,
                      "tflops_alg": plan.products * 2 * d ** 3 * B / us / 1e6}))
