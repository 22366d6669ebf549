"""Quick engine timing (harness-only): nseries_matmul and full plan evals, CUDA events."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_11843_b200 as P
from paper_2602_11843_b200 import build as B
B.build()
h = P.nseries_create(0)
out = {}
for d in [int(x) for x in (sys.argv[1:] or ["1024", "2048", "4096", "8192"])]:
    X = torch.randn(d, d, dtype=torch.float64, device="cuda") / d ** 0.5
    Y = torch.randn(d, d, dtype=torch.float64, device="cuda") / d ** 0.5
    C = torch.empty_like(X)
    for _ in range(3): P.nseries_matmul(h, X, Y, C, d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = max(3, int(2e12 / (2 * d ** 3)))
    e0.record()
    for _ in range(n): P.nseries_matmul(h, X, Y, C, d)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    ref = X @ Y
    err = float((C - ref).norm() / ref.norm())
    out[f"matmul_{d}"] = {"ms": ms, "tflops": 2 * d ** 3 / ms / 1e9, "rel_err_vs_cublas": err}
    print(json.dumps({f"matmul_{d}": out[f"matmul_{d}"]}), flush=True)
d = 4096
A = (torch.randn(d, d, dtype=torch.float64, device="cuda") * (0.9 / d ** 0.5))
S = torch.empty_like(A)
for steps in ([15, 15, 15], [9, 9, 9, 9], [2] * 12):
    k = 1
    for s in steps: k *= s
    fl = P.NSERIES_ALLOW_APPROX if 15 in steps else 0
    plan = P.nseries_plan_finalize(steps, k, fl)
    P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3): P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    prods = plan.products
    print(json.dumps({"plan": steps, "k": k, "ms": ms, "products": prods,
                      "tflops": prods * 2 * d ** 3 / ms / 1e9}), flush=True)
P.nseries_destroy(h)
