"""Config 4 timing (harness-only): 16384 x 32x32 fp32 batched, one launch per eval.
NSERIES_BATCHED_WPM selects warps per matrix (library tuning knob); NSERIES_LIB an A/B build.
Also prints the worst relative Frobenius error over a 512-matrix sample against an fp64 torch
power-sum reference (sanity for A/B variants; parity lives in tests/)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_11843_b200 as P
from paper_2602_11843_b200 import inputs
h = P.nseries_create(0)
Ab = torch.from_numpy(inputs.cfg4()).cuda()
S = torch.empty_like(Ab)
B, d = Ab.shape[0], Ab.shape[1]
samp = torch.arange(0, B, 1 if os.environ.get("ALL") else B // 512, device="cuda")
A64 = Ab[samp].double()


def ref_series(k):
    W = torch.eye(d, dtype=torch.float64, device="cuda").expand_as(A64).clone()
    out = W.clone()
    for _ in range(k - 1):
        W = torch.bmm(A64, W)
        out += W
    return out


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
    R = ref_series(k)
    errs = (S[samp].double() - R).flatten(1).norm(dim=1) / R.flatten(1).norm(dim=1)
    err = errs.max().item()
    if os.environ.get("ALL"):
        top = torch.topk(errs, 5)
        print("worst matrices", [(int(samp[i]), float(v)) for v, i in zip(top.values, top.indices)],
              "p99", float(torch.quantile(errs.float(), 0.99)), "n>2e-5", int((errs > 2e-5).sum()))
    print(json.dumps({"lib": os.path.basename(os.environ.get("NSERIES_LIB", "libnseries.so")),
                      "wpm": os.environ.get("NSERIES_BATCHED_WPM", "default"), "plan": steps, "k": k,
                      "us": round(us, 1), "matrices_per_s": B / us * 1e6,
                      "hbm_gbs": 2 * B * d * d * 4 / us / 1e3,
                      "tflops_alg": plan.products * 2 * d ** 3 * B / us / 1e6, "max_rel_err": err}))
