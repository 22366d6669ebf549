"""Harness: row-sharded chain (NEXT-3) on one GPU, all row blocks local: ms per eval against
the single-matrix engine, gathers per eval (env TIME_D, default 4096; plan x15^3 at 4096,
AUTO k=10000 at 8192); each block count also with NSERIES_SHARDED_DIRECT (no gathers)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402

d = int(os.environ.get("TIME_D", "4096"))
h = P.nseries_create(0)
g = torch.Generator(device="cuda").manual_seed(0)
A = (0.9 * torch.randn(d, d, device="cuda", dtype=torch.float64, generator=g) / d ** 0.5).contiguous()
if d <= 4096:
    k, plan = 3375, P.nseries_plan_finalize([15, 15, 15], 3375, P.NSERIES_ALLOW_APPROX)
else:
    k, plan = 10000, P.nseries_plan_build(10000, P.NSERIES_PLAN_AUTO, flags=P.NSERIES_ALLOW_APPROX)
fl = P.NSERIES_ALLOW_APPROX
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


S = torch.empty_like(A)
n_it = 3 if d <= 4096 else 1
dense = timed(lambda: P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl), n_it)
out = {"d": d, "k": k, "dense_ms": round(dense, 3)}
for n in (1, 2, 8):
    blocks = [P.nseries_shard_rows(d, n, s) for s in range(n)]
    As = [A[r0:r0 + m].contiguous() for r0, m in blocks]
    Ss = [torch.empty_like(a) for a in As]
    ms = timed(lambda: P.nseries_eval_sharded(h, As, 0, n, d, k, plan=plan, S_shards=Ss, flags=fl), n_it)
    st = P.nseries_last_stats(h)
    out[f"sharded{n}_ms"] = round(ms, 3)
    out[f"sharded{n}_gathers"] = st["gathers"]
    out[f"sharded{n}_prefetched"] = st["gathers_prefetched"]
    msd = timed(lambda: P.nseries_eval_sharded(h, As, 0, n, d, k, plan=plan, S_shards=Ss,
                                               flags=fl | P.NSERIES_SHARDED_DIRECT), n_it)
    out[f"sharded{n}_direct_ms"] = round(msd, 3)
    out[f"sharded{n}_direct_gathers"] = P.nseries_last_stats(h)["gathers"]
print(json.dumps(out))
