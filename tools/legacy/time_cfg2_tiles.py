"""Harness: config-2 plans (d = 1024 fp64, BASELINE.json configs[1]) per fp64 tile configuration
NSERIES_F64_TILE (0 = library choice, 4 = 32x32 / 16x16 warps, 10 = 32x32 with 4 warps on the
whole tile over 1/4 of K each, 11 = 32x32 with 32x16 warp tiles over 1/2 of K, 12 = 64x64 with
32x32 warp tiles over 1/2 of K): ms per eval, fraction of the DMMA peak, and the largest relative
difference from the library-choice result (set TILE_REF=1 to store it, else read)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

PEAK = 37.161
h = P.nseries_create(0)
A = torch.from_numpy(inputs.cfg2()).cuda()
S = torch.empty_like(A)
stream = torch.cuda.current_stream()
out = {"tile": os.environ.get("NSERIES_F64_TILE", "0")}
ref_path = "gpurun_out/cfg2_ref.pt"
refs = torch.load(ref_path) if os.path.exists(ref_path) and not os.environ.get("TILE_REF") else {}
new_refs = {}
for name, (stp, kk) in {"x9^3": ([9] * 3, 729), "x5^4": ([5] * 4, 625), "x2^10": ([2] * 10, 1024)}.items():
    plan = P.nseries_plan_finalize(stp, kk, 0)
    for _ in range(3):
        P.nseries_eval(h, A, 1024, kk, plan=plan, S=S, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 30
    e0.record(stream)
    for _ in range(n):
        P.nseries_eval(h, A, 1024, kk, plan=plan, S=S, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    frac = plan.products * 2.0 * 1024 ** 3 / (ms * 1e-3) / 1e12 / PEAK
    diff = None
    if name in refs:
        r = refs[name].cuda()
        diff = float(((S - r).abs().max() / r.abs().max()).item())
    new_refs[name] = S.cpu().clone()
    out[name] = [round(ms, 4), round(frac, 4), diff]
if os.environ.get("TILE_REF"):
    torch.save(new_refs, ref_path)
print(json.dumps(out), flush=True)
