"""Harness: engine efficiency across sizes (one fused-engine product through nseries_matmul,
CUDA events, device-resident inputs): fp64 TFLOP/s vs the DMMA peak, fp32 (3xTF32) algorithmic
and tensor TFLOP/s vs the TF32 peak, and the batched path across batch sizes.  Writes one JSON
object (profiles/r01_sweep.json)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402

FP64_PEAK, TF32_PEAK = 37.161, 1631.8 * 1.1 / 2.25
h = P.nseries_create(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


out = {"fp64_matmul": {}, "fp32_matmul": {}, "batched_x9x9_d32_fp32": {}}
g = torch.Generator(device="cuda").manual_seed(0)
for d in (512, 1024, 1536, 2048, 3072, 4096, 6144, 8192):
    for dt, key in ((torch.float64, "fp64_matmul"), (torch.float32, "fp32_matmul")):
        X = torch.randn(d, d, device="cuda", dtype=dt, generator=g)
        Y = torch.randn(d, d, device="cuda", dtype=dt, generator=g)
        C = torch.empty_like(X)
        n = max(3, int(2e11 / (2 * d ** 3)))
        ms = timed(lambda: P.nseries_matmul(h, X, Y, C, d), n)
        tf = 2.0 * d ** 3 / (ms * 1e-3) / 1e12
        rec = {"ms": round(ms, 4), "tflops": round(tf, 2)}
        if dt == torch.float64:
            rec["frac_of_dmma_peak"] = round(tf / FP64_PEAK, 3)
        else:
            rec["ms_includes"] = "2 plane-split launches + GEMM"
            rec["tf32_tensor_tflops"] = round(3 * tf, 1)
            rec["frac_of_tf32_peak"] = round(3 * tf / TF32_PEAK, 3)
        out[key][str(d)] = rec
        del X, Y, C
plan = P.nseries_plan_finalize([9, 9], 81, 0)
for B in (148, 1184, 4096, 16384, 65536):
    A = (torch.eye(32, device="cuda") * 0.5 + 0.02 * torch.randn(B, 32, 32, device="cuda", generator=g)).contiguous()
    S = torch.empty_like(A)
    ms = timed(lambda: P.nseries_eval_batched_strided(h, A, 1024, B, 32, 81, plan=plan, S=S), 10)
    out["batched_x9x9_d32_fp32"][str(B)] = {"us": round(ms * 1e3, 1), "matrices_per_s": round(B / (ms * 1e-3)),
                                           "hbm_gbs": round(2 * B * 4096 / (ms * 1e-3) / 1e9, 1)}
print(json.dumps(out))
