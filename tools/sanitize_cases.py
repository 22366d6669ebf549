"""Harness: small evaluations that drive each hand-synchronised kernel once, for
compute-sanitizer (memcheck / racecheck / synccheck).  Run under the sanitizer as

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py CASE

CASE in: cluster2d, warp_f32, cta_f32, cta_f64, splitk_f32, tf32, f64_tiled.
Every case checks its result against a torch fp64 product chain (sanity only; parity lives in
tests/) and exits non-zero on a mismatch.  No graphs (NSERIES_NO_GRAPH): each op is its own
launch so the sanitizer attributes every report to one kernel.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_11843_b200 as P  # noqa: E402


def series_ref(A, steps):
    """S_k(A) by S_{mn} = S_n (I + B + ... + B^{m-1}), B = A^n, in fp64 torch (sanity
    reference for the harness only; exact steps)."""
    A = A.double()
    I = torch.eye(A.shape[0], dtype=torch.float64, device=A.device)
    S, B = I.clone(), A.clone()
    for m in steps:
        if m == 1:
            S, B = S + B, B @ A
            continue
        T, P = I.clone(), I.clone()
        for _ in range(m - 1):
            P = P @ B
            T = T + P
        S, B = S @ T, P @ B
    return S


def rel(a, b):
    return float((a.double() - b).norm() / b.norm())


def run_single(h, d, steps, dt, tol, flags=0, R=False):
    g = torch.Generator().manual_seed(d)
    A = (0.5 * torch.randn(d, d, generator=g, dtype=torch.float64) / d ** 0.5).cuda()
    if dt == P.NSERIES_F32:
        A = A.float()
    k = 1
    for s in steps:
        k = k + 1 if s == 1 else k * s
    plan = P.nseries_plan_finalize(steps, k, flags)
    S = torch.empty_like(A)
    Rb = torch.empty_like(A) if R else None
    P.nseries_eval(h, A, d, k, plan=plan, S=S, R_out=Rb, flags=flags | P.NSERIES_NO_GRAPH)
    torch.cuda.synchronize()
    if 15 in steps:
        return  # approximate plan: the sanitizer report is what matters here
    e = rel(S, series_ref(A, steps))
    print(f"d={d} steps={steps} dt={dt} rel={e:.2e}")
    if e > tol:
        raise SystemExit(f"mismatch {e}")


def run_batched(h, d, batch, steps, dt, tol):
    g = torch.Generator().manual_seed(batch)
    A = (0.5 * torch.randn(batch, d, d, generator=g, dtype=torch.float64) / d ** 0.5).cuda()
    if dt == P.NSERIES_F32:
        A = A.float()
    k = 1
    for s in steps:
        k = k + 1 if s == 1 else k * s
    plan = P.nseries_plan_finalize(steps, k, 0)
    S = torch.empty_like(A)
    P.nseries_eval_batched_strided(h, A, d * d, batch, d, k, plan=plan, S=S, strideS=d * d)
    torch.cuda.synchronize()
    worst = max(rel(S[b], series_ref(A[b], steps)) for b in range(0, batch, max(1, batch // 8)))
    print(f"batched d={d} batch={batch} steps={steps} rel={worst:.2e}")
    if worst > tol:
        raise SystemExit(f"mismatch {worst}")


def main(case):
    h = P.nseries_create(0)
    ap = P.NSERIES_ALLOW_APPROX
    try:
        if case == "cluster2d":
            for d in (33, 64):
                run_single(h, d, [9, 9], P.NSERIES_F64, 1e-12)
                run_single(h, d, [5, 1, 5], P.NSERIES_F64, 1e-12)
                run_single(h, d, [2] * 6, P.NSERIES_F64, 1e-12, R=True)
                run_single(h, d, [15, 15], P.NSERIES_F64, 0, flags=ap)
            # a long plan (> 32 ops): per-op mbarriers and decode beyond one warp's ops
            run_single(h, 64, [2] * 17, P.NSERIES_F64, 1e-11)
            run_single(h, 40, [3, 9, 5, 2, 2, 1, 2], P.NSERIES_F64, 1e-11)
        elif case == "warp_f32":
            run_batched(h, 32, 600, [9, 9], P.NSERIES_F32, 5e-5)
            run_batched(h, 32, 300, [5, 1, 5], P.NSERIES_F32, 5e-5)
            run_batched(h, 17, 200, [2, 2, 2], P.NSERIES_F32, 5e-5)
        elif case == "cta_f32":
            run_batched(h, 48, 40, [9, 9], P.NSERIES_F32, 5e-5)
            run_batched(h, 64, 20, [5, 5], P.NSERIES_F32, 5e-5)
        elif case == "cta_f64":
            run_batched(h, 32, 40, [9, 9], P.NSERIES_F64, 1e-12)
        elif case == "splitk_f32":
            for d in (1024, 700):
                X = torch.randn(d, d, device="cuda") / d ** 0.5
                Y = torch.randn(d, d, device="cuda") / d ** 0.5
                C = torch.empty_like(X)
                P.nseries_matmul(h, X, Y, C, d)
                torch.cuda.synchronize()
                e = rel(C, X.double() @ Y.double())
                print(f"matmul f32 d={d} rel={e:.2e}")
                if e > 1e-5:
                    raise SystemExit(f"mismatch {e}")
        elif case == "tf32":
            run_single(h, 200, [9, 9], P.NSERIES_F32, 5e-5)
            run_single(h, 130, [15, 1, 2], P.NSERIES_F32, 0, flags=ap)
            run_single(h, 64, [5, 5], P.NSERIES_F32, 5e-5, R=True)
        elif case == "f64_tiled":
            run_single(h, 200, [9, 1, 2], P.NSERIES_F64, 1e-12)
            run_single(h, 130, [15, 5], P.NSERIES_F64, 0, flags=ap)
        else:
            raise SystemExit(f"unknown case {case}")
    finally:
        P.nseries_destroy(h)
    print(f"case {case} ok")


if __name__ == "__main__":
    main(sys.argv[1])
