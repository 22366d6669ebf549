"""Diagnose fp32 plan accuracy at config 3 (harness-only): nseries fp32 vs a plain-fp32 torch
evaluation of the same circuits, both against nseries fp64 on fl32(A)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_11843_b200 as P
from paper_2602_11843_b200 import inputs
torch.backends.cuda.matmul.allow_tf32 = False
h = P.nseries_create(0)
A64, _, _ = inputs.cfg3(device="cuda")
A32 = A64.float().contiguous()
A = A32.double().contiguous()
d = A.shape[0]
r15 = [float(x) for x in P.nseries_kernel_info(15)["coeffs"]]  # (only to confirm availability)
import re
src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2602_11843_b200/csrc/plan.cc")).read()
blk = src[src.index("kRadix15 = {"):src.index("};", src.index("kRadix15 = {"))]
nums = [float(x) for x in re.findall(r"-?\d+\.\d+(?:e-?\d+)?", blk)]
L2, R2, L3, R3, L4, R4, g = nums[0:3], nums[3:6], nums[6:10], nums[10:14], nums[14:19], nums[19:24], nums[24:28]

def circuit(Y, R, A, step, tele=False):
    I = torch.eye(d, dtype=Y.dtype, device=Y.device)
    if step == 15:
        P1 = R @ R
        B2 = [I, R, P1]
        lin = lambda w, B: sum(wi * Bi for wi, Bi in zip(w, B))
        P2 = lin(L2, B2) @ lin(R2, B2); B3 = B2 + [P2]
        P3 = lin(L3, B3) @ lin(R3, B3); B4 = B3 + [P3]
        P4 = lin(L4, B4) @ lin(R4, B4)
        f = I + g[0] * R + g[1] * P1 + g[2] * P2 + g[3] * P3 + P4
        Yn = Y @ f
        Rn = (I - f + f @ R) if tele else (I - Yn + A @ Yn)
        return Yn, Rn
    if step == 9:
        U = R @ R; V = U @ (R + 2 * U)
        Pm = 0.15 * R + 2 * U + V; Q = 0.275 * R - 0.125 * U + 0.25 * V
        T = Pm @ Q + I + R + (767 / 800) * U + (15 / 32) * V
    elif step == 2:
        T = I + R
    return Y @ T, I - T + T @ R

for steps in ([15, 15, 15], [9, 9, 9, 9], [2] * 12):
    k = 1
    for s in steps: k *= s
    fl = P.NSERIES_ALLOW_APPROX if 15 in steps else 0
    plan = P.nseries_plan_finalize(steps, k, fl)
    S64 = torch.empty_like(A); P.nseries_eval(h, A, d, k, plan=plan, S=S64, flags=fl)
    S32 = torch.empty_like(A32); P.nseries_eval(h, A32, d, k, plan=plan, S=S32, flags=fl)
    torch.cuda.synchronize()
    e_ours = float((S32.double() - S64).norm() / S64.norm())
    for dt in (torch.float32, torch.float64):
        Y = torch.eye(d, dtype=dt, device="cuda"); R = A.to(dt)
        for s in steps: Y, R = circuit(Y, R, A.to(dt), s)
        e_t = float((Y.double() - S64).norm() / S64.norm())
        print(f"{steps[0]}x{len(steps)}: nseries fp32 err {e_ours:.3e} | torch {dt} circuit err {e_t:.3e}", flush=True)
    if 15 in steps:
        Y = torch.eye(d, dtype=torch.float32, device="cuda"); R = A32.clone()
        for s in steps: Y, R = circuit(Y, R, A32, s, tele=True)
        print(f"   torch fp32 telescope R-form err {float((Y.double() - S64).norm() / S64.norm()):.3e}")
