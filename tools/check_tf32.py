"""Quick fp32 engine check (harness-only): C = X Y via 3xTF32 tcgen05 vs float64 reference."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_11843_b200 as P
h = P.nseries_create(0)
for d in [int(x) for x in (sys.argv[1:] or ["128", "256", "300", "1024", "4096"])]:
    g = torch.Generator(device="cuda").manual_seed(d)
    X = torch.randn(d, d, device="cuda", generator=g) / d ** 0.5
    Y = torch.randn(d, d, device="cuda", generator=g) / d ** 0.5
    C = torch.zeros_like(X)
    P.nseries_matmul(h, X, Y, C, d)
    torch.cuda.synchronize()
    ref = X.double() @ Y.double()
    err = float((C.double() - ref).norm() / ref.norm())
    bias = float(((C.double() - ref) * ref.sign()).mean() / ref.abs().mean())
    t = None
    if d >= 1024:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): P.nseries_matmul(h, X, Y, C, d)
        e1.record(); torch.cuda.synchronize(); t = e0.elapsed_time(e1) / 10
    print(f"d={d} rel_err={err:.3e} bias={bias:.2e} ms={t}", flush=True)
