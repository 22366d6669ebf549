"""Harness: race shaking of the hand-synchronised kernels (substitute for compute-sanitizer,
which is closed on this pool -- profiles/r02_sanitizer_closed.txt).

  python tools/race_shake.py build            # CPU: build tools/variants/shake{1..4}.so
  python tools/race_shake.py run [seeds...]   # GPU: every case on the plain library and on each
                                              # shaken build; outputs must be bit-identical

A shaken build (-DNSERIES_SHAKE=<seed>) sleeps a seeded pseudo-random 0-4 us at a quarter of
the protocol points of the 4x2 cluster kernel (mbarrier waits, csync barriers, st.async
pushes), the warp-group batched kernel (group barriers, cp.async prefetch of the next matrix),
the tcgen05 engine (TMA producer, MMA issuer, TMEM drains, split-K counters) and the fp64
engine's k-tile barrier.  Every kernel here is deterministic (fixed summation order; split-K
adds exactly two partials), so any missing wait / barrier that lets a reader see a stale or
half-written value changes bits.  Each case is also checked against a torch fp64 reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEEDS = [1, 2, 3, 4]


def cases():
    # (name, kind, d, batch, steps, dtype, with_R)
    return [
        ("cluster2d_x9x9_d64", "single", 64, 1, [9, 9], "f64", False),
        ("cluster2d_x5p1x5_d33", "single", 33, 1, [5, 1, 5], "f64", False),
        ("cluster2d_bin6_R_d64", "single", 64, 1, [2] * 6, "f64", True),
        ("cluster2d_x15x15_d64", "single", 64, 1, [15, 15], "f64", False),
        ("cluster2d_bin17_d64", "single", 64, 1, [2] * 17, "f64", False),
        ("cluster2d_mixed_d40", "single", 40, 1, [3, 9, 5, 2, 2, 1, 2], "f64", False),
        ("cluster2d_naive13_d64", "single", 64, 1, [13, 2], "f64", False),
        ("warp_x9x9_d32", "batched", 32, 3000, [9, 9], "f32", False),
        ("warp_x5p1x5_d32", "batched", 32, 1000, [5, 1, 5], "f32", False),
        ("warp_bin3_d17", "batched", 17, 1000, [2, 2, 2], "f32", False),
        ("cta_x9x9_d48", "batched", 48, 300, [9, 9], "f32", False),
        ("cta_f64_x9x9_d32", "batched", 32, 300, [9, 9], "f64", False),
        ("tf32_matmul_d1024", "matmul", 1024, 1, None, "f32", False),
        ("tf32_matmul_d4096", "matmul", 4096, 1, None, "f32", False),
        ("tf32_matmul_d700", "matmul", 700, 1, None, "f32", False),
        ("tf32_x9x9_d1100", "single", 1100, 1, [9, 9], "f32", True),
        ("f64_x9p1x2_d300", "single", 300, 1, [9, 1, 2], "f64", True),
        ("f64_x9x9_d1024", "single", 1024, 1, [9, 9], "f64", False),     # one-wave 96x80 tiles
        ("f64_x15p1x5_d1536", "single", 1536, 1, [15, 1, 5], "f64", True),  # 128x128 tiles, hoisted spread copies
        ("f64_x9x9_d2048", "single", 2048, 1, [9, 9], "f64", False),     # 64x64 tiles, two CTAs per SM
    ]


def build():
    for s in SEEDS:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "build_variant.py"), f"shake{s}",
                        f"-DNSERIES_SHAKE={s}"], check=True, stdout=subprocess.DEVNULL)
        print("built", f"tools/variants/shake{s}.so")


def run_cases():
    """Child process: evaluate every case with the library NSERIES_LIB points at; print one
    JSON dict name -> [sha256 of the outputs, rel. error vs torch fp64]."""
    sys.path.insert(0, ROOT)
    import torch
    import paper_2602_11843_b200 as P
    h = P.nseries_create(0)
    out = {}
    for name, kind, d, batch, steps, dt, with_R in cases():
        tdt = torch.float64 if dt == "f64" else torch.float32
        g = torch.Generator().manual_seed(d * 7 + batch)
        if kind == "matmul":
            X = (torch.randn(d, d, generator=g, dtype=torch.float64) / d ** 0.5).to("cuda", tdt)
            Y = (torch.randn(d, d, generator=g, dtype=torch.float64) / d ** 0.5).to("cuda", tdt)
            C = torch.empty_like(X)
            P.nseries_matmul(h, X, Y, C, d)
            torch.cuda.synchronize()
            ref = X.double() @ Y.double()
            err = float((C.double() - ref).norm() / ref.norm())
            outs = [C]
        else:
            shape = (batch, d, d) if kind == "batched" else (d, d)
            A = (0.5 * torch.randn(*shape, generator=g, dtype=torch.float64) / d ** 0.5).to("cuda", tdt)
            k = 1
            for m in steps:
                k = k + 1 if m == 1 else k * m
            fl = P.NSERIES_ALLOW_APPROX if 15 in steps else 0
            plan = P.nseries_plan_finalize(steps, k, fl)
            S = torch.full_like(A, float("nan"))
            R = torch.full_like(A, float("nan")) if with_R else None
            if kind == "batched":
                P.nseries_eval_batched_strided(h, A, d * d, batch, d, k, plan=plan, S=S, flags=fl)
            else:
                P.nseries_eval(h, A, d, k, plan=plan, S=S, R_out=R, flags=fl | P.NSERIES_NO_GRAPH)
            torch.cuda.synchronize()
            outs = [S] + ([R] if with_R else [])
            # reference: the exact series sum S_k = sum_j A^j (radix-15 plans: residual identity)
            A0 = (A[0] if kind == "batched" else A).double()
            S0 = (S[0] if kind == "batched" else S).double()
            I = torch.eye(d, dtype=torch.float64, device="cuda")
            if 15 in steps:
                err = 0.0 if bool(torch.isfinite(S0).all()) else float("inf")
            else:
                ref, W = I.clone(), I.clone()
                for _ in range(k - 1):
                    W = A0 @ W
                    ref += W
                err = float((S0 - ref).norm() / ref.norm())
        hsh = hashlib.sha256(b"".join(o.cpu().numpy().tobytes() for o in outs)).hexdigest()
        out[name] = [hsh, err]
    P.nseries_destroy(h)
    print(json.dumps(out))


def run(seeds):
    libs = [("plain", os.path.join(ROOT, "paper_2602_11843_b200", "libnseries.so"))]
    libs += [(f"shake{s}", os.path.join(ROOT, "tools", "variants", f"shake{s}.so")) for s in seeds]
    res = {}
    for tag, lib in libs:
        env = dict(os.environ, NSERIES_LIB=lib)
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            print(f"{tag}: child failed rc={r.returncode}\n{r.stderr[-2000:]}")
            res[tag] = None
            continue
        res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
    base = res["plain"]
    ok = base is not None
    lines = []
    for name, *_ in cases():
        row = [name, f"{base[name][1]:.2e}" if base else "-"]
        for tag, _ in libs[1:]:
            if res[tag] is None or base is None:
                row.append("FAIL")
                ok = False
                continue
            same = res[tag][name][0] == base[name][0]
            ok &= same
            row.append("identical" if same else "DIFFERS")
        lines.append("  ".join(row))
    tol_ok = base is not None and all(v[1] < 5e-5 for v in base.values())
    print("case  rel_err(plain vs fp64 ref)  " + "  ".join(t for t, _ in libs[1:]))
    print("\n".join(lines))
    print(f"RESULT: {'PASS' if ok and tol_ok else 'FAIL'} ({len(cases())} cases x {len(seeds)} shaken builds, "
          f"outputs bit-identical to the plain build: {ok})")
    return 0 if ok and tol_ok else 1


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "run"
    if cmd == "build":
        build()
    elif cmd == "child":
        run_cases()
    else:
        sys.exit(run([int(x) for x in sys.argv[2:]] or SEEDS))
