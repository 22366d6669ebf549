"""Write the probe-column goldens of configs 3 and 5 (tests/golden/*.npz) -- calls ONLY oracle/.

For each (config, plan, dtype) below this script
  1. builds A on the CPU with inputs.cpu_reproducible (numpy + OpenBLAS pinned to one thread
     and its Haswell kernels, so the GPU box rebuilds the same bits; the SHA-256 of A is stored
     and the GPU test refuses a golden whose A hash differs),
  2. draws the 16-column probe block V = [e_j1..e_j8 | g_1..g_8] of SURVEY.md 8(c) C-3
     (inputs.probe_block(d, seed): default_rng(1000 + seed), seed = the config seed),
  3. runs the long-double oracle on it:
       exact plans      C-1  S_k(A) V = sum_{j<k} A^j V            (definition)
       radix-15 plans   C-2  Y_n V of the residual iteration
       config 5 AUTO    C-1  with the rigorous tail stop ||A||_2 <= 0.99 (reading R8)
     fp32 goldens use fl32(A) (the exact bits the GPU sees),
  4. stores S V as a double-double pair (SV_hi + SV_lo = the long-double result to ~1e-32) with
     the metadata (plan, k, oracle, A hash, V hash, threads, seconds).

No value here comes from the CUDA path.  Usage:
    python tools/make_goldens.py [name ...]          (default: every golden; ~1 h on 8 cores)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle import plan as OP  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")

# name -> (config, A-builder kwargs, probe seed, steps, dtype, oracle)
GOLDENS = {
    "cfg3_x15x3_f64": ("cfg3", {}, 2, [15, 15, 15], "f64", "C-2"),
    "cfg3_x9x4_f64": ("cfg3", {}, 2, [9, 9, 9, 9], "f64", "C-1"),
    "cfg3_x2x12_f64": ("cfg3", {}, 2, [2] * 12, "f64", "C-1"),
    "cfg3_x15x3_f32": ("cfg3", {}, 2, [15, 15, 15], "f32", "C-2"),
    "cfg3_x9x4_f32": ("cfg3", {}, 2, [9, 9, 9, 9], "f32", "C-1"),
    "cfg3_x2x12_f32": ("cfg3", {}, 2, [2] * 12, "f32", "C-1"),
    "cfg5_auto_f64": ("cfg5", {}, 4, [15, 1, 5, 5, 5, 5], "f64", "C-1 tail"),
}

CITES = {
    "C-1": "S_k(A) V = sum_{j<k} A^j V by long-double Horner (definition, PAPER.md:56-59, 137-139)",
    "C-2": "Y_n V of the radix plan's residual iteration Y' = Y f(R), R' = I - (I-A) Y' "
           "(PAPER.md:551-558), radix-15 kernel of PAPER.md:338-353 (polished, reading R1)",
    "C-1 tail": "C-1 truncated rigorously with ||A||_2 <= 0.99 (+1e-9): tail <= 1e-20 relative "
                "(DESIGN.md reading R8); the AUTO plan's deviation from S_k is below 1e-40",
}


def golden_path(name):
    return os.path.join(GOLDEN_DIR, name + ".npz")


def load_golden(name):
    """(SV as long double, metadata dict) of a committed golden."""
    z = np.load(golden_path(name))
    meta = json.loads(str(z["meta"]))
    sv = z["SV_hi"].astype(np.longdouble) + z["SV_lo"].astype(np.longdouble)
    return sv, meta


def make(name, cache):
    cfg, kw, pseed, steps, dt, oracle = GOLDENS[name]
    key = (cfg, tuple(sorted(kw.items())))
    if key not in cache:
        t = time.time()
        cache[key] = inputs.cpu_reproducible(cfg, **kw)
        print(f"[{name}] built A {cfg} in {time.time() - t:.1f}s", flush=True)
    A = cache[key]
    A_sha = inputs.sha256(A)
    if dt == "f32":
        A = A.astype(np.float32).astype(np.float64)     # fl32(A), widened exactly
    d = A.shape[0]
    V, idx = inputs.probe_block(d, pseed)
    k = OP.plan_reaches(steps)
    t = time.time()
    used = None
    if oracle == "C-2":
        SV = O.plan_apply(A, steps, V)
    elif oracle == "C-1":
        SV, used = O.series_sum(A, k, V)
    else:
        SV, used = O.series_sum(A, k, V, norm_bound=0.99 + 1e-9, tail_tol=1e-20)
    secs = time.time() - t
    hi = SV.astype(np.float64)
    lo = (SV - hi.astype(np.longdouble)).astype(np.float64)
    meta = {"name": name, "config": cfg, "d": d, "dtype": dt, "steps": steps, "k": k,
            "oracle": oracle, "cite": CITES[oracle], "A_sha256": A_sha,
            "A_builder": f"inputs.cpu_reproducible({cfg!r}, **{kw!r})", "A_env": inputs.REPRO_ENV,
            "probe_seed": pseed, "probe_cols": int(V.shape[1]), "probe_unit_idx": [int(i) for i in idx],
            "V_sha256": inputs.sha256(V), "terms_used": used, "oracle_threads": O.num_threads(),
            "oracle_seconds": round(secs, 1), "script": "tools/make_goldens.py"}
    os.makedirs(GOLDEN_DIR, exist_ok=True)
    np.savez_compressed(golden_path(name), SV_hi=hi, SV_lo=lo, meta=json.dumps(meta))
    print(f"[{name}] {oracle} k={k} {V.shape[1]} probes: {secs:.1f}s -> {golden_path(name)}", flush=True)
    return meta


def main(names):
    cache = {}
    manifest_path = os.path.join(GOLDEN_DIR, "MANIFEST.json")
    manifest = json.load(open(manifest_path)) if os.path.exists(manifest_path) else {}
    for n in names:
        meta = make(n, cache)
        manifest[n] = {k: meta[k] for k in ("config", "d", "dtype", "steps", "k", "oracle", "cite",
                                            "A_sha256", "probe_cols", "oracle_threads", "oracle_seconds")}
        with open(manifest_path, "w") as f:
            json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(GOLDENS))
