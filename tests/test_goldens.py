"""CPU pins of the committed oracle goldens (tests/golden/, written by tools/make_goldens.py).

The goldens are oracle output, so they are pinned to something other than the oracle itself:
  - config 3 is symmetric with a known factorisation A = Q diag(ev) Q^T (inputs.cfg3 returns Q
    and ev): S_k(A) V = Q diag(s_k(ev)) Q^T V with the geometric-series closed form
    s_k(x) = (1 - x^k) / (1 - x) for exact plans, and for the radix-15 plan
    the paper's residual recursion run on each eigenvalue as a SCALAR,
    y' = y f(r), r' = 1 - (1 - x) y' with f's monomial coefficients
    (a different code path from the C oracle's matrix iteration);
  - the fp32 goldens (oracle on fl32(A)) differ from the fp64 ones only by the input rounding;
  - config 5's golden is pinned at test time on the GPU box by an LU solve
    (tests/test_gpu_golden.py::test_config5_golden).
"""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from make_goldens import GOLDENS, golden_path, load_golden  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle.kernels import kernel_coeffs  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

LD = np.longdouble


def _have(name):
    if not os.path.exists(golden_path(name)):
        pytest.fail(f"golden {name} missing (tools/make_goldens.py {name})")


@pytest.mark.parametrize("name", sorted(GOLDENS))
def test_golden_metadata(name):
    _have(name)
    sv, meta = load_golden(name)
    cfg, kw, pseed, steps, dt, oracle = GOLDENS[name]
    assert (meta["config"], meta["steps"], meta["dtype"], meta["oracle"]) == (cfg, steps, dt, oracle)
    assert meta["A_env"] == inputs.REPRO_ENV
    V, idx = inputs.probe_block(meta["d"], pseed)
    assert V.shape[1] == 16 and meta["probe_cols"] == 16          # 8 unit + 8 Gaussian
    assert inputs.sha256(V) == meta["V_sha256"]
    assert sv.shape == (meta["d"], 16) and np.all(np.isfinite(sv.astype(np.float64)))
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "MANIFEST.json")))
    assert man[name]["A_sha256"] == meta["A_sha256"]


def _scalar_plan(x, steps):
    """Y_n(x) of a radix plan as a scalar recursion in long double."""
    y = np.ones_like(x)
    r = x.copy()
    for m in steps:
        c = [O._frac_to_ld(v) for v in kernel_coeffs(m, "polished")]
        f = np.zeros_like(x)
        for cj in reversed(c):                          # Horner in r
            f = f * r + cj
        y = y * f
        r = 1 - (1 - x) * y
    return y


@pytest.fixture(scope="module")
def cfg3_factors():
    A, Q, ev = inputs.cpu_reproducible("cfg3", full=True)
    return A, Q, ev


@pytest.mark.parametrize("name", ["cfg3_x15x3_f64", "cfg3_x9x4_f64", "cfg3_x2x12_f64"])
def test_cfg3_golden_closed_form(cfg3_factors, name):
    _have(name)
    A, Q, ev = cfg3_factors
    sv, meta = load_golden(name)
    assert inputs.sha256(A) == meta["A_sha256"]
    V, _ = inputs.probe_block(meta["d"], meta["probe_seed"])
    x = ev.astype(LD)
    if meta["oracle"] == "C-2":
        s = _scalar_plan(x, meta["steps"])
    else:
        s = (1 - x ** meta["k"]) / (1 - x)              # geometric series per eigenvalue
    QtV = Q.T @ V
    ref = Q @ (np.asarray(s, dtype=np.float64)[:, None] * QtV)
    err = O.rel_fro(np.asarray(sv, dtype=np.float64), ref)
    # measured 3.4e-14 (Q is orthogonal to rounding, A = Q diag Q^T symmetrised in binary64);
    # a wrong term, sign or index would show as O(1e-3) or more
    print(f"{name}: golden vs closed form {err:.2e}")
    assert err <= 1e-12, (name, err)


@pytest.mark.parametrize("plan", ["x15x3", "x9x4", "x2x12"])
def test_cfg3_f32_golden_near_f64(plan):
    _have(f"cfg3_{plan}_f32")
    _have(f"cfg3_{plan}_f64")
    s32, m32 = load_golden(f"cfg3_{plan}_f32")
    s64, m64 = load_golden(f"cfg3_{plan}_f64")
    assert m32["A_sha256"] == m64["A_sha256"]             # same A, fl32 applied by the script
    e = O.rel_fro(s32, s64)
    # input rounding alone moves S_k by ~2e-7 at config 3; the two must differ
    print(f"{plan}: fp32 golden vs fp64 golden {e:.2e}")
    assert 1e-9 < e <= 2e-6, e
