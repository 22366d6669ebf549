"""GPU parity at BASELINE.json's full sizes -- configs 3 (d = 4096, fp64 and fp32) and 5
(d = 8192, AUTO k = 10000) -- on the 16-column probe block of SURVEY.md 8(c) C-3, against
oracle goldens committed under tests/golden/ (written by tools/make_goldens.py, which calls only
oracle/).

A is rebuilt on the host exactly as the golden script built it (inputs.cpu_reproducible: numpy
with OpenBLAS pinned to one thread and its Haswell kernels) and its SHA-256 must equal the one
stored in the golden; the GPU evaluates that same A, S_gpu V is formed in long double on the
host (oracle matvec) and compared column-block-wise with the golden: relative Frobenius
<= 1e-11 (fp64) / 2e-5 (fp32, oracle on fl32(A)) -- BASELINE.json north_star.
"""
import os
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")

import paper_2602_11843_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import plan as OP  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from make_goldens import GOLDENS, golden_path, load_golden  # noqa: E402

TOL = {"f64": 1e-11, "f32": 2e-5}
LD = np.longdouble


@pytest.fixture(scope="module")
def h():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    handle = P.nseries_create(0)
    yield handle
    P.nseries_destroy(handle)


_A_CACHE = {}


def _A_for(name):
    cfg, kw, _, _, _, _ = GOLDENS[name]
    key = (cfg, tuple(sorted(kw.items())))
    if key not in _A_CACHE:
        _A_CACHE.clear()                      # hold one config's A at a time (cfg5: 512 MiB)
        _A_CACHE[key] = inputs.cpu_reproducible(cfg, **kw)
    return _A_CACHE[key]


def _check(h, name, flags=0):
    if not os.path.exists(golden_path(name)):
        pytest.fail(f"golden {name} missing: run tools/make_goldens.py {name}")
    sv_ref, meta = load_golden(name)
    A = _A_for(name)
    assert inputs.sha256(A) == meta["A_sha256"], "host rebuilt a different A than the golden's"
    d, steps, k, dt = meta["d"], meta["steps"], meta["k"], meta["dtype"]
    V, _ = inputs.probe_block(d, meta["probe_seed"])
    assert V.shape[1] == 16 and inputs.sha256(V) == meta["V_sha256"]
    approx = 15 in steps
    flags |= P.NSERIES_ALLOW_APPROX if approx else 0
    plan = P.nseries_plan_finalize(steps, k, flags)
    tdt = torch.float64 if dt == "f64" else torch.float32
    At = torch.from_numpy(A).to("cuda", tdt)
    S = torch.full_like(At, float("nan"))
    R = torch.full_like(At, float("nan")) if dt == "f64" else None
    P.nseries_eval(h, At, d, k, plan=plan, S=S, R_out=R, flags=flags)
    torch.cuda.synchronize()
    st = P.nseries_last_stats(h)
    assert st["products"] == OP.plan_products(steps), st
    S_h = S.cpu().numpy().astype(np.float64)
    got = O.matvec(S_h, V)
    err = O.rel_fro(got, sv_ref)
    print(f"{name} flags={flags:#x}: rel_fro on 16 probes = {err:.3e} (tol {TOL[dt]:.0e})")
    assert err <= TOL[dt], (name, err)
    if R is not None:
        # property at full size: (I - A) S = I - R (telescoping / Lemma 5), on the probes
        SV = O.matvec(S_h, V)
        lhs = SV - O.matvec(A, np.asarray(SV, dtype=np.float64))
        rhs = V.astype(LD) - O.matvec(R.cpu().numpy(), V)
        assert O.rel_fro(lhs, rhs) <= 1e-10
    return err


@pytest.mark.parametrize("name", ["cfg3_x15x3_f64", "cfg3_x9x4_f64", "cfg3_x2x12_f64"])
def test_config3_f64_golden(h, name):
    _check(h, name)


def test_config3_f64_golden_symmetric(h):
    # config 3's A is symmetric by construction (bit-exact after symmetrisation)
    A = _A_for("cfg3_x15x3_f64")
    assert np.array_equal(A, A.T)
    _check(h, "cfg3_x15x3_f64", flags=P.NSERIES_SYMMETRIC)


@pytest.mark.parametrize("name", ["cfg3_x15x3_f32", "cfg3_x9x4_f32", "cfg3_x2x12_f32"])
def test_config3_f32_golden(h, name):
    _check(h, name)


def test_config3_f32_golden_symmetric(h):
    _check(h, "cfg3_x15x3_f32", flags=P.NSERIES_SYMMETRIC)


def test_config5_golden(h):
    # BASELINE.json configs[4]: the plan builder's AUTO plan over {15, 9, 5, 2} for k = 10000
    plan = P.nseries_plan_build(10000, radices=[15, 9, 5, 2], flags=P.NSERIES_ALLOW_APPROX)
    assert plan.steps == GOLDENS["cfg5_auto_f64"][3]
    _check(h, "cfg5_auto_f64")
    # independent pin of the golden itself: ||A^k|| <= 0.99^10000 ~ 2e-44, so S_k(A) V equals
    # (I - A)^{-1} V to far below 1e-11 -- one LU solve in float64 (numpy/LAPACK)
    sv_ref, meta = load_golden("cfg5_auto_f64")
    A = _A_for("cfg5_auto_f64")
    V, _ = inputs.probe_block(meta["d"], meta["probe_seed"])
    X = np.linalg.solve(np.eye(meta["d"]) - A, V)
    err = O.rel_fro(X, sv_ref)
    print(f"cfg5 golden vs LU solve of (I - A) X = V: {err:.2e}")
    assert err <= 1e-11
