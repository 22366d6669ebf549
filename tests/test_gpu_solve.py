"""GPU tests of the adaptive approximate-inverse driver nseries_solve:
residual radix-kernel iteration with the fused residual-norm epilogue and adaptive stopping.
Reproduces the product counts of App. A.3 (Table 7)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2602_11843_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

LD = np.longdouble


@pytest.fixture(scope="module")
def h():
    from paper_2602_11843_b200 import build as B
    B.build()
    handle = P.nseries_create(0)
    yield handle
    P.nseries_destroy(handle)


def _a3_matrix(d=64, seed=0):
    """App. A.3 workload, reading Z14: SPD, eigenvalues of I - A geometric in [1e-4, 1]
    (kappa(I - A) = 1e4); A = Q diag(1 - mu) Q^T."""
    rng = np.random.default_rng(seed)
    Q, R = np.linalg.qr(rng.standard_normal((d, d)))
    Q = Q * np.sign(np.diag(R))[None, :]
    mu = np.geomspace(1e-4, 1.0, d)
    A = (Q * (1.0 - mu)[None, :]) @ Q.T
    return np.ascontiguousarray(0.5 * (A + A.T))


def _normalized_residual(A, Y):
    d = A.shape[0]
    R = np.eye(d, dtype=LD) - Y.astype(LD) + O.matvec(A, Y)
    return float(np.sqrt(np.sum(R * R)) / np.sqrt(d))


# App. A.3 Table 7: products to reach 1e-13.  The radix-9 row prints 32
# while the cost model (5 per step, 9^6 = 531441 > 2.8e5 needed) gives 30.
@pytest.mark.parametrize("m,products", [(2, 38), (3, 36), (5, 32), (9, 30), (15, 30)])
def test_table7_products(h, m, products):
    A = _a3_matrix()
    d = A.shape[0]
    At = torch.from_numpy(A).cuda()
    Y = torch.empty_like(At)
    R = torch.empty_like(At)
    flags = P.NSERIES_RFORM_TELESCOPE if m == 15 else 0
    info = P.nseries_solve(h, At, d, m, 1e-13, 40, Y=Y, R_out=R, flags=flags)
    torch.cuda.synchronize()
    assert info["converged"], info
    assert info["products"] == products, info
    # residual history is monotone decreasing for this SPD matrix (Stability)
    hist = info["history"]
    assert all(b <= a * 1.0001 for a, b in zip(hist, hist[1:]))
    Yh = Y.cpu().numpy()
    # the fused device norm tracks the iterated residual R_n; the residual of the ROUNDED Y,
    # I - (I - A) Y, has an fp64 evaluation floor ~ eps ||Y|| ~ 1e-12 here (kappa = 1e4; the
    # paper's Table 3 shows the same floor, ~1e-13 at d=500)
    host = _normalized_residual(A, Yh)
    assert info["residual"] <= 1e-13
    assert host <= 2e-12
    # Y ~ (I - A)^{-1} (kappa = 1e4)
    inv = np.linalg.inv(np.eye(d) - A)
    assert np.linalg.norm(Yh - inv) / np.linalg.norm(inv) <= 1e-9


@pytest.mark.parametrize("m,steps", [(9, 2), (5, 3), (2, 6), (15, 2), (3, 4)])
def test_solve_fixed_steps_vs_oracle(h, m, steps):
    # tol = 0 runs exactly max_steps steps: Y is the plan polynomial of [m] * steps (oracle)
    d = 40
    A = inputs.random_matrix(d, 11, 0.7)
    At = torch.from_numpy(A).cuda()
    Y = torch.empty_like(At)
    info = P.nseries_solve(h, At, d, m, 0.0, steps, Y=Y)
    torch.cuda.synchronize()
    assert info["steps"] == steps and not info["converged"]
    assert info["products"] == (P.nseries_kernel_info(m)["mu"] + 2) * steps
    ref = O.plan_apply(A, [m] * steps, np.eye(d))
    assert O.rel_fro(Y.cpu().numpy(), ref) <= 1e-11


def test_solve_early_stop_copies_out(h):
    # stopping before the planned last step copies the workspace iterate into Y
    d = 32
    A = inputs.random_matrix(d, 3, 0.3)
    At = torch.from_numpy(A).cuda()
    Y = torch.full_like(At, float("nan"))
    R = torch.full_like(At, float("nan"))
    info = P.nseries_solve(h, At, d, 9, 1e-14, 10, Y=Y, R_out=R)
    torch.cuda.synchronize()
    assert info["converged"] and info["steps"] < 10
    Yh, Rh = Y.cpu().numpy(), R.cpu().numpy()
    assert np.all(np.isfinite(Yh)) and np.all(np.isfinite(Rh))
    res = np.eye(d, dtype=LD) - Yh.astype(LD) + O.matvec(A, Yh)
    assert float(np.max(np.abs(res - Rh))) <= 1e-14
