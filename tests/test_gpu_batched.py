"""GPU parity of the batched small-matrix path (one launch per batch) vs the oracle.

fp32 runs compare against the oracle evaluated on fl32(A) (the exact bits the GPU sees) with
the fp32 tolerance 2e-5 relative Frobenius per matrix (BASELINE.json north_star); fp64 runs
use 1e-11.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2602_11843_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import plan as OP  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

TOL32, TOL64 = 2e-5, 1e-11


@pytest.fixture(scope="module")
def h():
    from paper_2602_11843_b200 import build as B
    B.build()
    handle = P.nseries_create(0)
    yield handle
    P.nseries_destroy(handle)


def _oracle(A, steps):
    d = A.shape[0]
    if 15 in steps:
        return O.plan_apply(A, steps, np.eye(d))
    return O.full_series(A, OP.plan_reaches(steps))


def _batch(h, Ab, steps, dtype, flags=0):
    batch, d, _ = Ab.shape
    k = OP.plan_reaches(steps)
    flags |= P.NSERIES_ALLOW_APPROX if 15 in steps else 0
    plan = P.nseries_plan_finalize(steps, k, flags)
    At = torch.from_numpy(np.ascontiguousarray(Ab)).to("cuda", dtype)
    S = torch.full_like(At, float("nan"))
    P.nseries_eval_batched_strided(h, At, d * d, batch, d, k, plan=plan, S=S, flags=flags)
    torch.cuda.synchronize()
    st = P.nseries_last_stats(h)
    assert st["launches"] == (1 if batch else 0)
    assert st["products"] == OP.plan_products(steps, bool(flags & P.NSERIES_ELIDE_TRIVIAL))
    return S.cpu().numpy()


PLANS = [[9, 9], [5, 5], [2] * 5, [15], [15, 1, 5], [1, 9], [1], [2], [15, 15]]


@pytest.mark.parametrize("d", [1, 5, 16, 31, 32, 33, 48, 64])
@pytest.mark.parametrize("steps", PLANS)
def test_batched_f32(h, d, steps):
    rng = np.random.default_rng(d)
    batch = 7
    Ab = (0.6 * rng.standard_normal((batch, d, d)) / np.sqrt(d)).astype(np.float32)
    S = _batch(h, Ab, steps, torch.float32)
    for b in range(batch):
        ref = _oracle(Ab[b].astype(np.float64), steps)
        assert O.rel_fro(S[b], ref) <= TOL32, (d, steps, b)


@pytest.mark.parametrize("wpm", ["1", "2", "4"])
@pytest.mark.parametrize("d", [17, 32])
@pytest.mark.parametrize("steps", [[9, 9], [15, 15], [1, 2, 2], [5, 1, 9]])
def test_batched_f32_warps_per_matrix(h, wpm, d, steps, monkeypatch):
    # the warp-group kernel's tuning knob NSERIES_BATCHED_WPM (1, 2 = default, 4 warps per
    # matrix): each variant tiles the fragments and finds the diagonal tiles differently
    monkeypatch.setenv("NSERIES_BATCHED_WPM", wpm)
    rng = np.random.default_rng(100 + d)
    batch = 300                                  # > 148 x groups: every warp group takes several
    Ab = (0.6 * rng.standard_normal((batch, d, d)) / np.sqrt(d)).astype(np.float32)
    S = _batch(h, Ab, steps, torch.float32)
    for b in (0, 1, 148, 149, batch - 1):
        ref = _oracle(Ab[b].astype(np.float64), steps)
        assert O.rel_fro(S[b], ref) <= TOL32, (wpm, d, steps, b)


@pytest.mark.parametrize("d", [1, 4, 16, 17, 32])
@pytest.mark.parametrize("steps", [[9, 9], [5, 5, 5], [15, 15], [1, 2, 2]])
def test_batched_f64(h, d, steps):
    rng = np.random.default_rng(100 + d)
    batch = 5
    Ab = 0.6 * rng.standard_normal((batch, d, d)) / np.sqrt(d)
    S = _batch(h, Ab, steps, torch.float64)
    for b in range(batch):
        assert O.rel_fro(S[b], _oracle(Ab[b], steps)) <= TOL64, (d, steps, b)


def test_batched_elided_and_pointer_api(h):
    d, batch = 32, 9
    rng = np.random.default_rng(1)
    Ab = (0.5 * rng.standard_normal((batch, d, d)) / np.sqrt(d)).astype(np.float32)
    S = _batch(h, Ab, [9, 9], torch.float32, flags=P.NSERIES_ELIDE_TRIVIAL)
    for b in range(batch):
        assert O.rel_fro(S[b], _oracle(Ab[b].astype(np.float64), [9, 9])) <= TOL32
    At = torch.from_numpy(Ab).cuda()
    St = torch.zeros_like(At)
    Ap = torch.tensor([At[b].data_ptr() for b in range(batch)], dtype=torch.int64, device="cuda")
    Sp = torch.tensor([St[b].data_ptr() for b in range(batch)], dtype=torch.int64, device="cuda")
    plan = P.nseries_plan_finalize([9, 9], 81, 0)
    P.nseries_eval_batched(h, Ap, batch, d, 81, plan=plan, dtype=P.NSERIES_F32, S_ptrs=Sp)
    torch.cuda.synchronize()
    for b in range(batch):
        assert O.rel_fro(St[b].cpu().numpy(), _oracle(Ab[b].astype(np.float64), [9, 9])) <= TOL32


def test_batched_empty_and_too_big(h):
    A = torch.zeros(0, 32, 32, device="cuda")
    plan = P.nseries_plan_finalize([9, 9], 81, 0)
    P.nseries_eval_batched_strided(h, A, 1024, 0, 32, 81, plan=plan, dtype=P.NSERIES_F32, S=A)
    B = torch.zeros(2, 65, 65, device="cuda")
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_eval_batched_strided(h, B, 65 * 65, 2, 65, 81, plan=plan, dtype=P.NSERIES_F32, S=B.clone())
    assert e.value.status == 9


@pytest.mark.parametrize("steps", [[9, 9], [5, 5]])
@pytest.mark.parametrize("rows", [128, 256])
def test_config4(h, steps, rows):
    # BASELINE.json configs[3]: 16384 MIMO matrices 32x32 fp32 (rows=256: convergent variant, R12).
    # SURVEY 8(d) T6 asks for the full oracle on a 1024-matrix sample; the batched C-1 oracle is
    # fast enough to take EVERY matrix in full (V = I, fl32(A_b), relative Frobenius <= 2e-5)
    Ab = inputs.cfg4(rows=rows)
    S = _batch(h, Ab, steps, torch.float32)
    assert np.all(np.isfinite(S))
    k = OP.plan_reaches(steps)
    n, d = Ab.shape[0], Ab.shape[1]
    worst, worst_b = 0.0, -1
    for b0 in range(0, n, 2048):
        blk = slice(b0, min(n, b0 + 2048))
        ref = O.series_sum_batch(Ab[blk], k, np.broadcast_to(np.eye(d), (blk.stop - b0, d, d)))
        got = S[blk].astype(np.float64).astype(np.longdouble)
        e = np.sqrt(np.sum((got - ref) ** 2, axis=(1, 2))) / np.sqrt(np.sum(ref ** 2, axis=(1, 2)))
        if float(e.max()) > worst:
            worst, worst_b = float(e.max()), b0 + int(e.argmax())
    print(f"config 4 {steps} rows={rows}: worst relative Frobenius over {n} matrices {worst:.3e} (matrix {worst_b})")
    assert worst <= TOL32, (worst, worst_b)


@pytest.mark.parametrize("d,pad", [(32, 0), (32, 1), (31, 3), (8, 0)])
def test_batched_many_per_warp_strided(h, d, pad):
    # batch >> resident warps: each warp walks many matrices (prefetch double buffer); pad > 0
    # gives strides that break 16-byte alignment (scalar load/store paths)
    batch = 6000
    rng = np.random.default_rng(7 + d + pad)
    Ab = (0.5 * rng.standard_normal((batch, d, d)) / np.sqrt(d)).astype(np.float32)
    stride = d * d + pad
    flat = np.zeros((batch, stride), np.float32)
    flat[:, : d * d] = Ab.reshape(batch, -1)
    At = torch.from_numpy(flat).cuda()
    St = torch.full((batch, stride), float("nan"), device="cuda")
    plan = P.nseries_plan_finalize([9, 9], 81, 0)
    P.nseries_eval_batched_strided(h, At, stride, batch, d, 81, plan=plan, dtype=P.NSERIES_F32, S=St,
                                   strideS=stride)
    torch.cuda.synchronize()
    S = St.cpu().numpy()
    assert np.all(np.isnan(S[:, d * d:]))            # padding between matrices untouched
    S = S[:, : d * d].reshape(batch, d, d)
    for b in list(range(0, batch, 397)) + [batch - 1]:
        assert O.rel_fro(S[b], _oracle(Ab[b].astype(np.float64), [9, 9])) <= TOL32, b


@pytest.mark.parametrize("d,dtype", [(32, torch.float32), (17, torch.float32), (48, torch.float32), (32, torch.float64)])
@pytest.mark.parametrize("steps", [[7, 7], [11, 9], [13], [1, 4, 4]])
def test_batched_naive_radix(h, d, dtype, steps):
    # naive radix-m splitting through the one-launch batched kernels
    rng = np.random.default_rng(40 + d)
    batch = 5
    Ab = 0.6 * rng.standard_normal((batch, d, d)) / np.sqrt(d)
    if dtype == torch.float32:
        Ab = Ab.astype(np.float32)
    S = _batch(h, Ab, steps, dtype)
    tol = TOL32 if dtype == torch.float32 else TOL64
    for b in range(batch):
        assert O.rel_fro(S[b], _oracle(Ab[b].astype(np.float64), steps)) <= tol, (d, steps, b)
