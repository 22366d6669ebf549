"""GPU parity: the CUDA path (through the C ABI) against the long-double oracle.

Tolerances (BASELINE.json north_star): relative Frobenius <= 1e-11 for fp64 (column-wise on
probe blocks for large d).  Exact plans are compared with C-1 (the definition S_k = sum A^j);
approximate (radix-15) plans with C-2 (the plan's own polynomial, reading R7).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2602_11843_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import plan as OP  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402

TOL64 = 1e-11
LD = np.longdouble


@pytest.fixture(scope="module")
def h():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2602_11843_b200 import build as B
    B.build()
    handle = P.nseries_create(0)
    yield handle
    P.nseries_destroy(handle)


def _flags(steps, extra=0):
    return extra | (P.NSERIES_ALLOW_APPROX if 15 in steps else 0)


def _oracle_full(A, steps, want_R=False):
    d = A.shape[0]
    k = OP.plan_reaches(steps)
    if 15 in steps:
        return O.plan_apply(A, steps, np.eye(d), want_R=want_R)
    S = O.full_series(A, k)
    if not want_R:
        return S
    R = np.eye(d, dtype=LD)
    for _ in range(k):
        R = O.matvec(A, R)
    return S, R


def _run(h, A, steps, flags=0, want_R=False, dtype=torch.float64):
    d = A.shape[0]
    k = OP.plan_reaches(steps)
    flags = _flags(steps, flags)
    plan = P.nseries_plan_finalize(steps, k, flags)
    At = torch.from_numpy(np.ascontiguousarray(A)).to("cuda", dtype)
    S = torch.full_like(At, float("nan"))
    R = torch.full_like(At, float("nan")) if want_R else None
    P.nseries_eval(h, At, d, k, plan=plan, S=S, R_out=R, flags=flags)
    torch.cuda.synchronize()
    st = P.nseries_last_stats(h)
    elide = bool(flags & P.NSERIES_ELIDE_TRIVIAL)
    extra = 1 if (elide and want_R and steps[-1] != 1) else 0   # R_out needs the final power
    assert st["products"] == OP.plan_products(steps, elide) + extra, (steps, st)
    return S.cpu().numpy(), (R.cpu().numpy() if want_R else None), st


PLANS = [[9, 9], [5, 5, 5], [2] * 6, [1, 2, 2], [15], [15, 15], [15, 1, 5], [9, 1, 2], [1], [2],
         [5, 1, 9], [1, 1, 1], [3, 3, 3], [3, 1, 9]]


@pytest.mark.parametrize("d", [1, 2, 3, 7, 8, 16, 31, 33, 64, 100, 130])
@pytest.mark.parametrize("steps", PLANS)
def test_parity_small_full(h, d, steps):
    A = inputs.random_matrix(d, 100 + d, 0.7)
    S, _, _ = _run(h, A, steps)
    ref = _oracle_full(A, steps)
    assert O.rel_fro(S, ref) <= TOL64, (d, steps)


@pytest.mark.parametrize("steps", [[9, 9], [5, 5, 5], [2] * 6, [15, 15], [15, 1, 5], [9, 1, 2], [2], [9], [1]])
@pytest.mark.parametrize("extra", [P.NSERIES_ELIDE_TRIVIAL, P.NSERIES_RFORM_TELESCOPE])
def test_parity_flags(h, steps, extra):
    d = 96
    A = inputs.random_matrix(d, 7, 0.7)
    S, _, _ = _run(h, A, steps, flags=extra)
    ref = _oracle_full(A, steps)
    assert O.rel_fro(S, ref) <= TOL64


@pytest.mark.parametrize("steps", [[9, 9], [5, 5], [2] * 5, [15, 15], [15, 1, 5], [1, 2], [1]])
def test_residual_output(h, steps):
    # R_out = A^k for exact plans (telescoping), R_n = I - (I-A) Y_n for radix-15
    d = 80
    A = inputs.random_matrix(d, 3, 0.8)
    S, R, _ = _run(h, A, steps, want_R=True)
    Sref, Rref = _oracle_full(A, steps, want_R=True)
    scale = float(np.sqrt(np.sum(np.asarray(Sref, dtype=LD) ** 2)))
    assert O.rel_fro(S, Sref) <= TOL64
    assert float(np.sqrt(np.sum((R.astype(LD) - Rref) ** 2))) / scale <= 1e-13
    # the paper's metric: I - (I-A)S = R (F7) at this d
    lhs = np.eye(d, dtype=LD) - S.astype(LD) + O.matvec(A, S)
    assert float(np.sqrt(np.sum((lhs - R.astype(LD)) ** 2))) / scale <= 1e-13


def test_auto_plan_k10000(h):
    d = 48
    A = inputs.random_matrix(d, 5, 0.6)
    flags = P.NSERIES_ALLOW_APPROX
    plan = P.nseries_plan_build(10000, radices=[15, 9, 5, 2], flags=flags)
    assert plan.steps == [15, 1, 5, 5, 5, 5] and plan.products == 23
    At = torch.from_numpy(A).cuda()
    S = torch.empty_like(At)
    P.nseries_eval(h, At, d, 10000, plan=plan, S=S, flags=flags)
    torch.cuda.synchronize()
    ref = O.plan_apply(A, plan.steps, np.eye(d))
    assert O.rel_fro(S.cpu().numpy(), ref) <= TOL64
    assert P.nseries_last_stats(h)["products"] == 23


def test_eval_default_plan_and_host_api(h):
    d, k = 50, 90
    A = inputs.random_matrix(d, 12, 0.7)
    At = torch.from_numpy(A).cuda()
    S = torch.empty_like(At)
    P.nseries_eval(h, At, d, k, S=S)            # plan=NULL -> AUTO over {9,5,2}
    torch.cuda.synchronize()
    ref = O.full_series(A, k)
    assert O.rel_fro(S.cpu().numpy(), ref) <= TOL64
    Sh = np.empty_like(A)
    P.nseries_eval_host(h, np.ascontiguousarray(A), d, k, S=Sh)
    assert O.rel_fro(Sh, ref) <= TOL64


def test_errors(h):
    A = torch.zeros(8, 8, dtype=torch.float64, device="cuda")
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_eval(h, A, 8, 10, S=A)
    assert e.value.status == 5
    plan = P.nseries_plan_build(81, kind=9)
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_eval(h, A, 8, 82, plan=plan, S=torch.empty_like(A))
    assert e.value.status == 3


# 990 / 1000 / 1024 / 1040: the one-wave 96x80 tiles (even d in 989..1040), ragged edges at 990 and 1000
@pytest.mark.parametrize("d", [1, 5, 64, 127, 300, 990, 1000, 1024, 1040, 1536, 2048])
def test_matmul_engine(h, d):
    rng = np.random.default_rng(d)
    X = rng.standard_normal((d, d))
    Y = rng.standard_normal((d, d))
    Xt, Yt = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    C = torch.empty_like(Xt)
    P.nseries_matmul(h, Xt, Yt, C, d)
    torch.cuda.synchronize()
    cols = np.arange(d) if d <= 300 else rng.choice(d, 16, replace=False)
    ref = O.matvec(X, Y[:, cols])
    err = O.rel_fro(C.cpu().numpy()[:, cols], ref)
    assert err <= 1e-15 * max(1.0, np.sqrt(d)), err


# ---------------------------------------------------------------- BASELINE.json configs


def _probe_parity(S_gpu, A, steps, V, approx_oracle):
    """S_gpu V vs oracle (C-1 or C-2) on the probe block V."""
    k = OP.plan_reaches(steps)
    if approx_oracle:
        ref = O.plan_apply(A, steps, V)
    else:
        ref, _ = O.series_sum(A, k, V)
    got = O.matvec(S_gpu, V)
    return O.rel_fro(got, ref)


def test_config1_full(h):
    A = inputs.cfg1()
    for steps in ([9, 9], [2] * 6, [5, 5, 5]):
        S, R, _ = _run(h, A, steps, want_R=True)
        assert O.rel_fro(S, _oracle_full(A, steps)) <= TOL64


@pytest.mark.slow
@pytest.mark.parametrize("steps", [[9, 9, 9], [5] * 4, [2] * 9, [2] * 10])
def test_config2_probes(h, steps):
    A = inputs.cfg2()
    V, _ = inputs.probe_block(A.shape[0], 1)
    S, _, _ = _run(h, A, steps)
    assert _probe_parity(S, A, steps, V, False) <= TOL64


@pytest.mark.parametrize("steps", [[15, 15], [9, 9], [5, 1, 2]])
def test_single_wave_tiles_d1000(h, steps):
    # d = 1000 runs the 96x80 one-wave tiles (11 x 13 = 143 CTAs, ragged last row and column of
    # tiles) through every epilogue form of these plans, S and R_out, on 16 probe columns
    d = 1000
    A = inputs.random_matrix(d, 41, 0.9)
    V, _ = inputs.probe_block(d, 1)
    S, R, _ = _run(h, A, steps, want_R=True)
    approx = 15 in steps
    assert _probe_parity(S, A, steps, V, approx) <= TOL64
    # R_out = I - (I - A) S (PAPER.md residual identity), checked on the probes against the oracle's S V
    k = OP.plan_reaches(steps)
    SV = O.plan_apply(A, steps, V) if approx else O.series_sum(A, k, V)[0]
    ref_R = V.astype(LD) - (SV - O.matvec(A, SV))
    scale = float(np.sqrt(np.sum(np.asarray(SV, dtype=LD) ** 2)))
    assert float(np.sqrt(np.sum((O.matvec(R, V) - ref_R) ** 2))) / scale <= 1e-12


# configs 3 and 5 (d = 4096 / 8192, 16 probe columns against committed oracle goldens):
# tests/test_gpu_golden.py


# ---------------------------------------------------------------- fp32 (3xTF32 on tcgen05)

TOL32 = 2e-5


@pytest.mark.parametrize("d", [1, 2, 7, 16, 31, 33, 64, 100, 130, 257])
@pytest.mark.parametrize("steps", [[9, 9], [5, 5, 5], [2] * 6, [15, 15], [15, 1, 5], [9, 1, 2], [1], [2]])
def test_parity_small_f32(h, d, steps):
    A = inputs.random_matrix(d, 300 + d, 0.7).astype(np.float32)
    S, _, _ = _run(h, A.astype(np.float64), steps, dtype=torch.float32)
    ref = _oracle_full(A.astype(np.float64), steps)     # oracle on fl32(A), the GPU's exact input
    assert O.rel_fro(S, ref) <= TOL32, (d, steps)


@pytest.mark.parametrize("d", [1, 16, 33, 64, 72])
@pytest.mark.parametrize("steps", [[9, 9], [15, 15], [2] * 5, [1, 2], [15, 1, 5]])
@pytest.mark.parametrize("extra", [0, P.NSERIES_ELIDE_TRIVIAL, P.NSERIES_RFORM_TELESCOPE])
def test_parity_f32_flags_and_R(h, d, steps, extra):
    # d <= 64 with R_out: the single-launch batched kernels have no R output, so these run on
    # the tiled tcgen05 engine (api.cu); d = 72 is tiled either way
    A = inputs.random_matrix(d, 9, 0.8).astype(np.float32)
    S, R, _ = _run(h, A.astype(np.float64), steps, flags=extra, want_R=True, dtype=torch.float32)
    Sref, Rref = _oracle_full(A.astype(np.float64), steps, want_R=True)
    assert O.rel_fro(S, Sref) <= TOL32
    if not (extra & P.NSERIES_ELIDE_TRIVIAL):
        scale = float(np.sqrt(np.sum(np.asarray(Sref, dtype=LD) ** 2)))
        assert float(np.sqrt(np.sum((R.astype(LD) - Rref) ** 2))) / scale <= 1e-5


@pytest.mark.parametrize("d", [5, 128, 300, 1024, 1100, 2048, 4096, 4100])
def test_matmul_engine_f32(h, d):
    # 4100: odd number of 128-row tiles (the second CTA of the last M-pair cluster lies past d)
    # and a ragged last column tile.  Split-K of the last partial wave (74 resident clusters):
    # 1024 -> 16 pair tiles in 2 K ranges, 1100 -> 25 tiles in 2 uneven K ranges (69 k-blocks),
    # 4096 -> the last 34 of 256 tiles in 2 K ranges
    # one 3xTF32 product vs the exact product of the fp32 inputs (<= 5e-7 budget)
    rng = np.random.default_rng(d + 7)
    X = rng.standard_normal((d, d)).astype(np.float32)
    Y = rng.standard_normal((d, d)).astype(np.float32)
    Xt, Yt = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    C = torch.empty_like(Xt)
    P.nseries_matmul(h, Xt, Yt, C, d)
    torch.cuda.synchronize()
    cols = np.arange(d) if d <= 300 else rng.choice(d, 16, replace=False)
    ref = O.matvec(X.astype(np.float64), Y[:, cols].astype(np.float64))
    assert O.rel_fro(C.cpu().numpy()[:, cols], ref) <= 5e-7


@pytest.mark.parametrize("d", [1024, 1100, 2100, 1024])
def test_splitk_f32_deterministic(h, d):
    # (the sizes alternate so the split-K counters left by one size are reused by another)
    # split-K tiles sum their K-range partials in K order whichever CTA finishes last, so two
    # evaluations are bit-identical; and they match the oracle on probe columns
    A = inputs.random_matrix(d, 77, 0.9).astype(np.float32)
    S1, _, _ = _run(h, A.astype(np.float64), [9, 9], dtype=torch.float32)
    S2, _, _ = _run(h, A.astype(np.float64), [9, 9], dtype=torch.float32)
    assert np.array_equal(S1, S2)
    V, _ = inputs.probe_block(d, 5, n_unit=2, n_gauss=2)
    assert _probe_parity(S1.astype(np.float64), A.astype(np.float64), [9, 9], V, False) <= TOL32


def _handle_with_small_mode(mode):
    import os
    os.environ["NSERIES_SMALL_MODE"] = str(mode)
    try:
        return P.nseries_create(0)
    finally:
        del os.environ["NSERIES_SMALL_MODE"]


@pytest.fixture(scope="module")
def h_small_modes():
    """Handles for the two d <= 64 fp64 paths: 0 = one launch of the 4 x 2 cluster kernel
    (default), 1 = the tiled engine, one launch per op (NSERIES_SMALL_MODE=1)."""
    hs = {m: _handle_with_small_mode(m) for m in (0, 1)}
    yield hs
    for x in hs.values():
        P.nseries_destroy(x)


@pytest.mark.parametrize("d", [1, 5, 17, 33, 64])
@pytest.mark.parametrize("steps,extra", [([9, 9], 0), ([9, 9], 1), ([15, 15], 0), ([15, 1, 5], 2),
                                         ([5, 5, 5], 1), ([1, 2, 2], 0), ([1], 0), ([2], 1), ([3, 1, 9], 2)])
@pytest.mark.parametrize("which", [0, 1])
def test_small_kernels_flags_and_R(h_small_modes, d, steps, extra, which):
    # the single-launch 4 x 2 cluster kernel and the tiled engine at d <= 64, with the elide /
    # telescoping flags and the residual output R_out
    flags = [0, P.NSERIES_ELIDE_TRIVIAL, P.NSERIES_RFORM_TELESCOPE][extra]
    handle = h_small_modes[which]
    A = inputs.random_matrix(d, 11 + d, 0.7)
    S, R, st = _run(handle, A, steps, flags=flags, want_R=True)
    if which == 0:
        assert st["launches"] == 1
    Sref, Rref = _oracle_full(A, steps, want_R=True)
    assert O.rel_fro(S, Sref) <= TOL64, (d, steps, flags, which)
    scale = float(np.sqrt(np.sum(np.asarray(Sref, dtype=LD) ** 2)))
    assert float(np.sqrt(np.sum((R.astype(LD) - Rref) ** 2))) / scale <= 1e-13



@pytest.mark.parametrize("d", [65, 130, 300, 513, 1024])
@pytest.mark.parametrize("steps,extra", [([9, 9], 0), ([15, 15], 0), ([15, 1, 5], 2), ([2] * 5, 1),
                                         ([5, 5], 0), ([3, 1, 9], 0)])
def test_symmetric_mode(h, d, steps, extra):
    # NSERIES_SYMMETRIC: upper-triangle tiles + mirrored stores (fp64 tiled engine, d > 64);
    # odd d exercises the scalar-store path; R_out and the residual form included
    flags = [0, P.NSERIES_ELIDE_TRIVIAL, P.NSERIES_RFORM_TELESCOPE][extra] | P.NSERIES_SYMMETRIC
    G = inputs.random_matrix(d, 500 + d, 0.7)
    A = 0.5 * (G + G.T)
    S, R, st = _run(h, A, steps, flags=flags, want_R=True)
    assert np.array_equal(S, S.T) and np.array_equal(R, R.T)        # mirrored, bit for bit
    Sref, Rref = _oracle_full(A, steps, want_R=True)
    assert O.rel_fro(S, Sref) <= TOL64, (d, steps, flags)
    scale = float(np.sqrt(np.sum(np.asarray(Sref, dtype=LD) ** 2)))
    assert float(np.sqrt(np.sum((R.astype(LD) - Rref) ** 2))) / scale <= 1e-13
    # same products as the general path
    S2, _, st2 = _run(h, A, steps, flags=flags & ~P.NSERIES_SYMMETRIC, want_R=True)
    assert st["products"] == st2["products"]
    assert O.rel_fro(S, S2) <= 1e-13


@pytest.mark.parametrize("d", [100, 300, 512, 1000])
@pytest.mark.parametrize("steps,extra", [([9, 9], 0), ([15, 15], 0), ([15, 1, 5], 1), ([2] * 5, 0),
                                         ([5, 5], 1), ([3, 1, 9], 0)])
def test_symmetric_mode_f32(h, d, steps, extra):
    # fp32 engine with NSERIES_SYMMETRIC: upper-triangle 256x256 pair tiles, mirrored x/hi/lo
    # planes (no transposed operand planes); tolerance 2e-5 against the oracle on fl32(A)
    flags = [0, P.NSERIES_ELIDE_TRIVIAL][extra] | P.NSERIES_SYMMETRIC
    G = inputs.random_matrix(d, 700 + d, 0.7)
    A = (0.5 * (G + G.T)).astype(np.float32).astype(np.float64)
    S, R, _ = _run(h, A, steps, flags=flags, want_R=True, dtype=torch.float32)
    assert np.array_equal(S, S.T) and np.array_equal(R, R.T)
    Sref = _oracle_full(A, steps)
    assert O.rel_fro(S.astype(np.float64), Sref) <= 2e-5, (d, steps, flags)
    S2, _, _ = _run(h, A, steps, flags=flags & ~P.NSERIES_SYMMETRIC, dtype=torch.float32)
    assert O.rel_fro(S.astype(np.float64), S2.astype(np.float64)) <= 2e-5


@pytest.mark.parametrize("d,steps,dt,flags", [(300, [15, 15], "f64", 0), (300, [9, 9], "f32", 0),
                                              (257, [5, 1, 2], "f64", 0), (40, [9, 9], "f64", 0),
                                              (512, [15, 15], "f64", 1)])
def test_host_api_overlapped_copy_out(h, d, steps, dt, flags):
    # nseries_eval_host copies S out on a side stream as soon as the op writing S finishes
    # (overlapping the trailing product); S and R must still be complete and correct, with and
    # without graph replay (second call replays the cached graph)
    G = inputs.random_matrix(d, 900 + d, 0.7)
    A = 0.5 * (G + G.T) if flags else G
    if dt == "f32":
        A = A.astype(np.float32).astype(np.float64)
    k = OP.plan_reaches(steps)
    fl = _flags(steps) | (P.NSERIES_SYMMETRIC if flags else 0)
    plan = P.nseries_plan_finalize(steps, k, fl)
    Ah = np.ascontiguousarray(A.astype(np.float32) if dt == "f32" else A)
    Sref, Rref = _oracle_full(A, steps, want_R=True)
    tol = 2e-5 if dt == "f32" else TOL64
    for _ in range(2):
        Sh = np.full_like(Ah, np.nan)
        Rh = np.full_like(Ah, np.nan)
        P.nseries_eval_host(h, Ah, d, k, plan=plan, S=Sh, R_out=Rh, flags=fl)
        assert O.rel_fro(Sh.astype(np.float64), Sref) <= tol
        assert np.all(np.isfinite(Rh))


@pytest.mark.parametrize("d,dt", [(200, "f64"), (300, "f32"), (40, "f64")])
def test_host_api_async_pipeline(h, d, dt):
    # NSERIES_HOST_ASYNC: 5 different matrices through nseries_eval_host without synchronizing
    # (two staging sets alternate, copy-in of matrix i+1 overlaps evaluation i); after
    # nseries_host_sync every S_i and R_i equals the synchronous call's bits and the oracle
    steps = [9, 2]
    k = OP.plan_reaches(steps)
    plan = P.nseries_plan_finalize(steps, k, 0)
    npdt = np.float32 if dt == "f32" else np.float64
    tdt = torch.float32 if dt == "f32" else torch.float64
    As = [torch.from_numpy(inputs.random_matrix(d, 40 + i, 0.7).astype(npdt)).pin_memory() for i in range(5)]
    Ss = [torch.full_like(a, float("nan")).pin_memory() for a in As]
    Rs = [torch.full_like(a, float("nan")).pin_memory() for a in As]
    for a, s_, r in zip(As, Ss, Rs):
        P.nseries_eval_host(h, a, d, k, plan=plan, S=s_, R_out=r, flags=P.NSERIES_HOST_ASYNC, dtype=P.NSERIES_F32 if dt == "f32" else P.NSERIES_F64)
    P.nseries_host_sync(h)
    tol = 2e-5 if dt == "f32" else TOL64
    for a, s_, r in zip(As, Ss, Rs):
        Sy = torch.empty_like(a)
        Ry = torch.empty_like(a)
        P.nseries_eval_host(h, a, d, k, plan=plan, S=Sy, R_out=Ry)
        assert torch.equal(s_, Sy) and torch.equal(r, Ry)
        ref = _oracle_full(a.numpy().astype(np.float64), steps)
        assert O.rel_fro(s_.numpy().astype(np.float64), ref) <= tol
    assert tdt == As[0].dtype


@pytest.mark.slow
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_large_ragged_d(h, dt):
    # d = 10000 (not a multiple of any tile size; 79 x 79 tiles of 128, odd M-pair count for the
    # fp32 clusters); k = 9 via radix-9 (5 products) checked on 16 seeded probe columns
    d, steps = 10000, [9]
    rng = np.random.default_rng(31)
    A = (0.6 / np.sqrt(d)) * rng.standard_normal((d, d))
    if dt == "f32":
        A = A.astype(np.float32).astype(np.float64)
    V, _ = inputs.probe_block(d, 31)
    S, _, _ = _run(h, A, steps, dtype=torch.float64 if dt == "f64" else torch.float32)
    err = _probe_parity(S.astype(np.float64), A, steps, V, False)
    assert err <= (TOL64 if dt == "f64" else 2e-5), err


@pytest.mark.slow
@pytest.mark.parametrize("dt,d", [("f64", 16384), ("f32", 16384), ("f64", 20000)])
def test_largest_sizes(h, dt, d):
    # beyond the BASELINE configs: d = 16384 (2 GiB per fp64 matrix, 4096 tiles of 128^2, 64
    # k-tiles per CTA ... 512 in the fp32 engine) and d = 20000 (ragged: 157 tiles per side);
    # k = 9 by radix-9 (5 products), 4 seeded probe columns against the long-double oracle
    steps = [9]
    rng = np.random.default_rng(d)
    A = (0.6 / np.sqrt(d)) * rng.standard_normal((d, d))
    if dt == "f32":
        A = A.astype(np.float32).astype(np.float64)
    V, _ = inputs.probe_block(d, 7, n_unit=2, n_gauss=2)
    S, _, _ = _run(h, A, steps, dtype=torch.float64 if dt == "f64" else torch.float32)
    err = _probe_parity(S.astype(np.float64), A, steps, V, False)
    assert err <= (TOL64 if dt == "f64" else 2e-5), err


@pytest.mark.parametrize("steps,printed", [([9, 9], 4.0e-4), ([5, 5, 5], 3.4e-6), ([2] * 7, 2.5e-6),
                                           ([2] * 9, None), ([5] * 4, None), ([9] * 3, None)])
def test_table3_on_gpu(h, steps, printed):
    # the paper's Table 3 workload (d = 500, normal A = 0.9 Omega D Omega^T,
    # D = linspace(-1, 1), reading R13) through the GPU engine: the normal residual
    # ||I - (I - A) S_k||_F of the returned S rounds to the printed value;
    # for k >= 512 the paper prints the binary64 floor (~1e-13), met here as <= 1e-12
    A, _, _ = inputs.table3_matrix()
    S, _, _ = _run(h, A, steps)
    d = A.shape[0]
    res = float(np.linalg.norm(np.eye(d) - S + A @ S))
    if printed is not None:
        assert float(f"{res:.1e}") == printed, res
    else:
        assert res <= 1e-12, res


def test_host_api_async_size_changes(h):
    # NSERIES_HOST_ASYNC calls of growing and shrinking d on one handle: the staging sets are
    # re-allocated (after draining the pipeline) when a larger matrix arrives; every result is
    # the synchronous call's
    steps = [5, 2]
    k = OP.plan_reaches(steps)
    plan = P.nseries_plan_finalize(steps, k, 0)
    mats, outs = [], []
    for i, d in enumerate([40, 300, 70, 520, 300]):
        a = torch.from_numpy(inputs.random_matrix(d, 60 + i, 0.7)).pin_memory()
        s_ = torch.full_like(a, float("nan")).pin_memory()
        P.nseries_eval_host(h, a, d, k, plan=plan, S=s_, flags=P.NSERIES_HOST_ASYNC)
        mats.append(a)
        outs.append(s_)
    P.nseries_host_sync(h)
    for a, s_ in zip(mats, outs):
        ref = torch.empty_like(a)
        P.nseries_eval_host(h, a, a.shape[0], k, plan=plan, S=ref)
        assert torch.equal(s_, ref)


# ---------------------------------------------------------------- naive radix-m (NEXT-2)

NAIVE_PLANS = [[7, 7, 7], [11, 9], [13], [7, 1, 11], [4, 4], [1, 13, 2], [32], [6, 15]]


@pytest.mark.parametrize("d", [1, 5, 33, 64, 100, 300])
@pytest.mark.parametrize("steps", NAIVE_PLANS)
@pytest.mark.parametrize("extra", [0, P.NSERIES_ELIDE_TRIVIAL])
def test_parity_naive_radix(h, d, steps, extra):
    # naive radix-m splitting: m - 2 powers with T_m accumulated in their
    # epilogues, concatenation, next power; exact plans against C-1, with radix 15 against C-2
    A = inputs.random_matrix(d, 500 + d, 0.7)
    S, R, st = _run(h, A, steps, flags=extra, want_R=True)
    Sref, Rref = _oracle_full(A, steps, want_R=True)
    assert O.rel_fro(S, Sref) <= TOL64, (d, steps)
    scale = float(np.sqrt(np.sum(np.asarray(Sref, dtype=LD) ** 2)))
    assert float(np.sqrt(np.sum((R.astype(LD) - Rref) ** 2))) / scale <= 1e-13


@pytest.mark.parametrize("d", [16, 64, 200])
@pytest.mark.parametrize("steps", [[7, 7], [11, 9], [13, 1, 4]])
def test_parity_naive_radix_f32(h, d, steps):
    A = inputs.random_matrix(d, 600 + d, 0.7).astype(np.float32)
    S, _, _ = _run(h, A.astype(np.float64), steps, dtype=torch.float32)
    assert O.rel_fro(S, _oracle_full(A.astype(np.float64), steps)) <= TOL32, (d, steps)


def test_naive_radix_probes_d1024(h):
    # config-2-sized A (d = 1024, rho ~ 0.93): x7^3 (k = 343, 21 products) on 16 probe columns
    A = inputs.cfg2()
    V, _ = inputs.probe_block(A.shape[0], 1)
    S, _, st = _run(h, A, [7, 7, 7])
    assert st["products"] == 21
    assert _probe_parity(S, A, [7, 7, 7], V, False) <= TOL64
