"""GPU checks of the boundary's accounting: paper vs executed product
counts, per-step device times under NSERIES_SYNC_STATS, and NSERIES_CHECK_FINITE (fused NaN/Inf
count of S; config 4's divergent matrices)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2602_11843_b200 as P  # noqa: E402
from oracle import plan as OP  # noqa: E402
from paper_2602_11843_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def h():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    handle = P.nseries_create(0)
    yield handle
    P.nseries_destroy(handle)


def _eval(h, A, steps, flags=0, R=False):
    d = A.shape[0]
    k = OP.plan_reaches(steps)
    flags |= P.NSERIES_ALLOW_APPROX if 15 in steps else 0
    plan = P.nseries_plan_finalize(steps, k, flags)
    S = torch.empty_like(A)
    Rb = torch.empty_like(A) if R else None
    P.nseries_eval(h, A, d, k, plan=plan, S=S, R_out=Rb, flags=flags)
    torch.cuda.synchronize()
    return S, P.nseries_last_stats(h)


@pytest.mark.parametrize("d,dt", [(64, torch.float64), (200, torch.float64), (32, torch.float32), (200, torch.float32)])
@pytest.mark.parametrize("steps", [[9, 9], [15, 1, 5], [2] * 5, [7, 3]])
def test_products_paper_and_exec(h, d, dt, steps):
    A = torch.from_numpy(inputs.random_matrix(d, 3, 0.5)).to("cuda", dt)
    paper = OP.plan_products(steps)
    _, st = _eval(h, A, steps)
    assert st["products_paper"] == paper and st["products_exec"] == paper == st["products"]
    _, st = _eval(h, A, steps, flags=P.NSERIES_ELIDE_TRIVIAL)
    assert st["products_paper"] == paper
    assert st["products_exec"] == st["products"] == OP.plan_products(steps, True) < paper


@pytest.mark.parametrize("d,dt", [(300, torch.float64), (300, torch.float32), (1024, torch.float64)])
def test_sync_stats_per_step_times(h, d, dt):
    A = torch.from_numpy(inputs.random_matrix(d, 4, 0.5)).to("cuda", dt)
    steps = [9, 1, 5, 2]
    S_ref, _ = _eval(h, A, steps)
    S, st = _eval(h, A, steps, flags=P.NSERIES_SYNC_STATS)
    assert torch.equal(S, S_ref)                       # eager launches, same kernels
    assert len(st["ms_step"]) == len(steps) and st["ms_total"] > 0
    assert all(t > 0 for t in st["ms_step"])
    assert abs(sum(st["ms_step"]) - st["ms_total"]) <= 0.05 * st["ms_total"] + 0.02
    # the radix-9 step (5 products) takes longer than the "+1" step (1 product)
    assert st["ms_step"][0] > st["ms_step"][1]


def test_sync_stats_single_launch_has_no_steps(h):
    A = torch.from_numpy(inputs.cfg1()).cuda()
    _, st = _eval(h, A, [9, 9], flags=P.NSERIES_SYNC_STATS)
    assert st["launches"] == 1 and st["ms_step"] == [] and st["ms_total"] > 0


def _blowup(d, dt, scale):
    A = np.eye(d) * scale + inputs.random_matrix(d, 5, 0.1)
    return torch.from_numpy(A).to("cuda", dt)


@pytest.mark.parametrize("d,dt,scale,steps", [
    (200, torch.float64, 40.0, [9, 9, 9]),     # tiled fp64: fused count in the final epilogue
    (64, torch.float64, 40.0, [9, 9, 9]),      # single-launch cluster kernel: separate pass
    (200, torch.float32, 8.0, [9, 9]),         # tiled fp32
    (32, torch.float32, 8.0, [9, 9]),          # one-launch warp-group kernel: fused
])
def test_check_finite_single(h, d, dt, scale, steps):
    ok = torch.from_numpy(inputs.random_matrix(d, 6, 0.5)).to("cuda", dt)
    _, st = _eval(h, ok, steps, flags=P.NSERIES_CHECK_FINITE)
    assert st["nonfinite"] == 0
    bad = _blowup(d, dt, scale)
    with pytest.raises(P.NSeriesError) as e:
        _eval(h, bad, steps, flags=P.NSERIES_CHECK_FINITE)
    assert e.value.status == 10
    st = P.nseries_last_stats(h)
    assert st["nonfinite"] > 0
    # the result is written and the count is exact; the handle stays usable (not sticky)
    k = OP.plan_reaches(steps)
    plan = P.nseries_plan_finalize(steps, k, 0)
    S = torch.empty_like(bad)
    P.nseries_eval(h, bad, d, k, plan=plan, S=S)
    torch.cuda.synchronize()
    assert st["nonfinite"] == int((~torch.isfinite(S)).sum())
    _, st = _eval(h, ok, steps, flags=P.NSERIES_CHECK_FINITE)
    assert st["nonfinite"] == 0


@pytest.mark.parametrize("d,dt", [(32, torch.float32), (48, torch.float32), (32, torch.float64)])
def test_check_finite_batched_config4(h, d, dt):
    # config 4 (84% of the A_b have rho > 1, up to 1.4): finite at k = 81, overflowing
    # at k = 9^4 for the divergent ones (1.4^6560 ~ 1e958); the count covers every matrix
    Ab = inputs.cfg4(batch=512, n=d)
    A = torch.from_numpy(Ab).to("cuda", dt)
    S = torch.empty_like(A)
    for steps, expect_bad in (([9, 9], False), ([9, 9, 9, 9], True)):
        k = OP.plan_reaches(steps)
        plan = P.nseries_plan_finalize(steps, k, 0)
        if expect_bad:
            with pytest.raises(P.NSeriesError) as e:
                P.nseries_eval_batched_strided(h, A, d * d, A.shape[0], d, k, plan=plan, S=S,
                                               flags=P.NSERIES_CHECK_FINITE)
            assert e.value.status == 10
        else:
            P.nseries_eval_batched_strided(h, A, d * d, A.shape[0], d, k, plan=plan, S=S,
                                           flags=P.NSERIES_CHECK_FINITE)
        torch.cuda.synchronize()
        st = P.nseries_last_stats(h)
        assert st["nonfinite"] == int((~torch.isfinite(S)).sum())
        assert (st["nonfinite"] > 0) == expect_bad
