"""GPU parity of the row-sharded chain (include/nseries.h
nseries_eval_sharded): the plan evaluated on row blocks with a gathered right factor per
product must match the single-matrix engine to rounding (the row split changes which CTA
computes an element, not its K loop, but the executor may take X.Y as Y.X to avoid a gather,
which reorders the rounding) and the oracle.  Covers all-local shards (device-copy gathers), the
NCCL allgather-v path with a one-rank communicator (grouped ncclBroadcast, every root local) and
NSERIES_SHARDED_DIRECT (right factors read in place from their row blocks, no gather)."""
import numpy as np
import pytest
import torch

import paper_2602_11843_b200 as P
from paper_2602_11843_b200 import inputs
from oracle import plan as OP
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    x = P.nseries_create(0)
    yield x
    P.nseries_destroy(x)


@pytest.fixture(scope="module")
def hc():
    """A handle with a one-rank NCCL communicator."""
    x = P.nseries_create(0)
    P.nseries_comm_init(x, P.nseries_comm_unique_id(), 1, 0)
    yield x
    P.nseries_destroy(x)


def _flags(steps, extra=0):
    return extra | (P.NSERIES_ALLOW_APPROX if 15 in steps else 0)


def _shards(T, n):
    d = T.shape[0]
    out = []
    for s in range(n):
        r0, m = P.nseries_shard_rows(d, n, s)
        out.append(T[r0:r0 + m].contiguous())
    return out


def _sharded(h, A, steps, n, want_R=False, extra=0):
    d = A.shape[0]
    k = OP.plan_reaches(steps)
    flags = _flags(steps, extra)
    plan = P.nseries_plan_finalize(steps, k, flags)
    As = _shards(A, n)
    Ss = [torch.full_like(a, float("nan")) for a in As]
    Rs = [torch.full_like(a, float("nan")) for a in As] if want_R else None
    P.nseries_eval_sharded(h, As, 0, n, d, k, plan=plan, S_shards=Ss, R_shards=Rs, flags=flags)
    torch.cuda.synchronize()
    st = P.nseries_last_stats(h)
    S = torch.cat(Ss).cpu().numpy()
    R = torch.cat(Rs).cpu().numpy() if want_R else None
    return S, R, st


def _dense(h, A, steps, want_R=False, extra=0):
    d = A.shape[0]
    k = OP.plan_reaches(steps)
    flags = _flags(steps, extra)
    plan = P.nseries_plan_finalize(steps, k, flags)
    S = torch.empty_like(A)
    R = torch.empty_like(A) if want_R else None
    P.nseries_eval(h, A, d, k, plan=plan, S=S, R_out=R, flags=flags)
    torch.cuda.synchronize()
    return S.cpu().numpy(), (R.cpu().numpy() if want_R else None)


@pytest.mark.parametrize("d", [9, 40, 65, 200, 1100])
@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("steps", [[9, 9], [15, 15], [2] * 6, [15, 1, 5], [5, 1, 9], [3, 3]])
def test_sharded_equals_dense(h, d, n, steps):
    A = torch.from_numpy(inputs.random_matrix(d, 500 + d, 0.8)).cuda()
    S, _, st = _sharded(h, A, steps, n)
    Sd, _ = _dense(h, A, steps)
    assert O.rel_fro(S, Sd) <= 1e-13, (d, n, steps)
    if d <= 200:                                            # and the oracle (C-1 / C-2)
        ref = (O.plan_apply(A.cpu().numpy(), steps, np.eye(d)) if 15 in steps
               else O.full_series(A.cpu().numpy(), OP.plan_reaches(steps)))
        assert O.rel_fro(S, ref) <= 1e-11
    assert st["products"] == OP.plan_products(steps, False)
    assert st["launches"] == n * st["n_ops"] and st["gathers"] >= 1


@pytest.mark.parametrize("n", [1, 3])
@pytest.mark.parametrize("extra", [0, P.NSERIES_ELIDE_TRIVIAL])
def test_sharded_residual_and_oracle(h, n, extra):
    d = 96
    steps = [9, 1, 2]
    An = inputs.random_matrix(d, 31, 0.7)
    A = torch.from_numpy(An).cuda()
    S, R, _ = _sharded(h, A, steps, n, want_R=True, extra=extra)
    Sd, Rd = _dense(h, A, steps, want_R=True, extra=extra)
    assert O.rel_fro(S, Sd) <= 1e-13 and O.rel_fro(R, Rd) <= 1e-12
    k = OP.plan_reaches(steps)
    assert O.rel_fro(S, O.full_series(An, k)) <= 1e-11      # exact plan: the C-1 oracle


@pytest.mark.parametrize("n", [1, 4])
def test_sharded_nccl_one_rank(hc, h, n):
    # the allgather-v code path (grouped ncclBroadcast) with every shard owned by rank 0
    d = 300
    A = torch.from_numpy(inputs.random_matrix(d, 8, 0.8)).cuda()
    S, _, st = _sharded(hc, A, [9, 9], n)
    Sd, _ = _dense(h, A, [9, 9])
    assert O.rel_fro(S, Sd) <= 1e-13 and st["gathers"] >= 1
    S2, _, _ = _sharded(h, A, [9, 9], n)                   # device-copy gathers: same bits
    assert np.array_equal(S, S2)


def test_sharded_config3():
    # config 3 at full size, 8 row blocks (512 rows each) on one GPU, headline plan
    hh = P.nseries_create(0)
    try:
        A, _, _ = inputs.cfg3(device="cuda")
        S, _, st = _sharded(hh, A, [15, 15, 15], 8)
        Sd, _ = _dense(hh, A, [15, 15, 15])
        assert O.rel_fro(S, Sd) <= 1e-12
        assert st["products"] == 18
        # gathers of factors that exist before the preceding product are issued ahead of it
        assert st["gathers"] == 14 and st["gathers_prefetched"] == 2
    finally:
        P.nseries_destroy(hh)


@pytest.mark.parametrize("d,n", [(256, 1), (256, 2), (256, 8), (96, 3), (1024, 8)])
@pytest.mark.parametrize("steps", [[9, 9], [15, 15], [2] * 6, [15, 1, 5], [5, 1, 9], [3, 3]])
def test_sharded_direct(h, d, n, steps):
    # NSERIES_SHARDED_DIRECT: every right factor read in place from its row blocks -- no gather
    A = torch.from_numpy(inputs.random_matrix(d, 700 + d + n, 0.8)).cuda()
    S, _, st = _sharded(h, A, steps, n, extra=P.NSERIES_SHARDED_DIRECT)
    Sd, _ = _dense(h, A, steps)
    assert O.rel_fro(S, Sd) <= 1e-13, (d, n, steps)
    if d <= 256:
        ref = (O.plan_apply(A.cpu().numpy(), steps, np.eye(d)) if 15 in steps
               else O.full_series(A.cpu().numpy(), OP.plan_reaches(steps)))
        assert O.rel_fro(S, ref) <= 1e-11
    assert st["gathers"] == 0 and st["launches"] == n * st["n_ops"]
    assert st["products"] == OP.plan_products(steps, False)


@pytest.mark.parametrize("n", [1, 4])
def test_sharded_direct_residual(h, n):
    d = 128
    steps = [9, 1, 2]
    An = inputs.random_matrix(d, 41, 0.7)
    A = torch.from_numpy(An).cuda()
    S, R, st = _sharded(h, A, steps, n, want_R=True, extra=P.NSERIES_SHARDED_DIRECT)
    Sd, Rd = _dense(h, A, steps, want_R=True)
    assert O.rel_fro(S, Sd) <= 1e-13 and O.rel_fro(R, Rd) <= 1e-12 and st["gathers"] == 0
    assert O.rel_fro(S, O.full_series(An, OP.plan_reaches(steps))) <= 1e-11


@pytest.mark.parametrize("d,n", [(200, 3), (100, 4), (1100, 8)])
def test_sharded_direct_falls_back(h, d, n):
    # non-uniform blocks or blocks of fewer than 32 / not a multiple of 32 rows: gathers
    A = torch.from_numpy(inputs.random_matrix(d, 900 + d, 0.8)).cuda()
    S, _, st = _sharded(h, A, [9, 9], n, extra=P.NSERIES_SHARDED_DIRECT)
    Sd, _ = _dense(h, A, [9, 9])
    assert O.rel_fro(S, Sd) <= 1e-13 and st["gathers"] >= 1


def test_sharded_direct_config3():
    # config 3 at full size in 8 row blocks of 512 rows, right factors read in place
    hh = P.nseries_create(0)
    try:
        A, _, _ = inputs.cfg3(device="cuda")
        S, _, st = _sharded(hh, A, [15, 15, 15], 8, extra=P.NSERIES_SHARDED_DIRECT)
        Sd, _ = _dense(hh, A, [15, 15, 15])
        assert O.rel_fro(S, Sd) <= 1e-12
        assert st["products"] == 18 and st["gathers"] == 0
    finally:
        P.nseries_destroy(hh)


@pytest.mark.parametrize("d,n,steps", [(256, 1, [9, 9]), (256, 4, [15, 15]), (512, 8, [15, 1, 5]),
                                        (1024, 2, [2] * 6), (96, 3, [5, 1, 9])])
def test_sharded_direct_peer_arena(d, n, steps):
    # the cross-process NSERIES_SHARDED_DIRECT path on one GPU: a one-rank communicator owning all
    # n shards, this rank's arena exported and "imported" (own entry), values' blocks in the arena,
    # a one-int all-reduce barrier after every op; no gathers
    hh = P.nseries_create(0)
    try:
        P.nseries_comm_init(hh, P.nseries_comm_unique_id(), 1, 0)
        k = OP.plan_reaches(steps)
        flags = _flags(steps, P.NSERIES_SHARDED_DIRECT)
        plan = P.nseries_plan_finalize(steps, k, flags)
        need = P.nseries_sharded_arena_bytes(d, n, n, k, plan, flags=flags)
        P.nseries_peer_import(hh, [P.nseries_peer_export(hh, need)])
        A = torch.from_numpy(inputs.random_matrix(d, 77 + d + n, 0.8)).cuda()
        As = _shards(A, n)
        Ss = [torch.full_like(a, float("nan")) for a in As]
        for _ in range(2):                  # repeated evals reuse the arena (start barrier)
            P.nseries_eval_sharded(hh, As, 0, n, d, k, plan=plan, S_shards=Ss, flags=flags)
        torch.cuda.synchronize()
        st = P.nseries_last_stats(hh)
        S = torch.cat(Ss).cpu().numpy()
        Sd, _ = _dense(hh, A, steps)
        assert O.rel_fro(S, Sd) <= 1e-13 and st["gathers"] == 0, (d, n, steps)
        ref = (O.plan_apply(A.cpu().numpy(), steps, np.eye(d)) if 15 in steps
               else O.full_series(A.cpu().numpy(), k))
        assert O.rel_fro(S, ref) <= 1e-11
    finally:
        P.nseries_destroy(hh)


def test_sharded_direct_needs_import(hc, h):
    # a communicator but no mapped arenas: NSERIES_SHARDED_DIRECT falls back to the gathers
    d, n = 256, 4
    A = torch.from_numpy(inputs.random_matrix(d, 5, 0.8)).cuda()
    S, _, st = _sharded(hc, A, [9, 9], n, extra=P.NSERIES_SHARDED_DIRECT)
    Sd, _ = _dense(h, A, [9, 9])
    assert O.rel_fro(S, Sd) <= 1e-13 and st["gathers"] >= 1


def test_sharded_rejects(h):
    A = torch.zeros(8, 8, dtype=torch.float64, device="cuda")
    plan = P.nseries_plan_finalize([2], 2, 0)
    with pytest.raises(P.NSeriesError) as e:      # fp32: fp64 only
        P.nseries_eval_sharded(h, [A.float()], 0, 1, 8, 2, plan=plan, S_shards=[A.float().clone()],
                               dtype=P.NSERIES_F32)
    assert e.value.status == 9
    with pytest.raises(P.NSeriesError) as e:      # remote shards without a communicator
        P.nseries_eval_sharded(h, [A[:4].clone()], 0, 2, 8, 2, plan=plan, S_shards=[A[:4].clone()])
    assert e.value.status == 1
    with pytest.raises(P.NSeriesError) as e:      # symmetric mode is not sharded
        P.nseries_eval_sharded(h, [A], 0, 1, 8, 2, plan=plan, S_shards=[A.clone()], flags=P.NSERIES_SYMMETRIC)
    assert e.value.status == 1
    with pytest.raises(P.NSeriesError) as e:      # S aliases A
        P.nseries_eval_sharded(h, [A], 0, 1, 8, 2, plan=plan, S_shards=[A])
    assert e.value.status == 5
