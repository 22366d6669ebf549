"""world_size-2 gloo tests (CPU) of the multi-rank bench plumbing: barrier, max-over-ranks
timing and the whole-job aggregate (replicas only, no data-path collective)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2602_11843_b200 import replicas as R
    r, w, local = R.setup(world, backend="gloo")
    R.barrier(w)
    elapsed = 100.0 + 50.0 * r            # rank 1 is the slow replica
    mx = R.max_over_ranks(elapsed, w, device="cpu")
    val = R.aggregate_rate(10, mx, w)
    q.put((r, w, mx, val))
    R.teardown(w)


@pytest.mark.timeout(120)
def test_two_rank_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=90) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for r, w, mx, val in res:
        assert w == 2
        assert mx == 150.0                  # max over ranks, not the local time
        assert abs(val - 2 * 10 / 0.150) < 1e-9


def test_single_process_defaults():
    from paper_2602_11843_b200 import replicas as R
    assert R.setup(1) == (0, 1, 0)
    assert R.max_over_ranks(3.5, 1) == 3.5
    assert R.aggregate_rate(4, 2000.0, 1) == 2.0


def _slice_worker(rank, world, port, n, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2602_11843_b200 import replicas as R
    r, w, _ = R.setup(world, backend="gloo")
    b0, b1 = R.batch_slice(n, w, r)
    counts = R.gather_counts(b1 - b0, w)
    # every rank sees the same partition: its neighbours' slices from the counts alone
    starts = [sum(counts[:i]) for i in range(w)]
    q.put((r, b0, b1, counts, starts[r] == b0))
    R.teardown(w)


@pytest.mark.timeout(120)
@pytest.mark.parametrize("n", [16384, 7, 1])
def test_batch_slices_two_rank_gloo(n):
    # config 4's batch split over 2 ranks: contiguous, disjoint, covering, sizes
    # within one -- checked from both ranks' own views, no data-path collective involved
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_slice_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=90) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    (r0, a0, a1, c0, ok0), (r1, b0, b1, c1, ok1) = res
    assert (r0, r1) == (0, 1) and ok0 and ok1 and c0 == c1
    assert a0 == 0 and a1 == b0 and b1 == n and abs((a1 - a0) - (b1 - b0)) <= 1


@pytest.mark.parametrize("n,world", [(16384, 8), (16384, 3), (5, 8), (0, 2)])
def test_batch_slice_partition(n, world):
    from paper_2602_11843_b200 import replicas as R
    sl = [R.batch_slice(n, world, r) for r in range(world)]
    assert sl[0][0] == 0 and sl[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
    sizes = [b - a for a, b in sl]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 0
