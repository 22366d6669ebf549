"""Host side of the multi-process row-sharded chain, world size 2
over gloo on CPU: the 128-byte NCCL unique id is created by rank 0 through the library and
shipped to rank 1 with torch.distributed (the plumbing bench/users run before
nseries_comm_init), every rank derives the same shard map from nseries_shard_rows, and (for
NSERIES_SHARDED_DIRECT across processes) every rank sizes the same arena with
nseries_sharded_arena_bytes and receives all ranks' 64-byte IPC handles in rank order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, d, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_11843_b200 as P
    try:
        uid = [P.nseries_comm_unique_id() if rank == 0 else None]
        have_uid = True
    except Exception:                       # no libnccl.so.2 on this host: ship a dummy id
        uid, have_uid = [bytes(128) if rank == 0 else None], False
    dist.broadcast_object_list(uid, src=0)
    # this rank's shard (one per rank) and everybody's, derived independently on every rank
    mine = P.nseries_shard_rows(d, world, rank)
    allb = [None] * world
    dist.all_gather_object(allb, mine)
    plan = P.nseries_plan_build(10000, P.NSERIES_PLAN_AUTO, flags=P.NSERIES_ALLOW_APPROX)
    arena = P.nseries_sharded_arena_bytes(d, world, 1, 10000, plan, flags=P.NSERIES_ALLOW_APPROX)
    from paper_2602_11843_b200 import replicas
    # stand-in for nseries_peer_export's handle (no GPU here): 64 rank-specific bytes
    handles = replicas.exchange_blobs(bytes([rank + 1]) * 64, world)
    q.put((rank, uid[0], allb, [P.nseries_shard_rows(d, world, s) for s in range(world)], have_uid,
           arena, handles))
    dist.destroy_process_group()


@pytest.mark.parametrize("d", [1100, 8193])
def test_uid_exchange_and_shard_map(d):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, d, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, uid0, all0, map0, ok0, ar0, hd0), (r1, uid1, all1, map1, ok1, ar1, hd1) = res
    rows_max = max(n for _, n in map0)
    assert ar0 == ar1 and ar0 > 0 and ar0 % (rows_max * d * 8) == 0   # (slots + A) row blocks
    assert hd0 == hd1 == [bytes([1]) * 64, bytes([2]) * 64]
    assert len(uid0) == 128 and uid0 == uid1
    if ok0:
        assert any(uid0)                    # a real NCCL id, not zeros
    assert all0 == all1 == map0 == map1
    assert sum(n for _, n in map0) == d and map0[1][0] == map0[0][1]
