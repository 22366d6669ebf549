"""Host side of the multi-process row-sharded chain, world size 2
over gloo on CPU: the 128-byte NCCL unique id is created by rank 0 through the library and
shipped to rank 1 with torch.distributed (the plumbing bench/users run before
nseries_comm_init), and every rank derives the same shard map from nseries_shard_rows."""
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
    q.put((rank, uid[0], allb, [P.nseries_shard_rows(d, world, s) for s in range(world)], have_uid))
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
    (r0, uid0, all0, map0, ok0), (r1, uid1, all1, map1, ok1) = res
    assert len(uid0) == 128 and uid0 == uid1
    if ok0:
        assert any(uid0)                    # a real NCCL id, not zeros
    assert all0 == all1 == map0 == map1
    assert sum(n for _, n in map0) == d and map0[1][0] == map0[0][1]
