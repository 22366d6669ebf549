"""Harness for a multi-GPU box (not runnable on this one-GPU pool): validates the row-sharded chain
across real ranks -- NCCL allgather-v gathers and NSERIES_SHARDED_DIRECT in-place peer reads over
NVLink (CUDA IPC arenas) -- against the single-GPU engine, and times both.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
      --master-port 29511 tools/check_sharded_multi.py [d] [plan...]

Every rank builds the same seeded A (inputs.cfg5 at d = 8192, else a random matrix), evaluates
its row block both ways, and rank 0 gathers the blocks and compares them with nseries_eval on the
full matrix (relative Frobenius <= 1e-12) and prints one JSON line."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_11843_b200 as P  # noqa: E402
from paper_2602_11843_b200 import inputs, replicas  # noqa: E402


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    steps = [int(x) for x in sys.argv[2:]] or None
    rank, world, local = replicas.setup(2 if "RANK" in os.environ else 1)
    torch.cuda.set_device(local)
    h = P.nseries_create(local)
    uid = replicas.exchange_blobs(P.nseries_comm_unique_id() if rank == 0 else b"", world)[0]
    P.nseries_comm_init(h, uid, world, rank)
    fl = P.NSERIES_ALLOW_APPROX
    if steps:
        k = 1
        for m in steps:                 # the k a step list reaches: x m multiplies, "+1" adds one
            k = k + 1 if m == 1 else k * m
        plan = P.nseries_plan_finalize(steps, k, fl)
    else:
        k = 10000
        plan = P.nseries_plan_build(k, P.NSERIES_PLAN_AUTO, [15, 9, 5, 2], fl)
    A = inputs.cfg5(device="cuda") if d == 8192 else torch.from_numpy(inputs.random_matrix(d, 5, 0.8)).cuda()
    r0, rows = P.nseries_shard_rows(d, world, rank)
    A_blk = A[r0:r0 + rows].contiguous()
    out = {"world": world, "d": d, "k": k}
    results = {}
    for mode in ("gather", "direct"):
        f = fl | (P.NSERIES_SHARDED_DIRECT if mode == "direct" else 0)
        if mode == "direct":
            need = P.nseries_sharded_arena_bytes(d, world, 1, k, plan, flags=f)
            P.nseries_peer_import(h, replicas.exchange_blobs(P.nseries_peer_export(h, need), world))
        S_blk = torch.empty_like(A_blk)
        run = lambda: P.nseries_eval_sharded(h, [A_blk], rank, world, d, k, plan=plan, S_shards=[S_blk], flags=f)
        run()
        torch.cuda.synchronize()
        replicas.barrier(world)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        out[f"{mode}_ms"] = replicas.max_over_ranks(e0.elapsed_time(e1), world)
        out[f"{mode}_gathers"] = P.nseries_last_stats(h)["gathers"]
        blocks = [torch.empty(P.nseries_shard_rows(d, world, r)[1], d, dtype=torch.float64, device="cuda")
                  for r in range(world)]
        if world > 1:
            if all(b.shape[0] == rows for b in blocks):
                dist.all_gather(blocks, S_blk)
            else:
                raise SystemExit("use d divisible by the rank count")
        else:
            blocks = [S_blk]
        results[mode] = torch.cat(blocks)
    if rank == 0:
        S = torch.empty_like(A)
        P.nseries_eval(h, A, d, k, plan=plan, S=S, flags=fl)
        torch.cuda.synchronize()
        for mode, Sm in results.items():
            out[f"{mode}_rel_fro_vs_dense"] = float((Sm - S).norm() / S.norm())
        out["ok"] = all(out[f"{m}_rel_fro_vs_dense"] <= 1e-12 for m in results)
        print(json.dumps(out))
    P.nseries_destroy(h)
    replicas.teardown(world)


if __name__ == "__main__":
    main()
