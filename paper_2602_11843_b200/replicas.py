"""Multi-GPU plumbing for bench.py: one process per GPU, independent replicas.

The single-matrix S_k(A) path is a serial chain of d x d products and does not shard
("replicas only"): N ranks each evaluate their own replica and no data-path
collective exists.  The batched path (config 4) shards by contiguous batch slices
(batch_slice), again without a collective.  torch.distributed is used only for the barrier around the timed region
and for the max-over-ranks reduction of the elapsed time; the whole-job value is
(ranks x steps) / max elapsed.  The same helpers run on CPU with the gloo backend (tests).
"""
from __future__ import annotations

import os


def setup(n_requested, backend=None):
    """Initialise the process group when launched under torchrun with n > 1.
    Returns (rank, world, local_rank)."""
    if n_requested <= 1 or "RANK" not in os.environ:
        return 0, 1, 0
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", 0))
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group(backend)
    return dist.get_rank(), dist.get_world_size(), local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world, device=None):
    """Maximum of a host float over all ranks (elapsed times: the job is as slow as its
    slowest replica)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    if device is None:
        device = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(units_per_rank, elapsed_ms_max, world):
    """Whole-job throughput: all ranks' units / the slowest rank's elapsed time."""
    return world * units_per_rank / (elapsed_ms_max / 1e3)


def batch_slice(n, world, rank):
    """Contiguous slice [b0, b1) of a batch of n independent matrices for `rank` of `world`
    (the batched path shards by batch slices, no collective): floor(n / world)
    matrices each, one more for the first n mod world ranks."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad slice request")
    q, r = divmod(n, world)
    b0 = rank * q + min(rank, r)
    return b0, b0 + q + (1 if rank < r else 0)


def gather_counts(local, world, device="cpu"):
    """All ranks' integers (e.g. matrices each rank evaluated) -- bookkeeping check only."""
    if world <= 1:
        return [int(local)]
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(local)], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [int(x.item()) for x in out]


def exchange_blobs(blob, world):
    """All ranks' byte strings, indexed by rank (e.g. the 64-byte CUDA IPC handles of
    nseries_peer_export, which nseries_peer_import takes in rank order)."""
    if world <= 1:
        return [bytes(blob)]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, bytes(blob))
    return out


def teardown(world):
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
