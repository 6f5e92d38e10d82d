"""Multi-GPU plumbing for the replica-parallel kNN_L.

The path shards without a data-path collective: every rank holds a full
replica of the BDL-tree and answers its own queries.  torch.distributed is
used only to (a) agree on the max-over-ranks elapsed time and (b) split a
query batch when a caller wants query sharding instead of replicas.
"""
from __future__ import annotations

import os


def rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def shard_range(n: int, rank: int, world: int):
    """contiguous [lo, hi) slice of n items for `rank` (sizes differ by at most 1)"""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(x: float, device=None) -> float:
    """max of a per-rank scalar (e.g. elapsed seconds) over the process group (identity when not distributed)"""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank: float, world: int, max_seconds: float) -> float:
    """units all ranks processed / the slowest rank's time (weak scaling: equal work per rank)"""
    return units_per_rank * world / max_seconds
