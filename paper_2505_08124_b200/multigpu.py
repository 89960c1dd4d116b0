"""Multi-GPU plumbing of the embedding pass: one process per GPU
(torch.distributed over NCCL), views sharded like the reference's workers
(pipeline.hpp:309-311: round-robin idx % workers == rank, or contiguous
blocks), one reduce-scatter of the N x D fp32 partial sums + N totals
(the paper's "sum tensors from all GPUs"), each rank then
normalises its row shard.  No other data-path collective exists.
"""
from __future__ import annotations


def shard_views(n_views: int, world: int, rank: int, contiguous: bool = False) -> list:
    """pipeline.hpp:307-311 assignment of manifest indices to a worker."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if contiguous:
        block = (n_views + world - 1) // world if n_views else 1
        return [v for v in range(n_views) if v // block == rank]
    return [v for v in range(n_views) if v % world == rank]


def padded_rows(n: int, world: int) -> int:
    """Rows padded to a multiple of the world size (reduce-scatter needs equal shards)."""
    return (n + world - 1) // world * world


def shard_rows(n: int, world: int, rank: int):
    """[lo, hi) rows of the table this rank normalises after the reduce-scatter."""
    per = padded_rows(n, world) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def reduce_scatter_rows(out_shard, full, group=None):
    """Sum `full` ([world*shard, ...]) over ranks, leave this rank's shard in
    `out_shard`.  NCCL: one reduce_scatter_tensor.  Backends without it (gloo
    on CPU, used by the tests) fall back to all_reduce + slice -- same result."""
    import torch.distributed as dist
    backend = dist.get_backend(group)
    if backend == "nccl":
        dist.reduce_scatter_tensor(out_shard, full, group=group)
        return out_shard
    rank = dist.get_rank(group)
    per = out_shard.shape[0]
    tmp = full.clone()
    dist.all_reduce(tmp, group=group)
    out_shard.copy_(tmp[rank * per:(rank + 1) * per])
    return out_shard
