"""Multi-GPU plumbing of the embedding pass: one process per GPU
(torch.distributed over NCCL), views sharded like the reference's workers
(pipeline.hpp:309-311: round-robin idx % workers == rank, or contiguous
blocks), one reduce-scatter of the N x D fp32 partial sums + N totals
(the paper's "sum tensors from all GPUs"), each rank then
normalises its row shard.  No other data-path collective exists.

Query over a row-sharded store: each rank answers every
query over its own rows, one all_gather of the per-rank (id, sim) top-k lists
(Q x k x 8 B per rank), and a merge by the reference's order (sim desc, id
asc; vecstore.hpp:107-110).
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


def merge_topk(ids, sims, counts, k: int):
    """Merge per-shard top-k lists.  ids/sims: [R, Q, k] torch tensors (R
    shards), counts: [R, Q] valid entries per list.  Returns (ids [Q, k],
    sims [Q, k], counts [Q]) -- the first min(k, sum counts) records of the
    union under (sim desc, id asc), exactly what a single store holding all
    shards' rows returns (vecstore.hpp:121-132)."""
    import torch
    r, q, kk = ids.shape
    valid = torch.arange(kk, device=ids.device).view(1, 1, kk) < counts.view(r, q, 1)
    s = torch.where(valid, sims, torch.full_like(sims, float("-inf")))
    i = torch.where(valid, ids.to(torch.int64), torch.full_like(ids, 0, dtype=torch.int64) + (1 << 40))
    s = s.permute(1, 0, 2).reshape(q, r * kk)
    i = i.permute(1, 0, 2).reshape(q, r * kk)
    # two stable sorts: id ascending, then sim descending
    o = torch.argsort(i, dim=1, stable=True)
    s, i = torch.gather(s, 1, o), torch.gather(i, 1, o)
    o = torch.argsort(s, dim=1, descending=True, stable=True)
    s, i = torch.gather(s, 1, o)[:, :k], torch.gather(i, 1, o)[:, :k]
    tot = torch.clamp(counts.sum(dim=0), max=k)
    return i.to(torch.int64), s, tot


def sharded_query_topk(local_topk, queries, k: int, group=None):
    """Top-k over a store whose rows are sharded across the ranks of `group`.
    `local_topk(queries, k) -> (ids [Q,k] u32, sims [Q,k] f32, counts [Q])` answers
    over this rank's rows (the product passes the device query,
    `Context.query_topk`).  One all_gather of the lists, then `merge_topk`."""
    import numpy as np
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    li, ls, lc = local_topk(queries, k)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    ti = torch.from_numpy(np.asarray(li, np.int64)).to(dev)
    ts = torch.from_numpy(np.asarray(ls, np.float32)).to(dev)
    tc = torch.from_numpy(np.asarray(lc, np.int64)).to(dev)
    gi = [torch.empty_like(ti) for _ in range(world)]
    gs = [torch.empty_like(ts) for _ in range(world)]
    gc = [torch.empty_like(tc) for _ in range(world)]
    dist.all_gather(gi, ti, group=group)
    dist.all_gather(gs, ts, group=group)
    dist.all_gather(gc, tc, group=group)
    mi, ms, mc = merge_topk(torch.stack(gi), torch.stack(gs), torch.stack(gc), k)
    return mi.cpu().numpy().astype(np.uint32), ms.cpu().numpy(), mc.cpu().numpy().astype(np.uint64)
