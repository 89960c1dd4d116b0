"""Multi-GPU plumbing of the embedding pass: one process per GPU
(torch.distributed over NCCL), views sharded like the reference's workers
(pipeline.hpp:309-311: round-robin idx % workers == rank, or contiguous
blocks), one reduce-scatter of the N x D fp32 partial sums + N totals per
combine round (the paper's "sum tensors from all GPUs"; issued
by libsemsplat_b200's own NCCL communicator, ss_encode_combine), each rank
then normalises the rows it received.  No other data-path collective exists.
This module holds the host-side mirror of that layout for the tests and the
bench (combine_layout == ss_combine_layout_for).

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


def combine_layout(n: int, world: int, combine_rows: int = 0) -> dict:
    """The block-cyclic row ownership of ss_encode_combine (include/semsplat_b200.h):
    block B = combine_rows (0 = one contiguous shard of ceil(n / world) rows),
    round q reduce-scatters rows [q*world*B, (q+1)*world*B) and rank r receives
    [q*world*B + r*B, +B).  Mirrors ss_combine_layout_for."""
    if world < 1:
        raise ValueError("world must be >= 1")
    shard = max((n + world - 1) // world, 1)
    block = min(combine_rows, shard) if combine_rows else shard
    rounds = max((n + world * block - 1) // (world * block), 1)
    return {"block_rows": block, "rounds": rounds, "rows_alloc": rounds * world * block,
            "rank_rows": rounds * block}


def rows_of(n: int, world: int, rank: int, combine_rows: int = 0):
    """Global table rows held by `rank` after the combine, in round order
    (rows >= n are padding)."""
    import numpy as np
    lay = combine_layout(n, world, combine_rows)
    b, r = lay["block_rows"], lay["rounds"]
    q = np.arange(r, dtype=np.int64)[:, None]
    i = np.arange(b, dtype=np.int64)[None, :]
    return (q * world * b + rank * b + i).reshape(-1)


def reduce_scatter_rounds(full, world: int, rank: int, combine_rows: int = 0, n: int | None = None,
                          group=None):
    """The combine's collective on host tensors, for backends without a
    reduce-scatter (gloo, used by the tests): per round an all_reduce of the
    round's rows, then this rank's block.  `full` holds rows_alloc rows of the
    layout for `n` table rows (first dim); returns this rank's rank_rows rows
    in round order.  The product issues the same rounds as ncclReduceScatter
    inside libsemsplat_b200 (ss_encode_combine)."""
    import torch
    import torch.distributed as dist
    lay = combine_layout(full.shape[0] if n is None else n, world, combine_rows)
    b = lay["block_rows"]
    if full.shape[0] != lay["rows_alloc"]:
        raise ValueError(f"expected {lay['rows_alloc']} accumulator rows, got {full.shape[0]}")
    out = []
    for q in range(lay["rounds"]):
        part = full[q * world * b:(q + 1) * world * b].clone()
        dist.all_reduce(part, group=group)
        out.append(part[rank * b:(rank + 1) * b])
    return torch.cat(out)


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


def sparse_combine_mirror(partials_sums, partials_totals, block: int):
    """Host mirror of ss_encode_combine's covered-row path (SS_OPT_COMBINE_SPARSE)
    for one round of world x block rows: covered flags (all-reduce max of
    total != 0), positions, each rank packs its covered rows per owner block
    into P-row segments (P = the largest owner's count), the reduce-scatter
    sums the packed buffers and hands segment k to rank k, which unpacks onto
    its block.  Returns, per rank, (summed rows [block, D], summed totals
    [block]) -- what the rank normalises; uncovered rows are zero."""
    import numpy as np

    world = len(partials_sums)
    d = partials_sums[0].shape[1]
    flags = np.zeros(world * block, bool)
    for t in partials_totals:
        flags |= t != 0
    pos = np.concatenate([[0], np.cumsum(flags)]).astype(np.int64)
    counts = [int(pos[(k + 1) * block] - pos[k * block]) for k in range(world)]
    P = max(counts) if counts else 0
    packed = []
    for s, t in zip(partials_sums, partials_totals):
        ps = np.zeros((world * P, d), s.dtype)
        pt = np.zeros(world * P, t.dtype)
        for i in np.nonzero(flags)[0]:
            k = i // block
            slot = k * P + (pos[i] - pos[k * block])
            ps[slot] = s[i]
            pt[slot] = t[i]
        packed.append((ps, pt))
    out = []
    for r in range(world):
        seg_s = sum(p[0][r * P:(r + 1) * P] for p in packed)
        seg_t = sum(p[1][r * P:(r + 1) * P] for p in packed)
        rows = np.zeros((block, d), partials_sums[0].dtype)
        tots = np.zeros(block, partials_totals[0].dtype)
        for k in range(block):
            i = r * block + k
            if flags[i]:
                j = pos[i] - pos[r * block]
                rows[k] = seg_s[j]
                tots[k] = seg_t[j]
        out.append((rows, tots))
    return out
