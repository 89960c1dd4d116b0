"""CPU, world_size 2 over gloo: the multi-GPU host logic of bench.py / the
paper's Fig. 4 combine -- views sharded round-robin, per-rank partial sums, one
reduce-scatter of the N x D sums + N totals, per-shard finalize -- reproduces
the single-worker encode (the reference's worker-count invariance,
test_pipeline.cpp:312-317, 1e-5 relative).  Each rank's partial sums come from
the oracle (the device kernels run only on the GPU box)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, combine_rows):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    from oracle.bindings import Oracle
    from paper_2505_08124_b200.multigpu import combine_layout, reduce_scatter_rounds, rows_of, shard_views
    from harness.workload import make_bench_workload

    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = make_bench_workload(n_gaussians=1501, n_views=5, width=64, height=48, masks_per_view=12, dim=32, seed=3)
    O = Oracle()
    mine = shard_views(5, world, rank)
    cams = [wl.cams[v] for v in mine]
    masks = [wl.masks[v] for v in mine]
    s, t = O.encode_partial(wl.scene, cams, masks, 32, 0, len(mine))
    n = 1501
    lay = combine_layout(n, world, combine_rows)
    full_s = torch.zeros((lay["rows_alloc"], 32), dtype=torch.float64)
    full_t = torch.zeros((lay["rows_alloc"],), dtype=torch.float64)
    full_s[:n] = torch.from_numpy(s)
    full_t[:n] = torch.from_numpy(t)
    sh_s = reduce_scatter_rounds(full_s, world, rank, combine_rows, n)
    sh_t = reduce_scatter_rounds(full_t, world, rank, combine_rows, n)
    held = rows_of(n, world, rank, combine_rows)
    keep = held < n
    sh_s, sh_t, held = sh_s.numpy()[keep].copy(), sh_t.numpy()[keep].copy(), held[keep]
    rows = np.zeros((held.size, 32), np.float32)
    cov = np.zeros(held.size, np.float32)
    O.L.sso_finalize(sh_s.ctypes.data, sh_t.ctypes.data, held.size, 32, rows.ctypes.data, cov.ctypes.data)
    q.put((rank, held, rows, cov))
    dist.destroy_process_group()


@pytest.mark.parametrize("combine_rows", [0, 97])
def test_two_rank_combine_matches_single_worker(combine_rows):
    """Round-robin view shards, per-rank partials, the block-cyclic combine
    rounds of ss_encode_combine (contiguous shards, and 97-row blocks: eight
    rounds with a ragged last one), per-rank finalize == one worker."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, combine_rows)) for r in range(2)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 1501
    rows = np.zeros((n, 32), np.float32)
    cov = np.zeros(n, np.float32)
    seen = np.zeros(n, np.int64)
    for _, held, r, c in parts:
        rows[held] = r
        cov[held] = c
        seen[held] += 1
    assert (seen == 1).all()  # every table row is finalised by exactly one rank

    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle.bindings import Oracle
    from harness.workload import make_bench_workload
    wl = make_bench_workload(n_gaussians=1501, n_views=5, width=64, height=48, masks_per_view=12, dim=32, seed=3)
    er, ec = Oracle().encode(wl.scene, wl.cams, wl.masks, 32)
    assert np.array_equal(cov > 0, ec > 0)
    e, g = er.astype(np.float64), rows.astype(np.float64)
    den = np.sqrt((e ** 2).sum(1))
    rel = np.sqrt(((e - g) ** 2).sum(1)) / np.where(den > 0, den, 1)
    assert rel.max() <= 1e-5
    np.testing.assert_allclose(cov, ec, rtol=1e-6)


def _query_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    from oracle.bindings import Oracle
    from paper_2505_08124_b200.multigpu import rows_of, sharded_query_topk

    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(44)
    n, d = 3001, 32
    O = Oracle()
    raw = rng.uniform(-0.5, 0.5, (n, d)).astype(np.float32)
    raw[1500:1510] = raw[7]  # exact ties across the shard boundary
    unit = np.stack([O.normalized_copy(r) for r in raw])
    ids = rng.permutation(n).astype(np.uint32)
    queries = np.concatenate([raw[[7, 100]], rng.uniform(-0.5, 0.5, (4, d)).astype(np.float32)])
    held = rows_of(n, world, rank)
    held = held[held < n]

    def local(qs, k):  # this rank's rows (the GPU product uses Context.query_topk)
        return O.query_topk(ids[held], unit[held], qs, k)

    for k in (1, 12, 5000):
        mi, ms, mc = sharded_query_topk(local, queries, k)
        q.put((rank, k, mi, ms, mc))
    dist.destroy_process_group()


def test_two_rank_sharded_query_matches_single_store():
    """§8(e) query: per-rank top-k over row shards + all_gather + merge equals
    the single-store answer bit for bit (ids, sims, counts; k > count too)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_query_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(6)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle.bindings import Oracle
    rng = np.random.default_rng(44)
    n, d = 3001, 32
    O = Oracle()
    raw = rng.uniform(-0.5, 0.5, (n, d)).astype(np.float32)
    raw[1500:1510] = raw[7]
    unit = np.stack([O.normalized_copy(r) for r in raw])
    ids = rng.permutation(n).astype(np.uint32)
    queries = np.concatenate([raw[[7, 100]], rng.uniform(-0.5, 0.5, (4, d)).astype(np.float32)])
    for rank, k, mi, ms, mc in got:
        ei, es, ec = O.query_topk(ids, unit, queries, k)
        kk = min(k, n)
        assert np.array_equal(mc, ec), (rank, k)
        assert np.array_equal(mi[:, :kk], ei[:, :kk]), (rank, k)
        assert ms[:, :kk].tobytes() == es[:, :kk].tobytes(), (rank, k)


@pytest.mark.parametrize("world,block", [(2, 50), (3, 17), (8, 9)])
def test_sparse_combine_mirror_equals_dense(world, block):
    """The covered-row combine (SS_OPT_COMBINE_SPARSE) moves only rows some
    rank touched, packed per owner into equal segments; every rank must end up
    with exactly the dense reduce-scatter's rows of its block (float64 sums
    here, so the check is exact)."""
    from paper_2505_08124_b200.multigpu import sparse_combine_mirror
    rng = np.random.default_rng(world * 100 + block)
    n, d = world * block, 6
    sums, tots = [], []
    for _ in range(world):
        touched = rng.random(n) < 0.15
        s = np.where(touched[:, None], rng.standard_normal((n, d)), 0.0)
        t = np.where(touched, rng.uniform(0.1, 2.0, n), 0.0)
        sums.append(s)
        tots.append(t)
    dense_s = sum(sums)
    dense_t = sum(tots)
    out = sparse_combine_mirror(sums, tots, block)
    for r, (rs, rt) in enumerate(out):
        assert np.array_equal(rs, dense_s[r * block:(r + 1) * block])
        assert np.array_equal(rt, dense_t[r * block:(r + 1) * block])
