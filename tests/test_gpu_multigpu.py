"""GPU: the multi-GPU combine of the embedding pass.

* ss_encode_combine (combine_partials + finalize_into, pipeline.hpp:90-141)
  without a communicator and through the library's own NCCL communicator
  (one rank: ss_comm_init and ss_comm_init_all) returns exactly the rows of
  ss_encode_finalize, for contiguous shards and block-cyclic rounds.
* Two processes sharing GPU 0 each run the product's device encode on their
  round-robin share of the views, combine the partials over gloo on host
  copies in the library's block-cyclic rounds, normalise their rows on the
  device (ss_normalize_device) and together match the oracle.  (One GPU is
  available here; ranks whose kernels wait on one another are not stacked on
  it, so the NCCL reduce-scatter itself runs with one rank.)
"""
import os
import socket

import numpy as np
import pytest

from tests.test_gpu_parity import EMB_COS_TOL, EMB_REL_TOL, _bench_style, row_errors

pytestmark = pytest.mark.gpu


def _encode_into(ctx, wl, dim):
    ctx.set_scene(wl.scene.mean, wl.scene.scale, wl.scene.quat_xyzw, wl.scene.opacity)
    ctx.encode_begin(dim)
    ctx.encode_views(wl.cams, wl.masks)


@pytest.mark.parametrize("combine_rows", [0, 1000, 333])
def test_combine_without_communicator_equals_finalize(combine_rows):
    from paper_2505_08124_b200._lib import Context
    wl = _bench_style(4001, 4, 80, 64, 24, 64, seed=201)
    ctx = Context(0)
    ctx.set_combine_rows(combine_rows)
    _encode_into(ctx, wl, 64)
    whole_rows, whole_cov = ctx.encode_finalize()
    rows, cov, held = ctx.combine()
    keep = held < 4001
    assert np.array_equal(np.sort(held[keep]), np.arange(4001))
    assert rows[keep].tobytes() == whole_rows[held[keep]].tobytes()
    assert cov[keep].tobytes() == whole_cov[held[keep]].tobytes()
    assert not rows[~keep].any() and not cov[~keep].any()
    ctx.close()


@pytest.mark.parametrize("how,combine_rows,sparse", [("rank", 0, 0), ("rank", 777, 0), ("all", 0, 0), ("rank", 0, 2),
                                                     ("rank", 777, 2), ("all", 333, 2)])
def test_combine_through_nccl_one_rank(how, combine_rows, sparse):
    """The NCCL path of ss_encode_combine (grouped reduce-scatter rounds on the
    communicator's stream, normalisation overlapped on the context stream), and
    the covered-row path (SS_OPT_COMBINE_SPARSE = 2 forces it for one rank:
    covered flags, positions, per-owner packing and unpacking) -- both give the
    rows of ss_encode_finalize bit for bit."""
    from paper_2505_08124_b200._lib import Context
    wl = _bench_style(3001, 3, 72, 56, 20, 32, seed=202)
    ctx = Context(0)
    if how == "rank":
        ctx.comm_init(1, 0, Context.comm_unique_id())
    else:
        Context.comm_init_all([ctx])
    ctx.set_combine_rows(combine_rows)
    ctx.set_combine_sparse(sparse)
    _encode_into(ctx, wl, 32)
    whole_rows, whole_cov = ctx.encode_finalize()
    rows, cov, held = ctx.combine()
    keep = held < 3001
    assert rows[keep].tobytes() == whole_rows[held[keep]].tobytes()
    assert cov[keep].tobytes() == whole_cov[held[keep]].tobytes()
    ctx.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, combine_rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    from harness.workload import make_bench_workload
    from paper_2505_08124_b200._lib import Context
    from paper_2505_08124_b200.multigpu import combine_layout, reduce_scatter_rounds, rows_of, shard_views

    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, dim = 5003, 512
    wl = make_bench_workload(n_gaussians=n, n_views=7, width=96, height=72, masks_per_view=40, dim=dim, seed=203)
    mine = shard_views(7, world, rank)
    lay = combine_layout(n, world, combine_rows)
    dev = torch.device("cuda", 0)
    sums = torch.zeros((lay["rows_alloc"], dim), dtype=torch.float32, device=dev)
    totals = torch.zeros((lay["rows_alloc"],), dtype=torch.float32, device=dev)
    ctx = Context(0)
    ctx.set_scene(wl.scene.mean, wl.scene.scale, wl.scene.quat_xyzw, wl.scene.opacity)
    ctx.encode_begin(dim, sums.data_ptr(), totals.data_ptr())
    ctx.encode_views([wl.cams[v] for v in mine], [wl.masks[v] for v in mine])
    ctx.synchronize()
    # the combine rounds over gloo on host copies of the device partials
    sh_s = reduce_scatter_rounds(sums.cpu(), world, rank, combine_rows, n).to(dev).contiguous()
    sh_t = reduce_scatter_rounds(totals.cpu(), world, rank, combine_rows, n).to(dev).contiguous()
    out_r = torch.empty_like(sh_s)
    out_c = torch.empty_like(sh_t)
    ctx.normalize_device(sh_s.data_ptr(), sh_t.data_ptr(), sh_s.shape[0], dim, out_r.data_ptr(), out_c.data_ptr())
    ctx.synchronize()
    q.put((rank, rows_of(n, world, rank, combine_rows), out_r.cpu().numpy(), out_c.cpu().numpy()))
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("combine_rows", [0, 1024])
def test_two_processes_combine_product_partials(oracle, combine_rows):
    import multiprocessing as mp
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    port = _free_port()
    procs = [mctx.Process(target=_rank_main, args=(r, 2, port, combine_rows, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, dim = 5003, 512
    rows = np.zeros((n, dim), np.float32)
    cov = np.zeros(n, np.float32)
    seen = np.zeros(n, np.int64)
    for _, held, r, c in parts:
        keep = held < n
        rows[held[keep]] = r[keep]
        cov[held[keep]] = c[keep]
        seen[held[keep]] += 1
    assert (seen == 1).all()
    wl = _bench_style(n, 7, 96, 72, 40, dim, seed=203)
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, dim)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)
