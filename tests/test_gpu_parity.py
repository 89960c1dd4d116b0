"""GPU parity: the sm_100a path through the C ABI against the oracle and the
reference's golden vectors.

Bars (BASELINE.json north_star): depth order, per-tile lists and per-pixel
contributor lists (ids, order, f32 weights) bit-exact; embeddings per-row
relative L2 <= 1e-4 and cosine >= 0.9999 with identical covered sets; query
top-k ids (and their fp32 similarities) exact.
"""
import numpy as np
import pytest

from tests.goldens import g_cams, g_masks, g_scene, golden
from tests.util import look_at, make_test_camera, plain_camera, random_scene, scene_ns

pytestmark = pytest.mark.gpu

EMB_REL_TOL = 1e-4    # per-row relative L2 (oracles.hpp:129-144 definition)
EMB_COS_TOL = 0.9999  # per covered row


def row_errors(got_rows, got_cov, exp_rows, exp_cov):
    cov_e = exp_cov > np.float32(1e-8)
    cov_g = got_cov > np.float32(1e-8)
    assert np.array_equal(cov_e, cov_g), "covered sets differ"
    e = exp_rows.astype(np.float64)
    g = got_rows.astype(np.float64)
    num = np.sqrt(((e - g) ** 2).sum(1))
    den = np.sqrt((e ** 2).sum(1))
    rel = np.where(den > 0, num / np.where(den > 0, den, 1), num)
    cos = (e * g).sum(1) / np.maximum(np.sqrt((e ** 2).sum(1) * (g ** 2).sum(1)), 1e-300)
    cos = np.where(cov_e, cos, 1.0)
    assert not got_rows[~cov_g].any(), "uncovered rows must be exactly zero"
    return float(rel.max(initial=0.0)), float(cos.min(initial=1.0))


def test_library_is_the_device_path(gpu_ctx):
    from paper_2505_08124_b200._lib import LIB_PATH
    import os
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert str(LIB_PATH) in maps


def test_projection_bitwise_vs_golden(gpu_ctx):
    z = golden("project")
    for i in range(int(z["n"])):
        s = g_scene(z, i)
        gpu_ctx.set_scene(s.mean, s.scale, s.quat_xyzw, s.opacity)
        got = gpu_ctx.project(g_cams(z, i)[0])
        exp = z[f"projected_{i}"]
        assert np.array_equal(got["visible"], exp["visible"])
        vis = exp["visible"] == 1
        for f in ("mu_x", "mu_y", "cov_xx", "cov_xy", "cov_yy", "depth"):
            assert got[f][vis].tobytes() == exp[f][vis].tobytes(), f"case {i} field {f}"


def _capture(ctx, s, cam, mode=0):
    ctx.set_scene(s.mean, s.scale, s.quat_xyzw, s.opacity)
    return ctx.raster_capture(cam, mode)


def _assert_capture_equal(got, exp, mode=0):
    assert got["entries"].shape == exp["entries"].shape
    assert np.array_equal(got["entries"]["pixel"], exp["entries"]["pixel"])
    assert np.array_equal(got["entries"]["gaussian_id"], exp["entries"]["gaussian_id"])
    assert got["entries"]["weight"].tobytes() == exp["entries"]["weight"].tobytes()
    assert got["per_pixel_total"].tobytes() == exp["per_pixel_total"].tobytes()
    if mode == 0:
        assert got["alpha"].tobytes() == exp["alpha"].tobytes()
    for k in ("splat_gid", "tile_offsets", "tile_splats"):
        if k in exp:
            assert np.array_equal(got[k], exp[k]), k


def test_raster_bitwise_vs_golden(gpu_ctx):
    z = golden("raster")
    for i in range(int(z["n"])):
        mode = int(z[f"mode_{i}"])
        got = _capture(gpu_ctx, g_scene(z, i), g_cams(z, i)[0], mode)
        exp = {"entries": z[f"entries_{i}"], "per_pixel_total": z[f"ppt_{i}"], "alpha": z[f"alpha_{i}"]}
        _assert_capture_equal(got, exp, mode)
        order = z[f"order_{i}"]
        assert np.array_equal(order[np.isin(order, got["splat_gid"])], got["splat_gid"])


@pytest.mark.parametrize("seed,n,w,h,dist,mode", [
    (1, 300, 64, 48, 7.0, 0), (2, 500, 100, 77, 6.0, 0), (3, 200, 17, 200, 8.0, 0), (4, 400, 90, 60, 7.0, 1),
    (5, 1000, 128, 128, 9.0, 0)])
def test_raster_bitwise_vs_oracle(gpu_ctx, oracle, seed, n, w, h, dist, mode):
    s = random_scene(n, seed)
    cam = make_test_camera(w, h, dist)
    got = _capture(gpu_ctx, s, cam, mode)
    exp = oracle.rasterize(s, cam, mode)
    _assert_capture_equal(got, exp, mode)


def test_depth_ties_break_by_id(gpu_ctx, oracle):
    """projection.hpp:59-64: equal depths fall back to id order."""
    s = random_scene(60, 9)
    s.mean[:, 2] = s.mean[0, 2]  # many identical depths under an axis-aligned camera
    cam = plain_camera(60.0, 60.0, 20.0, 20.0, 40, 40)
    s.mean[:, 2] += np.float32(5.0)
    got = _capture(gpu_ctx, s, cam)
    _assert_capture_equal(got, oracle.rasterize(s, cam))


def test_depth_order_exact_with_coarse_narrowed_keys(gpu_ctx, oracle):
    """A far outlier widens the depth range so the 32-bit narrowed sort keys
    collide across thousands of near-equal depths: the tie fixup must restore
    the exact (depth, id) order."""
    rng = np.random.default_rng(4)
    n = 3000
    mean = np.zeros((n, 3), np.float32)
    mean[:, 0] = rng.uniform(-1, 1, n)
    mean[:, 1] = rng.uniform(-1, 1, n)
    mean[:, 2] = (8.0 + rng.uniform(0, 1e-5, n)).astype(np.float32)
    mean[0] = [0.0, 0.0, 1.0e5]
    s = scene_ns(mean, np.full((n, 3), 0.05), np.tile([0, 0, 0, 1.0], (n, 1)), rng.uniform(0.1, 0.6, n))
    cam = plain_camera(40.0, 40.0, 24.0, 24.0, 48, 48)
    got = _capture(gpu_ctx, s, cam)
    _assert_capture_equal(got, oracle.rasterize(s, cam))


@pytest.mark.parametrize("n", [6000, 20000])
def test_oversized_tiles_sort_exactly(gpu_ctx, oracle, n):
    """Tiles whose lists exceed the shared-memory sort (4096 -> 512x32 class,
    16384 -> in-place bitonic class) keep the exact (depth, id) order."""
    rng = np.random.default_rng(n)
    mean = np.zeros((n, 3), np.float32)
    mean[:, 0] = rng.uniform(-0.2, 0.2, n)
    mean[:, 1] = rng.uniform(-0.2, 0.2, n)
    mean[:, 2] = rng.uniform(4.0, 6.0, n)
    mean[: n // 4, 2] = mean[0, 2]  # a block of exact depth ties
    s = scene_ns(mean, np.full((n, 3), 0.02), np.tile([0, 0, 0, 1.0], (n, 1)), rng.uniform(0.01, 0.05, n))
    cam = plain_camera(30.0, 30.0, 8.0, 8.0, 16, 16)
    got = _capture(gpu_ctx, s, cam)
    assert got["tile_offsets"][-1] == n  # one tile holds every splat
    _assert_capture_equal(got, oracle.rasterize(s, cam))


@pytest.mark.parametrize("seed,n,w,h,dist,scale", [
    (11, 50000, 1920, 1080, 9.0, 1.0),    # 13 chunks, 8160 tiles (4-warp scatter CTAs)
    (12, 30000, 640, 480, 7.0, 6.0),      # large boxes: hundreds of tiles per splat
    (13, 9000, 1152, 864, 8.0, 1.0),      # c4 geometry (8-warp scatter CTAs)
    (14, 4097, 64, 64, 7.0, 1.0)])        # one rank past a chunk
def test_direct_binning_equals_sort(gpu_ctx, oracle, seed, n, w, h, dist, scale):
    """SS_OPT_BIN_PATH: the count/scan/scatter binning gives the key sort's
    tile lists, ranges and contributor lists bit for bit."""
    s = random_scene(n, seed)
    s.scale[:] = (s.scale * np.float32(scale)).astype(np.float32)
    cam = make_test_camera(w, h, dist)
    try:
        gpu_ctx.set_bin_path(1)
        by_sort = _capture(gpu_ctx, s, cam)
        gpu_ctx.set_bin_path(2)
        direct = _capture(gpu_ctx, s, cam)
        gpu_ctx.set_bin_path(3)
        tile_sorted = _capture(gpu_ctx, s, cam)
    finally:
        gpu_ctx.set_bin_path(0)
    assert direct["tile_offsets"][-1] > 0
    _assert_capture_equal(direct, by_sort)
    _assert_capture_equal(tile_sorted, by_sort)
    if n <= 10000:
        _assert_capture_equal(direct, oracle.rasterize(s, cam))


def test_direct_binning_tile_limit(gpu_ctx, oracle):
    """Above 18000 tiles auto takes the key sort; forcing the direct path there
    is a contract error."""
    from paper_2505_08124_b200.errors import ContractError
    s = random_scene(3000, 15)
    cam = make_test_camera(3840, 2160, 8.0)
    auto = _capture(gpu_ctx, s, cam)
    try:
        gpu_ctx.set_bin_path(2)
        with pytest.raises(ContractError):
            _capture(gpu_ctx, s, cam)
    finally:
        gpu_ctx.set_bin_path(0)
    gpu_ctx.set_bin_path(1)
    try:
        _assert_capture_equal(auto, _capture(gpu_ctx, s, cam))
    finally:
        gpu_ctx.set_bin_path(0)


def test_empty_and_culled_scenes(gpu_ctx, oracle):
    cam = plain_camera(50, 50, 16, 16, 32, 32)
    behind = scene_ns([[0, 0, -1], [0, 0, 0.005]], [[0.1] * 3] * 2, [[0, 0, 0, 1]] * 2, [0.5, 0.5])
    got = _capture(gpu_ctx, behind, cam)
    assert got["entries"].shape[0] == 0 and got["splat_gid"].shape[0] == 0
    offscreen = scene_ns([[100, 0, 2]], [[0.1] * 3], [[0, 0, 0, 1]], [0.5])
    got = _capture(gpu_ctx, offscreen, cam)
    assert got["entries"].shape[0] == 0


def test_nan_scale_is_culled_like_the_reference(gpu_ctx, oracle):
    """A NaN covariance fails the det test silently and its box casts to
    INT_MIN (x86 cvttsd2si), so the splat is culled (rasterizer.hpp:66-71,171-179)."""
    s = scene_ns([[0, 0, 2], [0.1, 0, 2.5]], [[np.nan, 0.1, 0.1], [0.1, 0.1, 0.1]], [[0, 0, 0, 1]] * 2, [0.5, 0.7])
    cam = plain_camera(50, 50, 16, 16, 32, 32)
    got = _capture(gpu_ctx, s, cam)
    _assert_capture_equal(got, oracle.rasterize(s, cam))


def _encode(ctx, s, cams, masks, dim, mode=0):
    ctx.set_scene(s.mean, s.scale, s.quat_xyzw, s.opacity)
    ctx.encode_begin(dim)
    ctx.encode_views(cams, masks, mode)
    return ctx.encode_finalize()


def test_encode_fixtures_vs_reference_golden(gpu_ctx):
    z = golden("encode")
    for i in range(int(z["n"])):
        dim = z[f"clip_{i}"].shape[1]
        rows, cov = _encode(gpu_ctx, g_scene(z, i), g_cams(z, i), g_masks(z, i), dim)
        rel, cos = row_errors(rows, cov, z[f"rows_{i}"], z[f"coverage_{i}"])
        assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (i, rel, cos)
        cov_e = z[f"coverage_{i}"]
        np.testing.assert_allclose(cov, cov_e, rtol=1e-5)


def _bench_style(n, views, w, h, m, dim, seed):
    from harness.workload import make_bench_workload
    return make_bench_workload(n_gaussians=n, n_views=views, width=w, height=h, masks_per_view=m, dim=dim,
                               seed=seed, xy_extent=5.0)


@pytest.mark.parametrize("n,views,w,h,m,dim", [(2000, 3, 64, 48, 16, 512), (5000, 2, 96, 80, 70, 64),
                                               (3000, 2, 80, 64, 128, 32)])
def test_encode_bench_style_vs_oracle(gpu_ctx, oracle, n, views, w, h, m, dim):
    wl = _bench_style(n, views, w, h, m, dim, seed=n + m)
    rows, cov = _encode(gpu_ctx, wl.scene, wl.cams, wl.masks, dim)
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, dim)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)
    np.testing.assert_allclose(cov, ec, rtol=1e-5)


@pytest.mark.parametrize("m", [48, 64])  # 64: three views fill the 192 KB of staged CLIP half-rows
def test_group_contraction_d512(gpu_ctx, oracle, m):
    """D = 512 views with <= 64 masks are contracted in groups (auto: three at a
    time; the two-pass shared-memory group kernels), including a partial last
    group and a view with more masks that is contracted alone.  The per-row
    contraction order is the single-view one; with SS_OPT_DETERMINISTIC the
    per-(Gaussian, mask) scalars are exact fixed-point sums, so every CUDA-core
    configuration is bitwise identical; with the default f32 atomics (last-bit
    run-to-run differences) and on the tensor cores (split-fp16 operands)
    configurations agree to 1e-5 relative per row; each matches the oracle to
    the north-star tolerance."""
    wl = _bench_style(4000, 8, 80, 64, m, 512, seed=77)
    big = _bench_style(4000, 1, 80, 64, 100, 512, seed=78)
    cams = wl.cams[:5] + big.cams + wl.cams[5:]
    masks = wl.masks[:5] + big.masks + wl.masks[5:]
    out = {}
    try:
        for det in (1, 0):
            gpu_ctx.set_deterministic(det)
            for lanes, group, tc in [(4, 1, 0), (4, 0, 0), (4, 2, 0), (4, 3, 0), (1, 3, 0), (2, 0, 0), (4, 0, 1),
                                     (1, 2, 1)]:
                gpu_ctx.set_lanes(lanes)
                gpu_ctx.set_contract_group(group)
                gpu_ctx.set_contract_tc(tc)  # SS_OPT_CONTRACT_TC: groups on the tensor cores
                out[(lanes, group, tc, det)] = _encode(gpu_ctx, wl.scene, cams, masks, 512)
    finally:
        gpu_ctx.set_lanes(4)
        gpu_ctx.set_contract_group(0)
        gpu_ctx.set_contract_tc(0)
        gpu_ctx.set_deterministic(0)
    er, ec = oracle.encode(wl.scene, cams, masks, 512)
    ref_rows, ref_cov = out[(4, 1, 0, 1)]
    for key, (rows, cov) in out.items():
        if key[2] == 0 and key[3] == 1:
            assert np.array_equal(rows, ref_rows) and np.array_equal(cov, ref_cov), key
        rel, cos = row_errors(rows, cov, ref_rows, ref_cov)
        assert rel <= 1e-5, (key, rel)
        rel, cos = row_errors(rows, cov, er, ec)
        assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (key, rel, cos)


@pytest.mark.parametrize("lanes,group", [(1, 1), (3, 1), (4, 1), (4, 2), (4, 4), (1, 4), (3, 4), (6, 0), (5, 3)])
def test_encode_lane_count_does_not_change_results(gpu_ctx, oracle, lanes, group):
    """Views spread over 1..4 pipeline lanes (SS_OPT_LANES) and contracted in
    groups of 1..4 (SS_OPT_CONTRACT_GROUP) contract in view order; the result
    matches the oracle for every combination (7 views: partial last group)."""
    wl = _bench_style(3000, 7, 64, 64, 24, 64, seed=91)
    gpu_ctx.set_lanes(lanes)
    gpu_ctx.set_contract_group(group)
    try:
        rows, cov = _encode(gpu_ctx, wl.scene, wl.cams, wl.masks, 64)
    finally:
        gpu_ctx.set_lanes(4)
        gpu_ctx.set_contract_group(0)
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, 64)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (lanes, rel, cos)
    np.testing.assert_allclose(cov, ec, rtol=1e-5)


def test_encode_is_bitwise_deterministic(gpu_ctx, oracle):
    """pipeline.hpp:272-279: for a fixed worker count the table is bitwise
    identical run to run.  With SS_OPT_DETERMINISTIC the compositor adds exact
    f32 group sums into u64 fixed-point scalars (integer atomics: any arrival
    order gives the same bits) and the contraction runs in view order, so
    repeated runs -- and every lane count and contraction grouping -- give the
    same bits, which also match the oracle."""
    wl = _bench_style(4000, 7, 80, 64, 40, 512, seed=93)
    runs = []
    try:
        gpu_ctx.set_deterministic(1)
        for lanes, group in [(5, 0), (5, 0), (1, 1), (3, 3), (2, 2), (6, 0)]:
            gpu_ctx.set_lanes(lanes)
            gpu_ctx.set_contract_group(group)
            runs.append(((lanes, group), _encode(gpu_ctx, wl.scene, wl.cams, wl.masks, 512)))
    finally:
        gpu_ctx.set_lanes(4)
        gpu_ctx.set_contract_group(0)
        gpu_ctx.set_deterministic(0)
    (_, (rows0, cov0)) = runs[0]
    assert np.count_nonzero(cov0) > 100
    for key, (rows, cov) in runs[1:]:
        assert np.array_equal(rows, rows0) and np.array_equal(cov, cov0), key
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, 512)
    rel, cos = row_errors(rows0, cov0, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)


@pytest.mark.parametrize("prefix", [8, 48, 300])
def test_sort_prefix_resume_is_bitwise(gpu_ctx, oracle, prefix):
    """SS_OPT_SORT_PREFIX: tile lists ranked only over a prefix, the blocks
    that exhaust it resumed after the fixup sort.  Tiny prefixes force most
    blocks through the save / fixup / resume path; with fixed-point scalars
    the table is bitwise the one from full sorts, and matches the oracle."""
    wl = _bench_style(6000, 4, 96, 80, 40, 512, seed=121)
    out = {}
    try:
        gpu_ctx.set_deterministic(1)
        for pf in (0, prefix):
            gpu_ctx.set_sort_prefix(pf)
            out[pf] = _encode(gpu_ctx, wl.scene, wl.cams, wl.masks, 512)
    finally:
        gpu_ctx.set_sort_prefix(1024)
        gpu_ctx.set_deterministic(0)
    (r0, c0), (r1, c1) = out[0], out[prefix]
    assert np.count_nonzero(c0) > 100
    assert np.array_equal(r0, r1) and np.array_equal(c0, c1)
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, 512)
    rel, cos = row_errors(r1, c1, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)


def test_encode_falloff_mode_vs_oracle(gpu_ctx, oracle):
    wl = _bench_style(1500, 2, 64, 64, 20, 16, seed=77)
    rows, cov = _encode(gpu_ctx, wl.scene, wl.cams, wl.masks, 16, mode=1)
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, 16, mode=1)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL


def test_encode_finalize_sparse_equals_dense(gpu_ctx):
    """ss_encode_finalize_sparse (covered rows packed on the device, scattered
    by id into a zero table) gives the dense finalize_into bits, per chunk."""
    wl = _bench_style(5000, 3, 80, 64, 24, 512, seed=131)
    gpu_ctx.set_scene(wl.scene.mean, wl.scene.scale, wl.scene.quat_xyzw, wl.scene.opacity)
    gpu_ctx.encode_begin(512)
    gpu_ctx.encode_views(wl.cams, wl.masks, 0)
    rows, cov = gpu_ctx.encode_finalize()
    srows, scov, n_cov = gpu_ctx.encode_finalize_sparse()
    assert n_cov == int(np.count_nonzero(cov)) > 100
    assert np.array_equal(rows, srows) and np.array_equal(cov, scov)
    lo, hi = 1234, 4321
    crows, ccov, _ = gpu_ctx.encode_finalize_sparse(lo, hi)
    assert np.array_equal(crows, rows[lo:hi]) and np.array_equal(ccov, cov[lo:hi])


def test_encode_chunked_finalize_is_bitwise_chunk_invariant(gpu_ctx):
    """pipeline.hpp:276-279: the result does not depend on chunk_rows."""
    wl = _bench_style(1000, 2, 48, 48, 8, 32, seed=5)
    gpu_ctx.set_scene(wl.scene.mean, wl.scene.scale, wl.scene.quat_xyzw, wl.scene.opacity)
    gpu_ctx.encode_begin(32)
    gpu_ctx.encode_views(wl.cams, wl.masks)
    whole = gpu_ctx.encode_finalize()
    parts = [gpu_ctx.encode_finalize(lo, min(1000, lo + 237)) for lo in range(0, 1000, 237)]
    assert np.concatenate([p[0] for p in parts]).tobytes() == whole[0].tobytes()
    assert np.concatenate([p[1] for p in parts]).tobytes() == whole[1].tobytes()


def test_store_build_bitwise_vs_oracle(gpu_ctx, oracle):
    rng = np.random.default_rng(3)
    rows = rng.uniform(-1, 1, (300, 64)).astype(np.float32)
    cov = (rng.random(300) < 0.7).astype(np.float32) * 2.5
    cnt = gpu_ctx.store_build(rows, cov)
    ids, unit = gpu_ctx.store_fetch()
    exp_ids = np.flatnonzero(cov > 0).astype(np.uint32)
    assert cnt == exp_ids.shape[0] and np.array_equal(ids, exp_ids)
    for j, k in enumerate(exp_ids):
        assert unit[j].tobytes() == oracle.normalized_copy(rows[k]).tobytes()


@pytest.fixture
def query_path(gpu_ctx, request):
    gpu_ctx.set_query_path(request.param)
    yield request.param
    gpu_ctx.set_query_path(0)


@pytest.mark.parametrize("query_path", [1, 2], indirect=True)
def test_query_topk_vs_reference_golden(gpu_ctx, query_path):
    z = golden("query")
    gpu_ctx.store_set(z["ids"], z["rows"])
    ids, sims, cnt = gpu_ctx.query_topk(z["queries"], 37)
    assert np.array_equal(ids, z["topk_ids"])
    assert sims.tobytes() == z["topk_sims"].tobytes()
    for i in range(5):
        ti, ts = gpu_ctx.query_threshold(z["queries"][i], 0.05)
        assert np.array_equal(ti, z[f"thr_ids_{i}"]) and ts.tobytes() == z[f"thr_sims_{i}"].tobytes()


def test_query_edge_cases(gpu_ctx):
    from paper_2505_08124_b200 import NumericError
    ids = np.array([9, 3, 7], np.uint32)
    rows = np.array([[1, 0], [1, 0], [1, 0]], np.float32)
    gpu_ctx.store_set(ids, rows)
    i, s, c = gpu_ctx.query_topk(np.array([1.0, 0.0], np.float32), 3)
    assert list(i[0]) == [3, 7, 9]  # ties by ascending id (test_vecstore.cpp:172-183)
    i, s, c = gpu_ctx.query_topk(np.array([0.0, 2.0], np.float32), 5)
    assert int(c[0]) == 3  # k > count returns all
    with pytest.raises(NumericError):
        gpu_ctx.query_topk(np.array([0.0, 0.0], np.float32), 1)


@pytest.mark.parametrize("query_path", [1, 2], indirect=True)
def test_query_random_large_vs_oracle(gpu_ctx, oracle, query_path):
    rng = np.random.default_rng(11)
    raw = rng.uniform(-0.5, 0.5, (20000, 512)).astype(np.float32)
    cnt = gpu_ctx.store_build(raw, np.ones(20000, np.float32))
    ids, unit = gpu_ctx.store_fetch()
    q = rng.uniform(-0.5, 0.5, (70, 512)).astype(np.float32)
    gi, gs, gc = gpu_ctx.query_topk(q, 10)
    oi, os_, oc = oracle.query_topk(ids, unit, q, 10, threads=8)
    assert np.array_equal(gi, oi) and gs.tobytes() == os_.tobytes()


def _tc_vs_oracle(ctx, oracle, ids, unit, q, k):
    ctx.store_set(ids, unit)
    ctx.set_query_path(2)
    try:
        gi, gs, gc = ctx.query_topk(q, k)
    finally:
        ctx.set_query_path(0)
    oi, os_, oc = oracle.query_topk(ids, unit, q, k, threads=8)
    assert np.array_equal(gc, oc)
    assert np.array_equal(gi, oi)
    assert gs.tobytes() == os_.tobytes()


def _unit_rows(oracle, raw):
    return np.stack([oracle.normalized_copy(r) for r in raw]).astype(np.float32)


def test_query_tensor_core_chunked_ragged_vs_oracle(gpu_ctx, oracle):
    # > 1024 queries (two coarse-score passes), a row count that is not a
    # multiple of the 128-row tile nor of 8, and k at the device maximum
    rng = np.random.default_rng(21)
    raw = rng.standard_normal((5003, 128)).astype(np.float32)
    unit = _unit_rows(oracle, raw)
    ids = rng.permutation(1 << 20)[:5003].astype(np.uint32)
    q = rng.standard_normal((1100, 128)).astype(np.float32)
    _tc_vs_oracle(gpu_ctx, oracle, ids, unit, q, 64)


def test_query_tensor_core_duplicates_and_near_ties(gpu_ctx, oracle):
    # clusters of exact duplicates (ties by ascending id) and near-duplicates
    # closer than fp16 resolution: the coarse scores cannot order them, the
    # exact rescoring must
    rng = np.random.default_rng(22)
    base = rng.standard_normal((400, 256)).astype(np.float32)
    raw = np.repeat(base, 20, axis=0)
    raw[1::2] += rng.standard_normal((raw.shape[0] // 2, 256)).astype(np.float32) * 1e-4
    unit = _unit_rows(oracle, raw)
    ids = rng.permutation(raw.shape[0]).astype(np.uint32)
    q = np.concatenate([base[:40], rng.standard_normal((40, 256)).astype(np.float32)])
    _tc_vs_oracle(gpu_ctx, oracle, ids, unit, q, 25)


def test_query_tensor_core_candidate_overflow_falls_back_exactly(gpu_ctx, oracle):
    # 6000 identical rows: every row is a candidate (> the per-query cap), the
    # batch is answered by the exact scan and must still match
    rng = np.random.default_rng(23)
    raw = np.repeat(rng.standard_normal((1, 64)).astype(np.float32), 6000, axis=0)
    raw[::7] = rng.standard_normal((len(raw[::7]), 64)).astype(np.float32)
    unit = _unit_rows(oracle, raw)
    ids = np.arange(6000, dtype=np.uint32)[::-1].copy()
    q = np.concatenate([raw[:2], rng.standard_normal((3, 64)).astype(np.float32)])
    _tc_vs_oracle(gpu_ctx, oracle, ids, unit, q, 10)


@pytest.mark.parametrize("tau", [0.12, 0.18, 0.3])
def test_query_threshold_tensor_core_vs_oracle(gpu_ctx, oracle, tau):
    """Tensor-core threshold path (candidates >= tau - eps, exact rescoring)
    against the oracle restatement of query_threshold."""
    rng = np.random.default_rng(31)
    raw = rng.uniform(-0.5, 0.5, (30001, 128)).astype(np.float32)
    unit = _unit_rows(oracle, raw)
    ids = rng.permutation(1 << 22)[:30001].astype(np.uint32)
    gpu_ctx.store_set(ids, unit)
    gpu_ctx.set_query_path(2)
    try:
        for i in range(4):
            q = raw[i * 7] + rng.uniform(-0.2, 0.2, 128).astype(np.float32) if i < 2 else \
                rng.uniform(-0.5, 0.5, 128).astype(np.float32)
            gi, gs = gpu_ctx.query_threshold(q, tau)
            oi, os_ = oracle.query_threshold(ids, unit, q, tau)
            assert np.array_equal(gi, oi) and gs.tobytes() == os_.tobytes(), (i, len(gi), len(oi))
    finally:
        gpu_ctx.set_query_path(0)


def test_query_threshold_tensor_core_overflow_falls_back(gpu_ctx, oracle):
    """tau low enough that more rows qualify than the candidate cap: the exact
    scan answers, with the same result."""
    rng = np.random.default_rng(32)
    raw = rng.uniform(-0.5, 0.5, (20000, 64)).astype(np.float32)
    unit = _unit_rows(oracle, raw)
    ids = np.arange(20000, dtype=np.uint32)
    gpu_ctx.store_set(ids, unit)
    gpu_ctx.set_query_path(2)
    try:
        q = rng.uniform(-0.5, 0.5, 64).astype(np.float32)
        gi, gs = gpu_ctx.query_threshold(q, -0.05)
        oi, os_ = oracle.query_threshold(ids, unit, q, -0.05)
        assert len(oi) > 4096
        assert np.array_equal(gi, oi) and gs.tobytes() == os_.tobytes()
    finally:
        gpu_ctx.set_query_path(0)


def test_render_bitwise_vs_reference_golden(gpu_ctx):
    """rasterize (rasterizer.hpp:261-264): image, alpha, WeightMap and totals
    bit-identical to the reference build's RenderResult (golden_render.npz)."""
    z = golden("render")
    for i in range(int(z["n"])):
        s = g_scene(z, i)
        mode = int(z[f"mode_{i}"])
        gpu_ctx.set_scene(s.mean, s.scale, s.quat_xyzw, s.opacity)
        gpu_ctx.set_scene_color(z[f"color_{i}"])
        got = gpu_ctx.render(g_cams(z, i)[0], mode)
        assert got["image"].tobytes() == z[f"image_{i}"].tobytes(), i
        exp = {"entries": z[f"entries_{i}"], "per_pixel_total": z[f"ppt_{i}"], "alpha": z[f"alpha_{i}"]}
        _assert_capture_equal(got, exp, mode)


@pytest.mark.parametrize("seed,n,w,h,dist,mode", [(21, 600, 72, 60, 7.0, 0), (22, 800, 120, 90, 8.0, 1)])
def test_render_bitwise_vs_reference_live(gpu_ctx, ref, seed, n, w, h, dist, mode):
    s = random_scene(n, seed)
    cam = make_test_camera(w, h, dist)
    gpu_ctx.set_scene(s.mean, s.scale, s.quat_xyzw, s.opacity)
    gpu_ctx.set_scene_color(s.color)
    got = gpu_ctx.render(cam, mode)
    exp = ref.rasterize(s, cam, mode, full_render=True)
    assert got["image"].tobytes() == exp["image"].tobytes()
    _assert_capture_equal(got, exp, mode)


def test_render_requires_colors(gpu_ctx):
    from paper_2505_08124_b200 import ContractError
    s = random_scene(50, 23)
    gpu_ctx.set_scene(s.mean, s.scale, s.quat_xyzw, s.opacity)
    with pytest.raises(ContractError):
        gpu_ctx.render(make_test_camera(32, 32, 7.0))


def test_render_through_the_reference_shaped_api(gpu_ctx, ref):
    """semsplat.rasterize (the Python mirror of rasterizer.hpp:261) returns a
    RenderResult equal to the reference's."""
    from paper_2505_08124_b200.semsplat import GaussianScene, rasterize
    s = random_scene(500, 24)
    scene = GaussianScene(s.mean, s.scale, s.quat_xyzw, s.opacity, s.color)
    cam = make_test_camera(70, 50, 7.5)
    r = rasterize(scene, cam)
    exp = ref.rasterize(s, cam, 0, full_render=True)
    assert r.image.tobytes() == exp["image"].tobytes()
    assert r.alpha.tobytes() == exp["alpha"].tobytes()
    assert r.weights.entries.tobytes() == exp["entries"].tobytes()


def test_query_topk_k_above_64_vs_oracle(gpu_ctx, oracle):
    """k beyond the top-k kernels' 64: full exact sort (vecstore.hpp:121-132)."""
    rng = np.random.default_rng(41)
    raw = rng.uniform(-0.5, 0.5, (6000, 64)).astype(np.float32)
    unit = _unit_rows(oracle, raw)
    ids = rng.permutation(6000).astype(np.uint32)
    q = rng.uniform(-0.5, 0.5, (3, 64)).astype(np.float32)
    gpu_ctx.store_set(ids, unit)
    for k in (65, 500, 7000):
        gi, gs, gc = gpu_ctx.query_topk(q, k)
        oi, os_, oc = oracle.query_topk(ids, unit, q, k)
        kk = min(k, 6000)
        assert np.array_equal(gc, oc)
        assert np.array_equal(gi[:, :kk], oi[:, :kk]) and gs[:, :kk].tobytes() == os_[:, :kk].tobytes()


@pytest.mark.parametrize("n,dim,nl", [(3000, 512, 20), (1500, 64, 70), (700, 32, 1)])
def test_assign_classes_bitwise_vs_reference(gpu_ctx, ref, n, dim, nl):
    """eval.hpp:122-158: sequential f64 cosines, arg max, ties to the lowest id,
    uncovered rows kUnlabeled -- identical to the reference."""
    rng = np.random.default_rng(n + nl)
    rows = rng.standard_normal((n, dim)).astype(np.float32)
    cov = (rng.random(n) < 0.8).astype(np.float32) * rng.uniform(0.01, 3.0, n).astype(np.float32)
    rows[5] = 0.0                                        # zero row: cos = -1 for every label
    ids = rng.permutation(1000)[:nl].astype(np.int32) - 500
    vecs = rng.standard_normal((nl, dim)).astype(np.float32)
    if nl > 3:
        vecs[2] = vecs[1]                                # exact tie: the lower id wins
    got = gpu_ctx.assign_classes(rows, cov, ids, vecs)
    exp = ref.assign_classes(rows, cov, ids, vecs)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("workers,contiguous", [(1, False), (2, False), (3, True)])
def test_encode_scene_api_vs_reference(gpu_ctx, ref, tmp_path, workers, contiguous):
    """semsplat.encode_scene (pipeline.hpp:280-470 mirror) on a reference-written
    fixture: table within tolerance, identical covered set, and the per-worker
    masked-weight entry counts summing to the reference's."""
    from paper_2505_08124_b200 import formats
    from paper_2505_08124_b200.semsplat import EncodeOptions, EncodeStats, GaussianScene, encode_scene
    mp = ref.write_fixture(str(tmp_path / "fx"), objects=3, per_object=15, views=5, resolution=40, mask_scale=1,
                           dim=24, seed=12)
    man = formats.load_manifest(mp)
    scene = GaussianScene.load(man.resolve("scene.ply"))
    stats = EncodeStats()
    table = encode_scene(scene, man, workers, 11, EncodeOptions(contiguous_batching=contiguous), stats)
    er, ec, rstats = ref.encode(scene, mp, workers, 11, 0, contiguous)
    rel, cos = row_errors(table.embeddings, table.coverage, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL
    assert np.array_equal(table.coverage > np.float32(1e-8), ec > np.float32(1e-8))
    assert sum(stats.worker_images) == 5 and len(stats.worker_entries) == workers
    assert sum(stats.worker_entries) == int(rstats[2])



def test_fp64_probe_rate_is_plausible(gpu_ctx):
    """ss_probe_fp64_rate (the compositor's fp64 roofline denominator): a B200
    runs 64 fp64 lanes per SM per clock, 148 SMs at up to ~2 GHz."""
    rate = gpu_ctx.probe_fp64_rate()
    assert 5e12 < rate < 2.2e13, rate


@pytest.mark.parametrize("bin_path", [0, 1])
def test_tile_list_overflow_reruns_exactly(oracle, bin_path):
    """Views whose tile lists exceed the list buffer (it starts at max(4N, 2^20)
    entries) are re-run with a larger one: captures and embeddings stay exact."""
    from paper_2505_08124_b200 import _lib
    s = random_scene(30000, 31)
    s.scale[:] = (s.scale * np.float32(4.0)).astype(np.float32)  # boxes of most of the view
    cam = make_test_camera(128, 128, 6.0)
    ctx = _lib.Context(0)  # fresh: the list buffer has its initial size
    ctx.set_bin_path(bin_path)
    got = _capture(ctx, s, cam)
    assert got["tile_offsets"][-1] > (1 << 20)
    _assert_capture_equal(got, oracle.rasterize(s, cam))
    wl = _bench_style(30000, 3, 96, 96, 8, 16, seed=33)
    wl.scene.scale[:] = (wl.scene.scale * np.float32(6.0)).astype(np.float32)
    ctx2 = _lib.Context(0)
    ctx2.set_bin_path(bin_path)
    rows, cov = _encode(ctx2, wl.scene, wl.cams, wl.masks, 16)
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, 16)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)


@pytest.mark.parametrize("lanes,group", [(5, 0), (1, 0), (4, 2)])
def test_encode_views_without_masks_interleaved(gpu_ctx, oracle, lanes, group):
    """Views with no masks contribute nothing and take no contraction; mixed
    into groups of D = 512 views they must not disturb the grouping or the
    per-row order (pipeline.hpp:320-350 skips them the same way)."""
    wl = _bench_style(3000, 5, 80, 64, 48, 512, seed=81)
    wl0 = _bench_style(3000, 3, 80, 64, 0, 512, seed=82)
    cams = [wl.cams[0], wl0.cams[0], wl.cams[1], wl.cams[2], wl0.cams[1], wl0.cams[2], wl.cams[3], wl.cams[4]]
    masks = [wl.masks[0], wl0.masks[0], wl.masks[1], wl.masks[2], wl0.masks[1], wl0.masks[2], wl.masks[3],
             wl.masks[4]]
    try:
        gpu_ctx.set_lanes(lanes)
        gpu_ctx.set_contract_group(group)
        rows, cov = _encode(gpu_ctx, wl.scene, cams, masks, 512)
    finally:
        gpu_ctx.set_lanes(5)
        gpu_ctx.set_contract_group(0)
    er, ec = oracle.encode(wl.scene, cams, masks, 512)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)


def test_failed_encode_leaves_no_stale_weights(gpu_ctx, oracle):
    """A batch that fails on view 2 (bad RLE length: FormatError, providers.hpp:97-107)
    after views 0 and 1 were composited into an open contraction group must
    not leak their per-(Gaussian, mask) scalars into the next encode, even when
    that encode has a different mask count."""
    from paper_2505_08124_b200 import FormatError
    wl = _bench_style(3000, 4, 80, 64, 40, 512, seed=101)
    bad = list(wl.masks)
    n, w, h, runs, offs, clip = bad[2]
    runs = runs.copy()
    runs[0] += 1
    bad[2] = (n, w, h, runs, offs, clip)
    gpu_ctx.set_scene(wl.scene.mean, wl.scene.scale, wl.scene.quat_xyzw, wl.scene.opacity)
    gpu_ctx.encode_begin(512)
    with pytest.raises(FormatError):
        gpu_ctx.encode_views(wl.cams, bad)
    good = _bench_style(3000, 3, 80, 64, 24, 512, seed=102)
    good.scene = wl.scene
    rows, cov = _encode(gpu_ctx, wl.scene, good.cams, good.masks, 512)
    er, ec = oracle.encode(wl.scene, good.cams, good.masks, 512)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)


def _singular_scene():
    """Rank-one, huge (1e7) Gaussians rotated off the image axes: after
    projection cov_xx * cov_yy - cov_xy^2 rounds below 1e-12 (rasterizer.hpp:66-69).
    Four of them; 10 has the smallest id but the first in depth order is 120
    (tied in depth with 250, so the id breaks the tie)."""
    s = random_scene(300, 41)
    c, sn = np.float32(np.cos(np.pi / 8)), np.float32(np.sin(np.pi / 8))
    for gid, z in [(10, 1.0), (250, -2.0), (120, -2.0), (77, 2.5)]:
        s.scale[gid] = [1e7, 1e-3, 1e-3]
        s.quat_xyzw[gid] = [0, 0, sn, c]
        s.mean[gid] = [0.1, 0.2, z]
    return s


def test_singular_covariance_names_first_in_depth_order(gpu_ctx, ref):
    """NumericError from conic_of names the first singular projection in depth
    order (rasterizer.hpp:66-69 inside the depth-sorted loop :187-191), as
    the reference build does; the encode path wraps it as the reference's
    per-image DataError (pipeline.hpp:350-351)."""
    from paper_2505_08124_b200 import DataError, NumericError
    from oracle.bindings import RefError
    s = _singular_scene()
    cam = make_test_camera(64, 48, 7.0, image_id=5)
    with pytest.raises(RefError) as er:
        ref.rasterize(s, cam)
    assert "gaussian 120" in str(er.value)
    gpu_ctx.set_scene(s.mean, s.scale, s.quat_xyzw, s.opacity)
    with pytest.raises(NumericError) as eg:
        gpu_ctx.raster_capture(cam, 0)
    assert str(eg.value).endswith("singular screen covariance for gaussian 120"), str(eg.value)
    from tests.util import rect_mask_runs
    runs, _ = rect_mask_runs(64, 48, [(3, 4, 40, 30)])
    masks = [(1, 64, 48, runs.astype(np.uint32), np.array([0, len(runs)], np.uint64),
              np.ones((1, 8), np.float32))]
    gpu_ctx.encode_begin(8)
    with pytest.raises(DataError) as ed:
        gpu_ctx.encode_views([cam], masks)
    assert str(ed.value).endswith("image 5: singular screen covariance for gaussian 120"), str(ed.value)


@pytest.mark.parametrize("m,dim", [(200, 512), (129, 64), (300, 16)])
def test_encode_more_than_128_masks_vs_oracle(gpu_ctx, oracle, m, dim):
    """Views with more SAM masks than one compositor pass holds (providers.hpp:135
    reads any u32 count; pipeline.hpp:323-336 loops over all of them): 128-mask
    windows, each a compositor pass, then the general contraction."""
    wl = _bench_style(3000, 3, 96, 72, m, dim, seed=m + dim)
    rows, cov = _encode(gpu_ctx, wl.scene, wl.cams, wl.masks, dim)
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, dim)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)
    np.testing.assert_allclose(cov, ec, rtol=1e-5)


@pytest.mark.parametrize("algo", [0, 1, 2])
@pytest.mark.parametrize("mode", [0, 1])
def test_compositor_schedules_match_oracle(gpu_ctx, oracle, mode, algo):
    """Every SS_OPT_RASTER schedule (0 staged evaluation, 1 CTA per tile, 2
    work-stealing warps -- the default): contributor lists bitwise and the
    encode within tolerance.  The work counters reset themselves, so a second
    capture on the same lane must match too."""
    s = random_scene(1200, 61)
    cam = make_test_camera(120, 90, 8.0)
    wl = _bench_style(3000, 3, 80, 64, 48, 512, seed=62)
    try:
        gpu_ctx.set_raster_algo(algo)
        got = _capture(gpu_ctx, s, cam, mode)
        again = _capture(gpu_ctx, s, cam, mode)
        rows, cov = _encode(gpu_ctx, wl.scene, wl.cams, wl.masks, 512, mode)
    finally:
        gpu_ctx.set_raster_algo(2)
    _assert_capture_equal(again, got, mode)
    _assert_capture_equal(got, oracle.rasterize(s, cam, mode), mode)
    er, ec = oracle.encode(wl.scene, wl.cams, wl.masks, 512, mode=mode)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)


def test_query_tensor_core_non_unit_store_vs_oracle(gpu_ctx, oracle):
    """The reference's VectorStore does not enforce unit rows (vecstore.hpp:61);
    ss_store_set bounds the row norms and widens the tensor-core margin with
    them, so non-unit stores stay exact on the tensor-core path, and stores
    whose norms could overflow fp16 are answered by the exact scan."""
    rng = np.random.default_rng(31)
    raw = rng.standard_normal((6000, 128)).astype(np.float32)
    unit = _unit_rows(oracle, raw)
    scale = rng.uniform(0.2, 40.0, (6000, 1)).astype(np.float32)
    rows = (unit * scale).astype(np.float32)
    ids = rng.permutation(6000).astype(np.uint32)
    q = rng.standard_normal((50, 128)).astype(np.float32)
    before = gpu_ctx.query_stats()
    _tc_vs_oracle(gpu_ctx, oracle, ids, rows, q, 10)
    after = gpu_ctx.query_stats()
    # answered on the tensor cores, no fallback
    assert after["tc_queries"] - before["tc_queries"] == 50
    assert after["exact_fallbacks"] == before["exact_fallbacks"]
    rows[17] *= 1.0e5  # beyond the fp16-safe bound: the exact scan answers
    _tc_vs_oracle(gpu_ctx, oracle, ids, rows, q, 10)
    assert gpu_ctx.query_stats()["tc_queries"] == after["tc_queries"]


@pytest.mark.parametrize("cell", [0.5, 1.0, 0.37, 1e-9])
def test_partition_store_vs_reference(gpu_ctx, ref, cell):
    """vecstore.hpp:169-213 partition_store on the device: cells, bounds, per-cell
    ids / rows / order identical to the reference build -- means on exact cell
    boundaries (half-open intervals), a NaN mean (skipped by the bbox, cell
    INT_MIN), and a cell size whose indices overflow int32 (x86 INT_MIN)."""
    from paper_2505_08124_b200 import semsplat
    rng = np.random.default_rng(int(cell * 1000) + 3)
    n, dim = 4000, 24
    ids = rng.permutation(1 << 20)[:n].astype(np.uint32)
    rows = rng.standard_normal((n, dim)).astype(np.float32)
    means = np.stack([np.floor(rng.uniform(-12, 12, n)) * 0.25, rng.uniform(-3, 3, n),
                      np.where(np.arange(n) % 7 == 0, 1.0, rng.uniform(0, 2, n))], 1).astype(np.float32)
    means[11, 1] = np.nan
    store = semsplat.VectorStore.from_unit_rows(ids, rows)
    snaps = semsplat.partition_store(store, means, cell)
    rc, rb, ro, rids, rrows = ref.partition_store(ids, rows, means, cell)
    assert len(snaps) == rc.shape[0]
    for c, sn in enumerate(snaps):
        assert sn.cell == tuple(int(v) for v in rc[c])
        assert sn.bounds_min.tobytes() == rb[c, :3].tobytes() and sn.bounds_max.tobytes() == rb[c, 3:].tobytes()
        lo, hi = int(ro[c]), int(ro[c + 1])
        assert np.array_equal(sn.ids, rids[lo:hi])
        assert sn.rows.tobytes() == rrows[lo:hi].tobytes()
    with pytest.raises(Exception):
        semsplat.partition_store(store, means, 0.0)


@pytest.mark.parametrize("lanes", [5, 2])
def test_encode_mixed_global_fallback_views_multilane(gpu_ctx, oracle, lanes):
    """A batch mixing views whose tile sort must fall back to the global depth
    sort (a tile holding thousands of exact depth ties, more than one bucket of
    the per-tile sort takes: bin_fallback 2, the view is re-run on the global
    path) with ordinary views, across several pipeline lanes: the fallback
    views are re-run while the others' results stand, and the table matches
    the oracle."""
    from harness.workload import rect_masks, synth_embedding
    rng = np.random.default_rng(91)
    n = 6000
    mean = np.zeros((n, 3), np.float32)
    mean[:2000, :2] = rng.uniform(-0.05, 0.05, (2000, 2))
    mean[:2000, 2] = 5.0  # exact depth ties under an axis-aligned camera
    mean[2000:, :2] = rng.uniform(-2.0, 2.0, (4000, 2))
    mean[2000:, 2] = rng.uniform(4.0, 6.0, 4000)
    s = scene_ns(mean, np.full((n, 3), 0.03), np.tile([0, 0, 0, 1.0], (n, 1)), rng.uniform(0.05, 0.4, n))
    cams, masks = [], []
    # principal points: the tie cluster on screen (fallback) or pushed off it (ordinary view)
    for i, (cx, cy) in enumerate([(24, 24), (-200, 24), (30, 20), (24, -300), (18, 28), (-150, -150), (26, 26)]):
        cams.append(plain_camera(60.0, 60.0, float(cx), float(cy), 48, 48, image_id=i))
        runs, offs = rect_masks(500 + i, 48, 48, 6)
        clip = np.stack([synth_embedding(f"fallback_{i}_{j}", 16) for j in range(6)])
        masks.append((6, 48, 48, runs, offs, clip))
    try:
        gpu_ctx.set_lanes(lanes)
        rows, cov = _encode(gpu_ctx, s, cams, masks, 16)
    finally:
        gpu_ctx.set_lanes(4)
    er, ec = oracle.encode(s, cams, masks, 16)
    rel, cos = row_errors(rows, cov, er, ec)
    assert rel <= EMB_REL_TOL and cos >= EMB_COS_TOL, (rel, cos)
    assert np.array_equal(cov > 0, ec > 0)
