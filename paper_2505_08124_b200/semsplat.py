"""Host-side mirror of the reference's C++ API for the embedding path.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/semsplat/*.hpp, so a caller (and the parity
tests) read like the reference's own code.  Every compute call goes to the
sm_100a kernels in libsemsplat_b200.so through the C ABI; this module only
moves data and maps status codes to the reference's exception classes.

  encode_scene            pipeline.hpp:280-470
  rasterize_weights_only  rasterizer.hpp:268-271
  project (batch of project_gaussian)  projection.hpp:33-55
  depth_sort order        projection.hpp:59-64 (as the capture's splat list)
  camera_scaled_to        pipeline.hpp:196-207
  build_store             vecstore.hpp:88-103
  query_topk              vecstore.hpp:121-132
  query_threshold         vecstore.hpp:135-146
"""
from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import formats
from ._lib import Context
from .errors import ContractError, DataError, DeviceError, PipelineError, SemsplatError  # noqa: F401
from .formats import CameraPose, DatasetManifest  # noqa: F401

K_COVERAGE_EPSILON = 1e-8  # pipeline.hpp:23
ALPHA_COMPOSITED, FALLOFF_ONLY = 0, 1  # WeightMode, rasterizer.hpp:33-36


@dataclass
class GaussianScene:
    """GaussianScene (scene.hpp:54-76) as SoA arrays; ids are 0..N-1."""
    mean: np.ndarray       # N x 3 f32
    scale: np.ndarray      # N x 3 f32 (activated std devs)
    quat_xyzw: np.ndarray  # N x 4 f32 (Eigen coeffs order)
    opacity: np.ndarray    # N f32
    color: np.ndarray | None = None

    def __len__(self) -> int:
        return int(self.opacity.shape[0])

    @staticmethod
    def load(path: str) -> "GaussianScene":
        return GaussianScene(*formats.load_scene_arrays(path))


@dataclass
class WeightMap:
    """WeightMap (rasterizer.hpp:48-53)."""
    image_id: int
    width: int
    height: int
    entries: np.ndarray         # structured (gaussian_id u4, pixel u4, weight f4), (pixel, rank) order
    per_pixel_total: np.ndarray


@dataclass
class RenderResult:
    """RenderResult (rasterizer.hpp:55-59): RGB image [H, W, 3] (black where the
    total weight is <= kRenderTotalEps), WeightMap and per-pixel alpha."""
    image: np.ndarray
    weights: WeightMap
    alpha: np.ndarray


@dataclass
class EmbeddingTable:
    """EmbeddingTable (pipeline.hpp:103-116)."""
    embeddings: np.ndarray  # N x D f32
    coverage: np.ndarray    # N f32

    @property
    def gaussian_count(self) -> int:
        return int(self.coverage.shape[0])

    @property
    def dim(self) -> int:
        return int(self.embeddings.shape[1])

    def covered(self, k=None):
        c = self.coverage > np.float32(K_COVERAGE_EPSILON)
        return c if k is None else bool(c[k])


@dataclass
class EncodeOptions:
    """EncodeOptions (pipeline.hpp:176-185); spill fields are accepted and
    ignored (device memory holds every partial: SURVEY.md 2.3)."""
    mode: int = ALPHA_COMPOSITED
    contiguous_batching: bool = False
    spill_memory_ceiling: int = 0
    spill_dir: str = ""


@dataclass
class EncodeStats:
    """EncodeStats (pipeline.hpp:187-193)."""
    phase1_seconds: float = 0.0
    phase2_seconds: float = 0.0
    worker_seconds: list = field(default_factory=list)
    worker_images: list = field(default_factory=list)
    worker_entries: list = field(default_factory=list)


_ctx_lock = threading.Lock()
_contexts: dict = {}


def device_context(device: int = 0) -> Context:
    """The process-wide context of one device (created on first use)."""
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def _bind_scene(ctx: Context, scene: GaussianScene) -> None:
    """Upload the scene for this call (N x 48 B); no identity caching, since
    arrays may be mutated in place between calls."""
    ctx.set_scene(scene.mean, scene.scale, scene.quat_xyzw, scene.opacity)


def camera_scaled_to(cam: CameraPose, width: int, height: int) -> CameraPose:
    """pipeline.hpp:196-207"""
    sx = float(width) / cam.width
    sy = float(height) / cam.height
    return replace(cam, fx=cam.fx * sx, cx=cam.cx * sx, fy=cam.fy * sy, cy=cam.cy * sy, width=int(width),
                   height=int(height))


def project(scene: GaussianScene, cam: CameraPose, device: int = 0) -> np.ndarray:
    """project_gaussian for every Gaussian (projection.hpp:33-55); structured
    array with gaussian_id, visible, mu_x, mu_y, cov_xx, cov_xy, cov_yy, depth."""
    ctx = device_context(device)
    _bind_scene(ctx, scene)
    return ctx.project(cam)


def rasterize_weights_only(scene: GaussianScene, cam: CameraPose, mode: int = ALPHA_COMPOSITED,
                           device: int = 0, with_binning: bool = False):
    """rasterizer.hpp:268-271.  Entries come back in (pixel, front-to-back
    rank) order.  with_binning=True also returns the depth-ordered splat list
    and the per-tile splat lists (rasterizer.hpp:183-194) for parity checks."""
    ctx = device_context(device)
    _bind_scene(ctx, scene)
    cap = ctx.raster_capture(cam, mode)
    wm = WeightMap(int(cam.image_id), int(cam.width), int(cam.height), cap["entries"], cap["per_pixel_total"])
    return (wm, cap) if with_binning else wm


def rasterize(scene: GaussianScene, cam: CameraPose, mode: int = ALPHA_COMPOSITED, device: int = 0) -> RenderResult:
    """rasterizer.hpp:261-264 on the device; needs scene.color (N x 3)."""
    if scene.color is None:
        raise ContractError("rasterize: the scene has no colors")
    ctx = device_context(device)
    _bind_scene(ctx, scene)
    ctx.set_scene_color(scene.color)
    r = ctx.render(cam, mode)
    wm = WeightMap(int(cam.image_id), int(cam.width), int(cam.height), r["entries"], r["per_pixel_total"])
    return RenderResult(r["image"], wm, r["alpha"])


def encode_scene(scene: GaussianScene, manifest: DatasetManifest, workers: int, chunk_rows: int,
                 options: EncodeOptions | None = None, stats: EncodeStats | None = None,
                 device: int = 0) -> EmbeddingTable:
    """pipeline.hpp:280-470 on the device.

    Views are assigned to `workers` logical workers exactly as the reference
    does (round-robin by manifest index, or contiguous blocks); on this host
    all workers share the single device context, so the per-worker partials
    are one fp32 accumulator (results agree across worker counts to fp32
    rounding, the reference's own cross-worker contract being 1e-5).
    chunk_rows bounds the rows normalised and copied back per finalize call.
    """
    options = options or EncodeOptions()
    if workers < 1:
        raise ContractError("encode_scene: workers must be >= 1")
    if manifest.raster_width == 0 or manifest.raster_height == 0:
        raise DataError("encode_scene: manifest has no raster resolution")
    cameras = formats.load_cameras(manifest.resolve(manifest.camera_file))
    by_id = {c.image_id: c for c in cameras}
    for e in manifest.images:
        if e.camera_id not in by_id:
            raise DataError(f"image {e.image_id}: no camera with id {e.camera_id}")

    ctx = device_context(device)
    _bind_scene(ctx, scene)
    dim = manifest.embedding_dim
    n_img = len(manifest.images)
    block = (n_img + workers - 1) // workers if n_img else 1
    t1 = time.perf_counter()
    ctx.encode_begin(dim)
    worker_images = [0] * workers
    worker_seconds = [0.0] * workers
    worker_entries = [0] * workers
    failures = [""] * workers
    status = ["pending"] * workers
    for rank in range(workers):
        t0 = time.perf_counter()
        # a worker's views go to the device as one batch (they overlap in the
        # device's pipeline lanes); host-side decoding errors stop the worker
        cams, sets, ids = [], [], []
        for idx, entry in enumerate(manifest.images):
            mine = (idx // block == rank) if options.contiguous_batching else (idx % workers == rank)
            if not mine:
                continue
            try:
                cam = camera_scaled_to(by_id[entry.camera_id], manifest.raster_width, manifest.raster_height)
                mr = formats.load_maskset_runs(manifest.resolve(entry.mask_path), entry.image_id)
                if mr.width != manifest.mask_width or mr.height != manifest.mask_height:
                    raise DataError(f"mask {int(mr.mask_ids[0]) if mr.n_masks else 0} of image {entry.image_id} "
                                    "does not match the manifest mask resolution")
                emb = formats.load_mask_embeddings(manifest.resolve(entry.embedding_path), dim, mr.n_masks)
                cams.append(replace(cam, image_id=entry.image_id))
                sets.append((mr.n_masks, mr.width, mr.height, mr.runs, mr.offsets, emb))
                ids.append(entry.image_id)
            except SemsplatError as ex:
                msg = str(ex)
                if not msg.startswith(f"image {entry.image_id}:"):
                    msg = f"image {entry.image_id}: {msg}"
                failures[rank] = msg
                status[rank] = msg
                break
        before = ctx.counters()["pairs"]
        if cams:
            try:
                ctx.encode_views(cams, sets, options.mode)
            except SemsplatError as ex:
                failures[rank] = failures[rank] or str(ex)  # per-image errors name the image
                status[rank] = failures[rank]
        worker_images[rank] = len(cams)
        worker_entries[rank] = ctx.counters()["pairs"] - before  # masked-weight (gid, mask) entries
        if not failures[rank]:
            status[rank] = "ok"
        worker_seconds[rank] = time.perf_counter() - t0
    if any(failures):
        if workers == 1:
            raise DataError(failures[0])
        raise PipelineError("scene encoding failed",
                            [f"worker {r}: {failures[r] or status[r]}" for r in range(workers)], True)
    ctx.synchronize()
    phase1 = time.perf_counter() - t1

    t2 = time.perf_counter()
    n = len(scene)
    rows = np.zeros((n, dim), np.float32)
    cov = np.zeros(n, np.float32)
    step = n if (chunk_rows == 0 or chunk_rows > n) else int(chunk_rows)
    step = max(step, 1)
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        r, c = ctx.encode_finalize(lo, hi)
        rows[lo:hi] = r
        cov[lo:hi] = c
    if stats is not None:
        stats.phase1_seconds = phase1
        stats.phase2_seconds = time.perf_counter() - t2
        stats.worker_seconds = worker_seconds
        stats.worker_images = worker_images
        stats.worker_entries = worker_entries
    return EmbeddingTable(rows, cov)


class VectorStore:
    """Device-resident flat cosine index (vecstore.hpp:52-85): ids + unit rows."""

    def __init__(self, ctx: Context, count: int, dim: int):
        self.ctx = ctx
        self._count = count
        self._dim = dim

    def count(self) -> int:
        return self._count

    def dim(self) -> int:
        return self._dim

    @staticmethod
    def from_unit_rows(ids, unit_rows, device: int = 0) -> "VectorStore":
        ctx = device_context(device)
        ctx.store_set(ids, unit_rows)
        return VectorStore(ctx, int(np.asarray(ids).shape[0]), int(np.asarray(unit_rows).shape[1]))

    def fetch(self):
        return self.ctx.store_fetch()


def build_store(table: EmbeddingTable, scene: GaussianScene | None = None, device: int = 0) -> VectorStore:
    """vecstore.hpp:88-103 (payloads are not kept: the query path only
    needs ids and unit rows)."""
    if scene is not None and table.gaussian_count != len(scene):
        raise ContractError("build_store: table rows and scene size differ")
    ctx = device_context(device)
    cnt = ctx.store_build(table.embeddings, table.coverage)
    return VectorStore(ctx, cnt, table.dim)


def query_topk(store: VectorStore, q, k: int):
    """vecstore.hpp:121-132 for one query (1-D) or a batch (2-D): returns
    (ids, sims) arrays, (sim desc, id asc)."""
    q = np.asarray(q, np.float32)
    single = q.ndim == 1
    if q.shape[-1] != store.dim():
        raise ContractError("query dimension differs from store dimension")
    ids, sims, cnt = store.ctx.query_topk(q, int(k))
    if single:
        n = int(cnt[0])
        return ids[0, :n], sims[0, :n]
    return [(ids[i, :int(cnt[i])], sims[i, :int(cnt[i])]) for i in range(ids.shape[0])]


def query_threshold(store: VectorStore, q, tau: float):
    """vecstore.hpp:135-146"""
    q = np.asarray(q, np.float32).reshape(-1)
    if not (-1.0 <= tau <= 1.0):
        raise ContractError("cosine threshold must lie in [-1, 1]")
    if q.shape[0] != store.dim():
        raise ContractError("query dimension differs from store dimension")
    return store.ctx.query_threshold(q, float(tau))


class PartitionSnapshot:
    """One grid cell of the partitioned store (vecstore.hpp:160-164): cell index,
    bounds (min, max as f64 3-vectors) and the cell's ids / unit rows."""

    def __init__(self, cell, bounds_min, bounds_max, ids, rows):
        self.cell = cell
        self.bounds_min = bounds_min
        self.bounds_max = bounds_max
        self.ids = ids
        self.rows = rows


def partition_store(store: VectorStore, means, cell_size: float) -> list:
    """vecstore.hpp:169-213 on the device: records grouped by the uniform grid
    cell of their payload means (means: [count, 3] in store order), cells in
    (x, y, z) order, records in store order within a cell; bounds = bbox.min
    + cell_size * cell (and + 1), the reference's f64 expressions."""
    if not (cell_size > 0):
        raise ContractError("partition_store: cell_size must be positive")
    if store.count() == 0:
        return []
    cells, offs, _order, ids, rows, bmin = store.ctx.store_partition(means, float(cell_size))
    out = []
    for c in range(cells.shape[0]):
        lo, hi = int(offs[c]), int(offs[c + 1])
        k = cells[c].astype(np.float64)
        out.append(PartitionSnapshot(tuple(int(v) for v in cells[c]), bmin + cell_size * k, bmin + cell_size * (k + 1.0),
                                     ids[lo:hi], rows[lo:hi]))
    return out
