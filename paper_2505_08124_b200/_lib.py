"""ctypes binding of libsemsplat_b200.so (include/semsplat_b200.h).

The library is the only compute path: there is no CPU fallback.  Loading fails
loudly if the in-tree .so is missing (run ``python -m paper_2505_08124_b200.build``
or ``__graft_entry__.build()``), and ``Context`` fails loudly without an sm_100
device.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import raise_for

# SS_LIB_PATH: load another build of the library (A/B timing of kernel variants)
LIB_PATH = Path(os.environ.get("SS_LIB_PATH") or Path(__file__).resolve().parent / "libsemsplat_b200.so")


class Camera(C.Structure):
    """ss_camera == CameraPose (scene.hpp:79-85) at raster resolution."""

    _fields_ = [
        ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
        ("R", C.c_double * 9), ("t", C.c_double * 3),
        ("width", C.c_uint32), ("height", C.c_uint32), ("image_id", C.c_uint32), ("pad", C.c_uint32),
    ]


class ViewMasks(C.Structure):
    _fields_ = [
        ("n_masks", C.c_uint32), ("mask_width", C.c_uint32), ("mask_height", C.c_uint32), ("flags", C.c_uint32),
        ("runs", C.POINTER(C.c_uint32)), ("run_offsets", C.POINTER(C.c_uint64)), ("clip", C.POINTER(C.c_float)),
        ("n_runs", C.c_uint64),
    ]


PROJECTED_DTYPE = np.dtype([
    ("gaussian_id", "<u4"), ("visible", "<u4"), ("mu_x", "<f8"), ("mu_y", "<f8"),
    ("cov_xx", "<f8"), ("cov_xy", "<f8"), ("cov_yy", "<f8"), ("depth", "<f8"),
])
ENTRY_DTYPE = np.dtype([("gaussian_id", "<u4"), ("pixel", "<u4"), ("weight", "<f4")])

K_NAMES = ["masks", "project", "sort", "bin", "raster", "contract", "normalize", "query", "h2d", "query_gemm",
           "query_select", "combine"]

_lib = None


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: the CUDA extension must be built (python -m paper_2505_08124_b200.build); "
            "there is no CPU fallback")
    L = C.CDLL(str(LIB_PATH))
    vp, u32, u64, i32, f32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_float
    pf, pu32, pu64, pd = C.POINTER(C.c_float), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_double)
    sig = {
        "ss_create": (i32, [i32, C.POINTER(vp)]),
        "ss_destroy": (None, [vp]),
        "ss_last_error": (C.c_char_p, []),
        "ss_last_error_kind": (i32, []),
        "ss_set_stream": (i32, [vp, C.c_size_t]),
        "ss_synchronize": (i32, [vp]),
        "ss_set_option": (i32, [vp, i32, C.c_int64]),
        "ss_query_stats": (i32, [vp, vp]),
        "ss_probe_fp64_rate": (i32, [vp, vp]),
        "ss_scene_set_color": (i32, [vp, vp, u64]),
        "ss_render": (i32, [vp, C.POINTER(Camera), i32, pu64, pu64, pu64]),
        "ss_render_fetch_image": (i32, [vp, vp]),
        "ss_assign_classes": (i32, [vp, vp, vp, u64, u32, vp, vp, u32, vp, i32]),
        "ss_scene_set": (i32, [vp, pf, pf, pf, pf, u64]),
        "ss_project": (i32, [vp, C.POINTER(Camera), vp]),
        "ss_raster_capture": (i32, [vp, C.POINTER(Camera), i32, pu64, pu64, pu64]),
        "ss_raster_fetch": (i32, [vp, vp, pf, pf, pu32, pu32, pu32]),
        "ss_encode_begin": (i32, [vp, u32, vp, vp]),
        "ss_encode_view": (i32, [vp, C.POINTER(Camera), C.POINTER(ViewMasks), i32]),
        "ss_encode_views": (i32, [vp, u32, C.POINTER(Camera), C.POINTER(ViewMasks), i32]),
        "ss_encode_finalize": (i32, [vp, u64, u64, vp, vp, i32]),
        "ss_encode_finalize_sparse": (i32, [vp, u64, u64, vp, vp, vp]),
        "ss_normalize_device": (i32, [vp, vp, vp, u64, u32, vp, vp]),
        "ss_store_build": (i32, [vp, pf, pf, u64, u32, pu64]),
        "ss_store_set": (i32, [vp, pu32, pf, u64, u32]),
        "ss_store_fetch": (i32, [vp, pu32, pf]),
        "ss_store_partition": (i32, [vp, pf, C.c_double, pu64]),
        "ss_store_partition_fetch": (i32, [vp, vp, pu64, pu32, pu32, pf, pd]),
        "ss_query_topk": (i32, [vp, pf, u32, u32, pu32, pf, pu64]),
        "ss_query_threshold": (i32, [vp, pf, f32, pu32, pf, u64, pu64]),
        "ss_profile_enable": (i32, [vp, i32]),
        "ss_profile_reset": (i32, [vp]),
        "ss_profile_read": (i32, [vp, pd, pu64, pd]),
        "ss_counters_read": (i32, [vp, pu64]),
        "ss_launch_count": (i32, [vp, pu64, pu64]),
        "ss_device_count": (i32, [C.POINTER(i32)]),
        "ss_comm_unique_id": (i32, [vp]),
        "ss_comm_init": (i32, [vp, i32, i32, vp]),
        "ss_comm_init_all": (i32, [vp, i32]),
        "ss_combine_layout": (i32, [vp, pu64, pu64, pu64, pu64]),
        "ss_encode_combine": (i32, [vp, vp, vp, i32]),
        "ss_combine_layout_for": (i32, [u64, i32, u64, pu64, pu64, pu64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        L = lib()
        raise_for(L.ss_last_error_kind(), L.ss_last_error().decode("utf-8", "replace"))


def camera_struct(cam) -> Camera:
    c = Camera()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    R = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
    t = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    for i in range(9):
        c.R[i] = R[i]
    for i in range(3):
        c.t[i] = t[i]
    c.width, c.height, c.image_id = int(cam.width), int(cam.height), int(cam.image_id)
    return c


class Context:
    """One device context (ss_ctx).  Owns the resident scene and accumulators."""

    def __init__(self, device: int = 0):
        self._L = lib()
        h = C.c_void_p()
        check(self._L.ss_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        self._n = 0
        self._nranks, self._rank = 1, 0
        self._dim = 0

    def close(self):
        if getattr(self, "h", None):
            self._L.ss_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- scene
    def set_scene(self, mean, scale, quat_xyzw, opacity):
        mean = np.ascontiguousarray(mean, np.float32)
        scale = np.ascontiguousarray(scale, np.float32)
        quat = np.ascontiguousarray(quat_xyzw, np.float32)
        op = np.ascontiguousarray(opacity, np.float32)
        n = op.shape[0]
        check(self._L.ss_scene_set(self.h, _ptr(mean, C.c_float), _ptr(scale, C.c_float), _ptr(quat, C.c_float),
                                   _ptr(op, C.c_float), n))
        self._n = n

    def set_stream(self, stream_ptr: int):
        check(self._L.ss_set_stream(self.h, int(stream_ptr)))

    def set_lanes(self, n: int):
        check(self._L.ss_set_option(self.h, 1, int(n)))

    def set_contract_group(self, n: int):
        check(self._L.ss_set_option(self.h, 3, int(n)))

    def set_contract_tc(self, on: bool):
        """SS_OPT_CONTRACT_TC: groups of 2-3 views on the tensor cores."""
        check(self._L.ss_set_option(self.h, 7, int(bool(on))))

    def set_sort_prefix(self, n: int):
        """SS_OPT_SORT_PREFIX: tile lists of the fused pass ranked over a prefix (0 = full sorts)."""
        check(self._L.ss_set_option(self.h, 10, int(n)))

    def set_deterministic(self, on: bool):
        """SS_OPT_DETERMINISTIC: fixed-point per-(Gaussian, mask) scalars, bitwise run-to-run results."""
        check(self._L.ss_set_option(self.h, 9, int(bool(on))))

    def assign_classes(self, rows, coverage, label_ids, label_vecs):
        """eval.hpp:122-158 on the device: class id per row (-1 = unlabeled)."""
        rows = np.ascontiguousarray(rows, np.float32)
        coverage = np.ascontiguousarray(coverage, np.float32)
        lid = np.ascontiguousarray(label_ids, np.int32)
        lv = np.ascontiguousarray(label_vecs, np.float32).reshape(lid.shape[0], -1)
        out = np.zeros(rows.shape[0], np.int32)
        check(self._L.ss_assign_classes(self.h, rows.ctypes.data_as(C.c_void_p), coverage.ctypes.data_as(C.c_void_p),
                                        rows.shape[0], rows.shape[1], lid.ctypes.data_as(C.c_void_p),
                                        lv.ctypes.data_as(C.c_void_p), lid.shape[0], out.ctypes.data_as(C.c_void_p), 0))
        return out

    def assign_classes_device(self, d_rows: int, d_coverage: int, n: int, dim: int, label_ids, label_vecs):
        """assign_classes on device-resident rows/coverage (SS_ROWS_ON_DEVICE)."""
        lid = np.ascontiguousarray(label_ids, np.int32)
        lv = np.ascontiguousarray(label_vecs, np.float32).reshape(lid.shape[0], -1)
        out = np.zeros(n, np.int32)
        check(self._L.ss_assign_classes(self.h, C.c_void_p(d_rows), C.c_void_p(d_coverage), n, dim,
                                        lid.ctypes.data_as(C.c_void_p), lv.ctypes.data_as(C.c_void_p), lid.shape[0],
                                        out.ctypes.data_as(C.c_void_p), 1))
        return out

    def set_query_path(self, path: int):
        """0 = auto, 1 = exact scan, 2 = tensor-core coarse + exact rescore."""
        check(self._L.ss_set_option(self.h, 2, int(path)))

    def set_raster_algo(self, algo: int):
        """SS_OPT_RASTER: 1 = per-step compositor (default), 0 = staged-evaluation compositor (same bits)."""
        check(self._L.ss_set_option(self.h, 5, int(algo)))

    def set_bin_path(self, path: int):
        """0 = auto (tile-sort binning up to 16384 tiles, else direct / key sort), 1 = stable key sort,
        2 = direct count/scan/scatter, 3 = tile-sort binning."""
        check(self._L.ss_set_option(self.h, 4, int(path)))

    def synchronize(self):
        check(self._L.ss_synchronize(self.h))

    # ---- multi-GPU combine (include/semsplat_b200.h, multi-GPU section)
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        check(lib().ss_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        check(self._L.ss_comm_init(self.h, int(nranks), int(rank), buf))
        self._nranks, self._rank = int(nranks), int(rank)

    @staticmethod
    def comm_init_all(ctxs):
        arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
        check(lib().ss_comm_init_all(arr, len(ctxs)))
        for i, c in enumerate(ctxs):
            c._nranks, c._rank = len(ctxs), i

    def set_combine_rows(self, rows: int):
        """SS_OPT_COMBINE_ROWS: block rows of the block-cyclic combine (0 = contiguous shards)."""
        check(self._L.ss_set_option(self.h, 6, int(rows)))

    def set_combine_sparse(self, mode: int):
        """SS_OPT_COMBINE_SPARSE: 0 dense, 1 covered rows with a multi-rank communicator, 2 forced."""
        check(self._L.ss_set_option(self.h, 8, int(mode)))

    def combine_layout(self):
        v = [C.c_uint64() for _ in range(4)]
        check(self._L.ss_combine_layout(self.h, *[C.byref(x) for x in v]))
        return dict(zip(("rows_alloc", "block_rows", "rounds", "rank_rows"), (x.value for x in v)))

    def combine_device(self, d_rows: int, d_coverage: int):
        """ss_encode_combine into device buffers (rank_rows x dim, rank_rows)."""
        check(self._L.ss_encode_combine(self.h, C.c_void_p(d_rows), C.c_void_p(d_coverage), 1))

    def combine(self):
        """ss_encode_combine to host: (rows [rank_rows, dim], coverage [rank_rows], global row ids)."""
        lay = self.combine_layout()
        rr = lay["rank_rows"]
        rows = np.zeros((rr, self._dim), np.float32)
        cov = np.zeros(rr, np.float32)
        check(self._L.ss_encode_combine(self.h, rows.ctypes.data_as(C.c_void_p), cov.ctypes.data_as(C.c_void_p), 0))
        return rows, cov, self.combine_rows_of(lay)

    def combine_rows_of(self, lay=None):
        """Global row index of every combined row this rank holds (block-cyclic, round order)."""
        lay = lay or self.combine_layout()
        B, R = lay["block_rows"], lay["rounds"]
        W, r = self._nranks, self._rank
        q = np.arange(R, dtype=np.int64)[:, None]
        i = np.arange(B, dtype=np.int64)[None, :]
        return (q * W * B + r * B + i).reshape(-1)

    # ---- parity entry points
    def project(self, cam) -> np.ndarray:
        out = np.zeros(self._n, PROJECTED_DTYPE)
        c = camera_struct(cam)
        check(self._L.ss_project(self.h, C.byref(c), out.ctypes.data_as(C.c_void_p)))
        return out

    def set_scene_color(self, rgb):
        rgb = np.ascontiguousarray(rgb, np.float32).reshape(-1, 3)
        check(self._L.ss_scene_set_color(self.h, rgb.ctypes.data_as(C.c_void_p), rgb.shape[0]))

    def render(self, cam, mode: int = 0):
        """rasterize (rasterizer.hpp:261): the capture dict plus "image" [H, W, 3]."""
        out = self.raster_capture(cam, mode, _render=True)
        img = np.zeros((int(cam.height), int(cam.width), 3), np.float32)
        check(self._L.ss_render_fetch_image(self.h, img.ctypes.data_as(C.c_void_p)))
        out["image"] = img
        return out

    def raster_capture(self, cam, mode: int = 0, _render: bool = False):
        c = camera_struct(cam)
        ne, ns, ni = C.c_uint64(), C.c_uint64(), C.c_uint64()
        fn = self._L.ss_render if _render else self._L.ss_raster_capture
        check(fn(self.h, C.byref(c), int(mode), C.byref(ne), C.byref(ns), C.byref(ni)))
        P = int(cam.width) * int(cam.height)
        tiles = ((int(cam.width) + 15) // 16) * ((int(cam.height) + 15) // 16)
        entries = np.zeros(ne.value, ENTRY_DTYPE)
        ppt = np.zeros(P, np.float32)
        alpha = np.zeros(P, np.float32)
        gid = np.zeros(ns.value, np.uint32)
        toff = np.zeros(tiles + 1, np.uint32)
        tspl = np.zeros(ni.value, np.uint32)
        check(self._L.ss_raster_fetch(self.h, entries.ctypes.data_as(C.c_void_p), _ptr(ppt, C.c_float),
                                      _ptr(alpha, C.c_float), _ptr(gid, C.c_uint32), _ptr(toff, C.c_uint32),
                                      _ptr(tspl, C.c_uint32)))
        return {"entries": entries, "per_pixel_total": ppt, "alpha": alpha, "splat_gid": gid,
                "tile_offsets": toff, "tile_splats": tspl}

    # ---- embedding pass
    def encode_begin(self, dim: int, d_sums: int = 0, d_totals: int = 0):
        check(self._L.ss_encode_begin(self.h, int(dim), d_sums or None, d_totals or None))
        self._dim = dim

    def encode_views(self, cams, masks, mode: int = 0):
        """cams: sequence of camera-likes (raster resolution); masks: sequence of
        (n_masks, mask_w, mask_h, runs u32, run_offsets u64, clip f32[n_masks, dim])."""
        nv = len(cams)
        carr = (Camera * max(nv, 1))()
        marr = (ViewMasks * max(nv, 1))()
        keep = []
        for i, (cam, m) in enumerate(zip(cams, masks)):
            carr[i] = camera_struct(cam)
            n_masks, mw, mh, runs, offs, clip = m
            runs = np.ascontiguousarray(runs, np.uint32)
            offs = np.ascontiguousarray(offs, np.uint64)
            clip = np.ascontiguousarray(clip, np.float32)
            keep += [runs, offs, clip]
            marr[i] = ViewMasks(int(n_masks), int(mw), int(mh), 0, _ptr(runs, C.c_uint32), _ptr(offs, C.c_uint64),
                                _ptr(clip, C.c_float), int(offs[-1] - offs[0]) if offs.size else 0)
        check(self._L.ss_encode_views(self.h, nv, carr, marr, int(mode)))

    def encode_views_device(self, cams, dev_masks, mode: int = 0):
        """dev_masks: per view (n_masks, mask_w, mask_h, runs_ptr, offsets_ptr, clip_ptr, n_runs) with
        device pointers (absolute run offsets)."""
        nv = len(cams)
        carr = (Camera * max(nv, 1))()
        marr = (ViewMasks * max(nv, 1))()
        for i, (cam, m) in enumerate(zip(cams, dev_masks)):
            carr[i] = camera_struct(cam)
            n_masks, mw, mh, rp, op, cp, nr = m
            marr[i] = ViewMasks(int(n_masks), int(mw), int(mh), 1, C.cast(C.c_void_p(rp), C.POINTER(C.c_uint32)),
                                C.cast(C.c_void_p(op), C.POINTER(C.c_uint64)), C.cast(C.c_void_p(cp), C.POINTER(C.c_float)),
                                int(nr))
        check(self._L.ss_encode_views(self.h, nv, carr, marr, int(mode)))

    def encode_finalize(self, row_lo: int = 0, row_hi: int | None = None):
        row_hi = self._n if row_hi is None else row_hi
        n = row_hi - row_lo
        rows = np.zeros((n, self._dim), np.float32)
        cov = np.zeros(n, np.float32)
        check(self._L.ss_encode_finalize(self.h, row_lo, row_hi, rows.ctypes.data_as(C.c_void_p),
                                         cov.ctypes.data_as(C.c_void_p), 0))
        return rows, cov

    def encode_finalize_sparse(self, row_lo: int = 0, row_hi: int | None = None):
        """ss_encode_finalize_sparse into zero-filled host arrays: only covered rows are written."""
        row_hi = self._n if row_hi is None else row_hi
        n = row_hi - row_lo
        rows = np.zeros((n, self._dim), np.float32)
        cov = np.zeros(n, np.float32)
        cnt = C.c_uint64()
        check(self._L.ss_encode_finalize_sparse(self.h, row_lo, row_hi, rows.ctypes.data_as(C.c_void_p),
                                                cov.ctypes.data_as(C.c_void_p), C.byref(cnt)))
        return rows, cov, int(cnt.value)

    def encode_finalize_into(self, rows_ptr: int, cov_ptr: int, row_lo: int = 0, row_hi: int | None = None,
                             on_device: bool = False):
        row_hi = self._n if row_hi is None else row_hi
        check(self._L.ss_encode_finalize(self.h, row_lo, row_hi, rows_ptr, cov_ptr, 1 if on_device else 0))

    def normalize_device(self, d_sums: int, d_totals: int, n: int, dim: int, d_rows: int, d_cov: int):
        check(self._L.ss_normalize_device(self.h, d_sums, d_totals, n, dim, d_rows, d_cov))

    # ---- store / query
    def store_build(self, rows, coverage) -> int:
        rows = np.ascontiguousarray(rows, np.float32)
        coverage = np.ascontiguousarray(coverage, np.float32)
        n, dim = rows.shape
        cnt = C.c_uint64()
        check(self._L.ss_store_build(self.h, _ptr(rows, C.c_float), _ptr(coverage, C.c_float), n, dim, C.byref(cnt)))
        self._store = (cnt.value, dim)
        return cnt.value

    def store_set(self, ids, unit_rows):
        ids = np.ascontiguousarray(ids, np.uint32)
        unit_rows = np.ascontiguousarray(unit_rows, np.float32)
        check(self._L.ss_store_set(self.h, _ptr(ids, C.c_uint32), _ptr(unit_rows, C.c_float), ids.shape[0],
                                   unit_rows.shape[1]))
        self._store = (ids.shape[0], unit_rows.shape[1])

    def store_fetch(self):
        cnt, dim = self._store
        ids = np.zeros(cnt, np.uint32)
        rows = np.zeros((cnt, dim), np.float32)
        check(self._L.ss_store_fetch(self.h, _ptr(ids, C.c_uint32), _ptr(rows, C.c_float)))
        return ids, rows

    def store_partition(self, means, cell_size: float):
        """vecstore.hpp:169-213 on the device store: (cells [c, 3] int32, offsets
        [c + 1], order [count] store record per position, ids, rows, bbox_min [3])."""
        cnt, dim = self._store
        means = np.ascontiguousarray(means, np.float32).reshape(cnt, 3)
        nc = C.c_uint64()
        check(self._L.ss_store_partition(self.h, _ptr(means, C.c_float), C.c_double(cell_size), C.byref(nc)))
        c = nc.value
        cells = np.zeros((max(c, 1), 3), np.int32)
        offs = np.zeros(c + 1, np.uint64)
        order = np.zeros(max(cnt, 1), np.uint32)
        ids = np.zeros(max(cnt, 1), np.uint32)
        rows = np.zeros((max(cnt, 1), dim), np.float32)
        bmin = np.zeros(3, np.float64)
        check(self._L.ss_store_partition_fetch(self.h, cells.ctypes.data_as(C.c_void_p), _ptr(offs, C.c_uint64),
                                               _ptr(order, C.c_uint32), _ptr(ids, C.c_uint32), _ptr(rows, C.c_float),
                                               _ptr(bmin, C.c_double)))
        if c == 0:
            offs = np.zeros(0, np.uint64)
        return cells[:c], offs, order[:cnt], ids[:cnt], rows[:cnt], bmin

    def query_topk(self, queries, k: int):
        q = np.ascontiguousarray(queries, np.float32)
        if q.ndim == 1:
            q = q[None, :]
        nq = q.shape[0]
        ids = np.zeros((nq, max(k, 1)), np.uint32)
        sims = np.zeros((nq, max(k, 1)), np.float32)
        cnt = np.zeros(nq, np.uint64)
        check(self._L.ss_query_topk(self.h, _ptr(q, C.c_float), nq, int(k), _ptr(ids, C.c_uint32),
                                    _ptr(sims, C.c_float), _ptr(cnt, C.c_uint64)))
        return ids, sims, cnt

    def query_threshold(self, query, tau: float):
        q = np.ascontiguousarray(query, np.float32).reshape(-1)
        cap = max(self._store[0], 1)
        ids = np.zeros(cap, np.uint32)
        sims = np.zeros(cap, np.float32)
        cnt = C.c_uint64()
        check(self._L.ss_query_threshold(self.h, _ptr(q, C.c_float), C.c_float(tau), _ptr(ids, C.c_uint32),
                                         _ptr(sims, C.c_float), cap, C.byref(cnt)))
        return ids[:cnt.value], sims[:cnt.value]

    # ---- instrumentation
    def profile(self, on: bool = True):
        check(self._L.ss_profile_enable(self.h, 1 if on else 0))

    def profile_reset(self):
        check(self._L.ss_profile_reset(self.h))

    def profile_read(self):
        ms = np.zeros(len(K_NAMES), np.float64)
        la = np.zeros(len(K_NAMES), np.uint64)
        by = np.zeros(len(K_NAMES), np.float64)
        check(self._L.ss_profile_read(self.h, _ptr(ms, C.c_double), _ptr(la, C.c_uint64), _ptr(by, C.c_double)))
        return {k: {"ms": float(ms[i]), "launches": int(la[i]), "bytes": float(by[i])} for i, k in enumerate(K_NAMES)}

    def counters(self):
        out = np.zeros(5, np.uint64)
        check(self._L.ss_counters_read(self.h, _ptr(out, C.c_uint64)))
        return dict(zip(["n_vis", "instances", "touched", "pairs", "views"], map(int, out)))

    def query_stats(self):
        out = np.zeros(4, np.uint64)
        check(self._L.ss_query_stats(self.h, out.ctypes.data_as(C.c_void_p)))
        return dict(zip(["tc_queries", "candidates", "max_candidates", "exact_fallbacks"], map(int, out)))

    def probe_fp64_rate(self) -> float:
        """DFMA lane-operations per second on this device (fp64 pipe peak)."""
        out = C.c_double(0.0)
        check(self._L.ss_probe_fp64_rate(self.h, C.byref(out)))
        return float(out.value)

    def launch_count(self):
        a, b = C.c_uint64(), C.c_uint64()
        self._L.ss_launch_count(self.h, C.byref(a), C.byref(b))
        return a.value, b.value
