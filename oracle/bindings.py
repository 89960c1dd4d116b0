"""ctypes bindings of the two CPU checkers -- TEST INFRASTRUCTURE ONLY.

  Oracle(): oracle/libssoracle.so, the C restatement (ssoracle.c)
  Ref():    oracle/_ref/libssref.so, the reference's own headers compiled here

Camera-likes are any object with fx, fy, cx, cy, rotation (3x3), translation,
width, height, image_id.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "libssoracle.so"
REF_SO = HERE / "_ref" / "libssref.so"

PROJECTED = np.dtype([("gaussian_id", "<u4"), ("visible", "<u4"), ("mu_x", "<f8"), ("mu_y", "<f8"),
                      ("cov_xx", "<f8"), ("cov_xy", "<f8"), ("cov_yy", "<f8"), ("depth", "<f8")])
ENTRY = np.dtype([("gaussian_id", "<u4"), ("pixel", "<u4"), ("weight", "<f4")])


class CCam(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("R", C.c_double * 9), ("t", C.c_double * 3), ("width", C.c_uint32), ("height", C.c_uint32),
                ("image_id", C.c_uint32), ("pad", C.c_uint32)]


def ccam(cam) -> CCam:
    c = CCam()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    R = np.asarray(cam.rotation, np.float64).reshape(9)
    t = np.asarray(cam.translation, np.float64).reshape(3)
    for i in range(9):
        c.R[i] = R[i]
    for i in range(3):
        c.t[i] = t[i]
    c.width, c.height, c.image_id = int(cam.width), int(cam.height), int(getattr(cam, "image_id", 0))
    return c


class CamView:
    """Plain camera record built from a CCam."""

    def __init__(self, c: CCam):
        self.fx, self.fy, self.cx, self.cy = c.fx, c.fy, c.cx, c.cy
        self.rotation = np.array(list(c.R), np.float64).reshape(3, 3)
        self.translation = np.array(list(c.t), np.float64)
        self.width, self.height, self.image_id = c.width, c.height, c.image_id


def _p(a, t=C.c_void_p):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(t)) if t is not C.c_void_p else a.ctypes.data_as(C.c_void_p)


def _scene_args(scene):
    mean = np.ascontiguousarray(scene.mean, np.float32)
    scale = np.ascontiguousarray(scene.scale, np.float32)
    quat = np.ascontiguousarray(scene.quat_xyzw, np.float32)
    op = np.ascontiguousarray(scene.opacity, np.float32)
    return (mean, scale, quat, op), (_p(mean, C.c_float), _p(scale, C.c_float), _p(quat, C.c_float),
                                     _p(op, C.c_float), op.shape[0])


class OracleNumericError(Exception):
    pass


class Oracle:
    """The C restatement of the path (oracle/ssoracle.c)."""

    class Args(C.Structure):
        _fields_ = [("mean", C.c_void_p), ("scale", C.c_void_p), ("quat", C.c_void_p), ("opacity", C.c_void_p),
                    ("n", C.c_uint64), ("cams", C.c_void_p), ("nviews", C.c_uint32), ("mask_w", C.c_uint32),
                    ("mask_h", C.c_uint32), ("masks_per_view", C.c_void_p), ("view_mask_offset", C.c_void_p),
                    ("runs", C.c_void_p), ("run_offsets", C.c_void_p), ("clip", C.c_void_p), ("dim", C.c_uint32),
                    ("mode", C.c_int)]

    class Raster(C.Structure):
        _fields_ = [("n_entries", C.c_uint64), ("entries", C.c_void_p), ("per_pixel_total", C.POINTER(C.c_float)),
                    ("alpha", C.POINTER(C.c_float)), ("n_splats", C.c_uint64), ("splat_gid", C.POINTER(C.c_uint32)),
                    ("tiles", C.c_uint32), ("tile_offsets", C.POINTER(C.c_uint32)),
                    ("tile_splats", C.POINTER(C.c_uint32)), ("status", C.c_int), ("bad_gid", C.c_uint32)]

    def __init__(self):
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run oracle/build_oracle.py")
        L = C.CDLL(str(ORACLE_SO))
        L.sso_exp.restype = C.c_double
        L.sso_exp.argtypes = [C.c_double]
        L.sso_exp_table.argtypes = [C.c_void_p]
        L.sso_project.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.POINTER(CCam), C.c_void_p]
        L.sso_rasterize.restype = C.POINTER(Oracle.Raster)
        L.sso_rasterize.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.POINTER(CCam), C.c_int]
        L.sso_raster_free.argtypes = [C.c_void_p]
        L.sso_rle_decode.restype = C.c_int
        L.sso_rle_decode.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p]
        L.sso_resample_mask.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        L.sso_mask_weights.restype = C.c_uint64
        L.sso_mask_weights.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        L.sso_encode.restype = C.c_int
        L.sso_encode.argtypes = [C.POINTER(Oracle.Args), C.c_void_p, C.c_void_p]
        L.sso_encode_partial.restype = C.c_int
        L.sso_encode_partial.argtypes = [C.POINTER(Oracle.Args), C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
        L.sso_finalize.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p]
        L.sso_dot_lanes.restype = C.c_float
        L.sso_dot_lanes.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.sso_normalized_copy.restype = C.c_int
        L.sso_normalized_copy.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.sso_query_threshold.restype = C.c_int
        L.sso_query_threshold.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_float,
                                          C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
        L.sso_query_topk.restype = C.c_int
        L.sso_query_topk.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint32,
                                     C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        self.L = L

    def exp(self, x):
        x = np.asarray(x, np.float64)
        return np.array([self.L.sso_exp(float(v)) for v in x.reshape(-1)], np.float64).reshape(x.shape)

    def exp_table(self):
        t = np.zeros(256, np.uint64)
        self.L.sso_exp_table(_p(t))
        return t

    def project(self, scene, cam):
        keep, a = _scene_args(scene)
        out = np.zeros(a[4], PROJECTED)
        c = ccam(cam)
        self.L.sso_project(*[C.cast(x, C.c_void_p) for x in a[:4]], a[4], C.byref(c), _p(out))
        return out

    def rasterize(self, scene, cam, mode: int = 0):
        keep, a = _scene_args(scene)
        c = ccam(cam)
        r = self.L.sso_rasterize(*[C.cast(x, C.c_void_p) for x in a[:4]], a[4], C.byref(c), int(mode))
        try:
            R = r.contents
            if R.status == 3:
                raise OracleNumericError(f"singular screen covariance for gaussian {R.bad_gid}")
            P = int(cam.width) * int(cam.height)
            ne = R.n_entries
            entries = np.frombuffer((C.c_char * (ne * 12)).from_address(R.entries), ENTRY, ne).copy() if ne else \
                np.zeros(0, ENTRY)
            out = {
                "entries": entries,
                "per_pixel_total": np.ctypeslib.as_array(R.per_pixel_total, (max(P, 1),))[:P].copy(),
                "alpha": np.ctypeslib.as_array(R.alpha, (max(P, 1),))[:P].copy(),
                "splat_gid": np.ctypeslib.as_array(R.splat_gid, (max(R.n_splats, 1),))[:R.n_splats].copy(),
                "tile_offsets": np.ctypeslib.as_array(R.tile_offsets, (R.tiles + 1,)).copy(),
            }
            ni = int(out["tile_offsets"][-1])
            out["tile_splats"] = np.ctypeslib.as_array(R.tile_splats, (max(ni, 1),))[:ni].copy()
            return out
        finally:
            self.L.sso_raster_free(C.cast(r, C.c_void_p))

    def rle_decode(self, runs, w, h):
        runs = np.ascontiguousarray(runs, np.uint32)
        out = np.zeros(w * h, np.uint8)
        st = self.L.sso_rle_decode(_p(runs), runs.shape[0], w, h, _p(out))
        if st:
            raise ValueError("mask RLE length mismatch")
        return out

    def resample_mask(self, bits, w, h, tw, th):
        bits = np.ascontiguousarray(bits, np.uint8)
        out = np.zeros(tw * th, np.uint8)
        self.L.sso_resample_mask(_p(bits), w, h, tw, th, _p(out))
        return out

    def mask_weights(self, entries, bits, n_gauss):
        entries = np.ascontiguousarray(entries, ENTRY)
        bits = np.ascontiguousarray(bits, np.uint8)
        scratch = np.zeros(max(n_gauss, 1), np.float64)
        seen = np.zeros(max(n_gauss, 1), np.uint8)
        gids = np.zeros(max(entries.shape[0], 1), np.uint32)
        sums = np.zeros(max(entries.shape[0], 1), np.float64)
        m = self.L.sso_mask_weights(_p(entries), entries.shape[0], _p(bits), _p(scratch), _p(seen), _p(gids),
                                    _p(sums))
        return gids[:m].copy(), sums[:m].copy()

    def _encode_args(self, scene, cams, masks, dim, mode):
        keep, a = _scene_args(scene)
        nv = len(cams)
        carr = (CCam * max(nv, 1))(*[ccam(c) for c in cams])
        mpv = np.array([m[0] for m in masks], np.uint32)
        vmo = np.zeros(nv + 1, np.uint64)
        vmo[1:] = np.cumsum(mpv)
        runs_l, offs_l, clip_l, base = [], [], [], 0
        for (nm, mw, mh, runs, offs, clip) in masks:
            offs = np.asarray(offs, np.uint64)
            runs_l.append(np.asarray(runs, np.uint32)[int(offs[0]):int(offs[-1])])
            offs_l.append((offs[:-1] - offs[0] + base).astype(np.uint64))
            base += int(offs[-1] - offs[0])
            clip_l.append(np.asarray(clip, np.float32).reshape(nm, dim))
        runs = np.concatenate(runs_l) if runs_l else np.zeros(1, np.uint32)
        offs = np.concatenate(offs_l + [np.array([base], np.uint64)])
        clip = np.ascontiguousarray(np.concatenate(clip_l) if clip_l else np.zeros((1, dim), np.float32))
        mw, mh = (masks[0][1], masks[0][2]) if masks else (0, 0)
        args = Oracle.Args(*[C.cast(x, C.c_void_p) for x in a[:4]], a[4], C.cast(carr, C.c_void_p), nv, mw, mh,
                           _p(mpv), _p(vmo), _p(runs), _p(offs), _p(clip), dim, mode)
        return args, (keep, carr, mpv, vmo, runs, offs, clip)

    def encode(self, scene, cams, masks, dim, mode: int = 0):
        """cams: raster cameras; masks: list of (n_masks, mw, mh, runs, run_offsets, clip).
        Returns (rows f32 N x dim, coverage f32 N) -- encode_scene with one worker."""
        args, keep = self._encode_args(scene, cams, masks, dim, mode)
        n = len(scene.opacity)
        rows = np.zeros((max(n, 1), dim), np.float32)
        cov = np.zeros(max(n, 1), np.float32)
        st = self.L.sso_encode(C.byref(args), _p(rows), _p(cov))
        if st == 3:
            raise OracleNumericError("singular screen covariance")
        if st:
            raise ValueError(f"oracle encode failed with status {st}")
        return rows[:n], cov[:n]

    def encode_partial(self, scene, cams, masks, dim, v_lo, v_hi, mode: int = 0):
        args, keep = self._encode_args(scene, cams, masks, dim, mode)
        n = len(scene.opacity)
        s = np.zeros((max(n, 1), dim), np.float64)
        t = np.zeros(max(n, 1), np.float64)
        st = self.L.sso_encode_partial(C.byref(args), v_lo, v_hi, _p(s), _p(t))
        if st:
            raise ValueError(f"oracle encode failed with status {st}")
        return s[:n], t[:n]

    def dot_lanes(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.L.sso_dot_lanes(_p(a), _p(b), a.shape[0])

    def normalized_copy(self, v):
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros_like(v)
        if self.L.sso_normalized_copy(_p(v), v.shape[0], _p(out)):
            raise OracleNumericError("cannot normalize a zero vector")
        return out

    def query_topk(self, ids, rows, queries, k, threads: int = 1):
        ids = np.ascontiguousarray(ids, np.uint32)
        rows = np.ascontiguousarray(rows, np.float32)
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, rows.shape[1] if rows.ndim == 2 else 1)
        nq = q.shape[0]
        oid = np.zeros((nq, max(k, 1)), np.uint32)
        osim = np.zeros((nq, max(k, 1)), np.float32)
        cnt = np.zeros(nq, np.uint64)
        st = self.L.sso_query_topk(_p(ids), _p(rows), ids.shape[0], rows.shape[1], _p(q), nq, k, threads, _p(oid),
                                   _p(osim), _p(cnt))
        if st == 3:
            raise OracleNumericError("cannot normalize a zero vector")
        return oid, osim, cnt


    def query_threshold(self, ids, rows, q, tau):
        ids = np.ascontiguousarray(ids, np.uint32)
        rows = np.ascontiguousarray(rows, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        oid = np.zeros(max(ids.shape[0], 1), np.uint32)
        osim = np.zeros(max(ids.shape[0], 1), np.float32)
        cnt = C.c_uint64()
        st = self.L.sso_query_threshold(_p(ids), _p(rows), ids.shape[0], rows.shape[1], _p(q), C.c_float(tau),
                                        _p(oid), _p(osim), oid.shape[0], C.byref(cnt))
        if st == 3:
            raise OracleNumericError("cannot normalize a zero vector")
        if st == 1:
            raise ValueError("cosine threshold must lie in [-1, 1]")
        return oid[:cnt.value].copy(), osim[:cnt.value].copy()


class RefError(Exception):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


class Ref:
    """The reference's own code (unmodified headers + eigen shim)."""

    def __init__(self):
        if not REF_SO.exists():
            raise RuntimeError(f"{REF_SO} missing (built only where /root/reference exists)")
        L = C.CDLL(str(REF_SO))
        L.ssref_last_error.restype = C.c_char_p
        L.ssref_dot_lanes.restype = C.c_float
        L.ssref_dot_lanes.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.ssref_hardware_threads.restype = C.c_uint32
        L.ssref_encode.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.c_char_p, C.c_uint32, C.c_uint64, C.c_int,
                                                      C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ssref_query_topk.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint32,
                                       C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ssref_query_threshold.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_float,
                                            C.c_void_p, C.c_void_p, C.c_void_p]
        L.ssref_look_at.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.POINTER(CCam)]
        L.ssref_camera_scaled_to.argtypes = [C.POINTER(CCam), C.c_uint32, C.c_uint32, C.POINTER(CCam)]
        L.ssref_write_fixture.argtypes = [C.c_uint32] * 6 + [C.c_uint64, C.c_char_p, C.c_char_p, C.c_uint64]
        L.ssref_rasterize.argtypes = [C.c_void_p] * 5 + [C.c_uint64, C.POINTER(CCam), C.c_int, C.c_int,
                                                         C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]
        L.ssref_weightmap_fetch.argtypes = [C.c_void_p] * 4
        L.ssref_image_fetch.argtypes = [C.c_void_p] * 2
        L.ssref_assign_classes.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p,
                                           C.c_uint32, C.c_void_p]
        L.ssref_image_fetch.restype = None
        L.ssref_weightmap_free.argtypes = [C.c_void_p]
        L.ssref_mask_weights.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        L.ssref_synth_embedding.argtypes = [C.c_char_p, C.c_uint32, C.c_void_p]
        L.ssref_load_scene_count.argtypes = [C.c_char_p, C.c_void_p]
        L.ssref_load_scene.argtypes = [C.c_char_p] + [C.c_void_p] * 5
        L.ssref_save_scene.argtypes = [C.c_char_p] + [C.c_void_p] * 5 + [C.c_uint64]
        L.ssref_load_cameras.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64, C.c_void_p]
        L.ssref_project.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.POINTER(CCam), C.c_void_p]
        L.ssref_depth_order.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.POINTER(CCam), C.c_void_p, C.c_void_p]
        L.ssref_resample_mask.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        L.ssref_normalized_copy.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.ssref_build_store.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
        L.ssref_partition_store.argtypes = [C.c_void_p] * 3 + [C.c_uint64, C.c_uint32, C.c_double] + [C.c_void_p] * 6
        self.L = L

    def _chk(self, rc):
        if rc:
            raise RefError(self.L.ssref_last_error_kind(), self.L.ssref_last_error().decode())

    def hardware_threads(self) -> int:
        return int(self.L.ssref_hardware_threads())

    def project(self, scene, cam):
        keep, a = _scene_args(scene)
        out = np.zeros(a[4], PROJECTED)
        c = ccam(cam)
        self._chk(self.L.ssref_project(*[C.cast(x, C.c_void_p) for x in a[:4]], a[4], C.byref(c), _p(out)))
        return out

    def depth_order(self, scene, cam):
        keep, a = _scene_args(scene)
        ids = np.zeros(max(a[4], 1), np.uint32)
        nv = C.c_uint64()
        c = ccam(cam)
        self._chk(self.L.ssref_depth_order(*[C.cast(x, C.c_void_p) for x in a[:4]], a[4], C.byref(c), _p(ids),
                                           C.byref(nv)))
        return ids[:nv.value].copy()

    def rasterize(self, scene, cam, mode: int = 0, full_render: bool = False, masks=None):
        """Returns entries, per_pixel_total (and alpha when full_render).  masks:
        optional list of raster-res u8 bitmaps; returns their mask_weights too."""
        keep, a = _scene_args(scene)
        color = None
        if full_render:
            color = np.ascontiguousarray(scene.color if getattr(scene, "color", None) is not None else
                                         np.zeros((a[4], 3), np.float32), np.float32)
        c = ccam(cam)
        h = C.c_void_p()
        ne = C.c_uint64()
        self._chk(self.L.ssref_rasterize(*[C.cast(x, C.c_void_p) for x in a[:4]], _p(color), a[4], C.byref(c),
                                         int(mode), 1 if full_render else 0, C.byref(h), C.byref(ne)))
        try:
            P = int(cam.width) * int(cam.height)
            entries = np.zeros(ne.value, ENTRY)
            ppt = np.zeros(P, np.float32)
            alpha = np.zeros(P, np.float32)
            self.L.ssref_weightmap_fetch(h, _p(entries), _p(ppt), _p(alpha) if full_render else None)
            out = {"entries": entries, "per_pixel_total": ppt}
            if full_render:
                out["alpha"] = alpha
                image = np.zeros(3 * P, np.float32)
                self.L.ssref_image_fetch(h, _p(image))
                out["image"] = image.reshape(int(cam.height), int(cam.width), 3)
            if masks is not None:
                mw = []
                for bits in masks:
                    bits = np.ascontiguousarray(bits, np.uint8)
                    g = np.zeros(max(ne.value, 1), np.uint32)
                    s = np.zeros(max(ne.value, 1), np.float64)
                    cnt = C.c_uint64()
                    self._chk(self.L.ssref_mask_weights(h, _p(bits), int(cam.width), int(cam.height), _p(g), _p(s),
                                                        C.byref(cnt)))
                    mw.append((g[:cnt.value].copy(), s[:cnt.value].copy()))
                out["mask_weights"] = mw
            return out
        finally:
            self.L.ssref_weightmap_free(h)

    def resample_mask(self, bits, w, h, tw, th):
        bits = np.ascontiguousarray(bits, np.uint8)
        out = np.zeros(tw * th, np.uint8)
        self._chk(self.L.ssref_resample_mask(_p(bits), w, h, tw, th, _p(out)))
        return out

    def encode(self, scene, manifest_path, workers=1, chunk_rows=0, mode=0, contiguous=False):
        keep, a = _scene_args(scene)
        import re
        dim = 512
        for line in Path(manifest_path).read_text().splitlines():
            m = re.match(r"\s*embedding_dim\s*=\s*(\d+)", line)
            if m:
                dim = int(m.group(1))
        n = a[4]
        rows = np.zeros((max(n, 1), dim), np.float32)
        cov = np.zeros(max(n, 1), np.float32)
        stats = np.zeros(3, np.float64)
        self._chk(self.L.ssref_encode(*[C.cast(x, C.c_void_p) for x in a[:4]], n, str(manifest_path).encode(),
                                      workers, chunk_rows, mode, 1 if contiguous else 0, _p(rows), _p(cov),
                                      _p(stats)))
        return rows[:n], cov[:n], stats

    def load_scene(self, path):
        n = C.c_uint64()
        self._chk(self.L.ssref_load_scene_count(str(path).encode(), C.byref(n)))
        N = n.value
        mean = np.zeros((N, 3), np.float32)
        scale = np.zeros((N, 3), np.float32)
        quat = np.zeros((N, 4), np.float32)
        op = np.zeros(N, np.float32)
        color = np.zeros((N, 3), np.float32)
        self._chk(self.L.ssref_load_scene(str(path).encode(), _p(mean), _p(scale), _p(quat), _p(op), _p(color)))
        return mean, scale, quat, op, color

    def save_scene(self, path, mean, scale, quat, opacity, color=None):
        arrs = [np.ascontiguousarray(x, np.float32) for x in (mean, scale, quat, opacity)]
        col = np.ascontiguousarray(color if color is not None else np.zeros((arrs[3].shape[0], 3)), np.float32)
        self._chk(self.L.ssref_save_scene(str(path).encode(), *[_p(x) for x in arrs], _p(col), arrs[3].shape[0]))

    def load_cameras(self, path):
        cap = 1 << 16
        arr = (CCam * cap)()
        n = C.c_uint64()
        self._chk(self.L.ssref_load_cameras(str(path).encode(), C.cast(arr, C.c_void_p), cap, C.byref(n)))
        return [CamView(arr[i]) for i in range(n.value)]

    def camera_scaled_to(self, cam, w, h):
        out = CCam()
        c = ccam(cam)
        self.L.ssref_camera_scaled_to(C.byref(c), w, h, C.byref(out))
        return CamView(out)

    def look_at(self, eye, target, w, h, focal):
        e = np.ascontiguousarray(eye, np.float64)
        t = np.ascontiguousarray(target, np.float64)
        out = CCam()
        self.L.ssref_look_at(_p(e), _p(t), w, h, float(focal), C.byref(out))
        return CamView(out)

    def write_fixture(self, directory, objects=3, per_object=12, views=4, resolution=32, mask_scale=1, dim=16,
                      seed=5):
        buf = C.create_string_buffer(4096)
        self._chk(self.L.ssref_write_fixture(objects, per_object, views, resolution, mask_scale, dim, seed,
                                             str(directory).encode(), buf, 4096))
        return buf.value.decode()

    def synth_embedding(self, label, dim):
        out = np.zeros(dim, np.float32)
        self._chk(self.L.ssref_synth_embedding(label.encode(), dim, _p(out)))
        return out

    def dot_lanes(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.L.ssref_dot_lanes(_p(a), _p(b), a.shape[0])

    def normalized_copy(self, v):
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros_like(v)
        self._chk(self.L.ssref_normalized_copy(_p(v), v.shape[0], _p(out)))
        return out

    def build_store(self, rows, coverage):
        rows = np.ascontiguousarray(rows, np.float32)
        coverage = np.ascontiguousarray(coverage, np.float32)
        n, dim = rows.shape
        ids = np.zeros(max(n, 1), np.uint32)
        out = np.zeros((max(n, 1), dim), np.float32)
        cnt = C.c_uint64()
        self._chk(self.L.ssref_build_store(_p(rows), _p(coverage), n, dim, _p(ids), _p(out), C.byref(cnt)))
        return ids[:cnt.value].copy(), out[:cnt.value].copy()

    def query_topk(self, ids, rows, queries, k, threads: int = 1):
        ids = np.ascontiguousarray(ids, np.uint32)
        rows = np.ascontiguousarray(rows, np.float32)
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, rows.shape[1])
        nq = q.shape[0]
        oid = np.zeros((nq, max(k, 1)), np.uint32)
        osim = np.zeros((nq, max(k, 1)), np.float32)
        cnt = np.zeros(nq, np.uint64)
        self._chk(self.L.ssref_query_topk(_p(ids), _p(rows), ids.shape[0], rows.shape[1], _p(q), nq, k, threads,
                                          _p(oid), _p(osim), _p(cnt)))
        return oid, osim, cnt

    def assign_classes(self, rows, coverage, label_ids, label_vecs):
        rows = np.ascontiguousarray(rows, np.float32)
        coverage = np.ascontiguousarray(coverage, np.float32)
        lid = np.ascontiguousarray(label_ids, np.int32)
        lv = np.ascontiguousarray(label_vecs, np.float32)
        out = np.zeros(rows.shape[0], np.int32)
        self._chk(self.L.ssref_assign_classes(_p(rows), _p(coverage), rows.shape[0], rows.shape[1], _p(lid), _p(lv),
                                              lid.shape[0], _p(out)))
        return out

    def query_threshold(self, ids, rows, q, tau):
        ids = np.ascontiguousarray(ids, np.uint32)
        rows = np.ascontiguousarray(rows, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        oid = np.zeros(max(ids.shape[0], 1), np.uint32)
        osim = np.zeros(max(ids.shape[0], 1), np.float32)
        cnt = C.c_uint64()
        self._chk(self.L.ssref_query_threshold(_p(ids), _p(rows), ids.shape[0], rows.shape[1], _p(q),
                                               C.c_float(tau), _p(oid), _p(osim), C.byref(cnt)))
        return oid[:cnt.value].copy(), osim[:cnt.value].copy()

    def partition_store(self, ids, rows, means, cell_size):
        """vecstore.hpp:169-213 on a store with payload means: (cells [c,3],
        bounds [c,6], offsets [c+1], ids, rows) in the reference's order."""
        ids = np.ascontiguousarray(ids, np.uint32)
        rows = np.ascontiguousarray(rows, np.float32)
        means = np.ascontiguousarray(means, np.float32)
        n = ids.shape[0]
        cap = max(n, 1)
        nc = C.c_uint64()
        cells = np.zeros((cap, 3), np.int32)
        bounds = np.zeros((cap, 6), np.float64)
        offs = np.zeros(cap + 1, np.uint64)
        oid = np.zeros(cap, np.uint32)
        orow = np.zeros((cap, rows.shape[1]), np.float32)
        self._chk(self.L.ssref_partition_store(_p(ids), _p(rows), _p(means), n, rows.shape[1], C.c_double(cell_size),
                                               C.byref(nc), _p(cells), _p(bounds), _p(offs), _p(oid), _p(orow)))
        c = nc.value
        return cells[:c], bounds[:c], offs[:c + 1], oid[:n], orow[:n]
