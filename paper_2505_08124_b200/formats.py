"""Readers/writers for the reference's on-disk formats (the step before the path).

Masks stay in their RLE encoding here: the run streams are handed to the device,
which decodes and resamples them.  Formats:
  manifest      providers.hpp:208-291   (text, key = value)
  cameras       scene_io.hpp:217-255    (text, one record per line)
  mask sets     providers.hpp:111-152   ("MRLE", runs zeros-first)
  embeddings    providers.hpp:154-204   ("EMBV", f32 records)
  scene PLY     scene_io.hpp:132-212    (3DGS binary_little_endian)
"""
from __future__ import annotations

import math
import os
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import DataError, FormatError, IoError

MASK_MAGIC = 0x454C524D  # "MRLE"
EMB_MAGIC = 0x56424D45   # "EMBV"
SH_C0 = 0.28209479177387814
LOGIT_CLAMP = 15.0


@dataclass
class ImageEntry:
    image_id: int
    rgb_path: str
    camera_id: int
    mask_path: str
    embedding_path: str


@dataclass
class DatasetManifest:
    """providers.hpp:220-235"""
    root: str = "."
    camera_file: str = ""
    mask_width: int = 0
    mask_height: int = 0
    raster_width: int = 0
    raster_height: int = 0
    embedding_dim: int = 512
    images: list = field(default_factory=list)

    def resolve(self, rel: str) -> str:
        return str(Path(self.root) / rel)

    def entry(self, image_id: int) -> ImageEntry:
        for e in self.images:
            if e.image_id == image_id:
                return e
        raise DataError(f"manifest has no image with id {image_id}")


def load_manifest(path: str) -> DatasetManifest:
    """providers.hpp:237-278"""
    try:
        text = Path(path).read_text()
    except OSError:
        raise IoError(f"cannot open manifest: {path}")
    m = DatasetManifest(root=str(Path(path).parent) or ".")
    for ln, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0]
        toks = line.split()
        if not toks:
            continue
        if len(toks) < 2 or toks[1] != "=":
            raise FormatError(f"manifest: expected 'key = value' at line {ln}")
        key, vals = toks[0], toks[2:]
        try:
            if key == "version":
                int(vals[0])
            elif key == "cameras":
                m.camera_file = vals[0]
            elif key == "mask_resolution":
                m.mask_width, m.mask_height = int(vals[0]), int(vals[1])
            elif key == "raster_resolution":
                m.raster_width, m.raster_height = int(vals[0]), int(vals[1])
            elif key == "embedding_dim":
                m.embedding_dim = int(vals[0])
            elif key == "image":
                m.images.append(ImageEntry(int(vals[0]), vals[1], int(vals[2]), vals[3], vals[4]))
            else:
                raise FormatError(f"manifest: unknown key '{key}' at line {ln}")
        except (IndexError, ValueError):
            raise FormatError(f"manifest: malformed value at line {ln}")
    return m


def save_manifest(m: DatasetManifest, path: str) -> None:
    """providers.hpp:280-291"""
    lines = ["version = 1", f"cameras = {m.camera_file}", f"mask_resolution = {m.mask_width} {m.mask_height}",
             f"raster_resolution = {m.raster_width} {m.raster_height}", f"embedding_dim = {m.embedding_dim}"]
    lines += [f"image = {e.image_id} {e.rgb_path} {e.camera_id} {e.mask_path} {e.embedding_path}" for e in m.images]
    Path(path).write_text("\n".join(lines) + "\n")


@dataclass
class CameraPose:
    """scene.hpp:79-85 (world-to-camera, +z forward, top-left origin)."""
    image_id: int = 0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    width: int = 0
    height: int = 0


def validate_camera(cam: CameraPose) -> None:
    """scene.hpp:88-98"""
    R = np.asarray(cam.rotation, np.float64)
    if np.abs(R.T @ R - np.eye(3)).max() > 1e-4:
        raise DataError(f"camera {cam.image_id}: rotation is not orthonormal")
    if np.linalg.det(R) < 0:
        raise DataError(f"camera {cam.image_id}: rotation has determinant -1")
    if not (cam.fx > 0) or not (cam.fy > 0):
        raise DataError(f"camera {cam.image_id}: focal lengths must be positive")
    if not (cam.cx > 0) or not (cam.cx < cam.width) or not (cam.cy > 0) or not (cam.cy < cam.height):
        raise DataError(f"camera {cam.image_id}: principal point outside the image")


def load_cameras(path: str) -> list:
    """scene_io.hpp:217-241"""
    try:
        text = Path(path).read_text()
    except OSError:
        raise IoError(f"cannot open camera file: {path}")
    cams = []
    for ln, line in enumerate(text.splitlines(), 1):
        toks = line.split("#", 1)[0].split()
        if not toks:
            continue
        if len(toks) < 19:
            raise FormatError(f"camera file: malformed record at line {ln}")
        try:
            v = [float(x) for x in toks[1:17]]
            cam = CameraPose(image_id=int(toks[0]), fx=v[0], fy=v[1], cx=v[2], cy=v[3],
                             rotation=np.array(v[4:13], np.float64).reshape(3, 3),
                             translation=np.array(v[13:16], np.float64), width=int(toks[17]), height=int(toks[18]))
        except ValueError:
            raise FormatError(f"camera file: malformed record at line {ln}")
        validate_camera(cam)
        cams.append(cam)
    return cams


def save_cameras(cams, path: str) -> None:
    """scene_io.hpp:243-255 (precision 17)"""
    out = ["# image_id fx fy cx cy r00 r01 r02 r10 r11 r12 r20 r21 r22 tx ty tz width height"]
    for c in cams:
        vals = [c.fx, c.fy, c.cx, c.cy, *np.asarray(c.rotation, np.float64).reshape(9),
                *np.asarray(c.translation, np.float64).reshape(3)]
        out.append(" ".join([str(c.image_id)] + [repr(float(x)) for x in vals] + [str(c.width), str(c.height)]))
    Path(path).write_text("\n".join(out) + "\n")


@dataclass
class MaskRuns:
    """A mask set in its RLE encoding: masks sorted by mask_id
    (providers.hpp:148-150); runs of mask j = runs[offsets[j]:offsets[j+1]]."""
    image_id: int
    width: int
    height: int
    mask_ids: np.ndarray
    runs: np.ndarray
    offsets: np.ndarray

    @property
    def n_masks(self) -> int:
        return int(self.mask_ids.shape[0])


def load_maskset_runs(path: str, image_id: int) -> MaskRuns:
    """providers.hpp:129-152, without decoding (the device decodes)."""
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise IoError(f"cannot open mask file: {path}")
    if len(data) < 16:
        raise FormatError("unexpected end of stream")
    magic, w, h, count = struct.unpack_from("<4I", data, 0)
    if magic != MASK_MAGIC:
        raise FormatError(f"bad mask file magic: {path}")
    pos = 16
    masks = []
    for _ in range(count):
        if pos + 12 > len(data):
            raise FormatError("unexpected end of stream")
        mid, nr = struct.unpack_from("<IQ", data, pos)
        pos += 12
        if pos + 4 * nr > len(data):
            raise FormatError("unexpected end of stream")
        runs = np.frombuffer(data, np.uint32, nr, pos).copy()
        pos += 4 * nr
        tot = int(runs.sum(dtype=np.uint64))
        if tot > w * h:
            raise FormatError("mask RLE length mismatch (overlong stream)")
        if tot != w * h:
            raise FormatError(f"mask RLE length mismatch: runs cover {tot} of {w * h} pixels")
        masks.append((mid, runs))
    masks.sort(key=lambda t: t[0])
    offs = np.zeros(len(masks) + 1, np.uint64)
    for j, (_, r) in enumerate(masks):
        offs[j + 1] = offs[j] + r.shape[0]
    runs = np.concatenate([r for _, r in masks]) if masks else np.zeros(0, np.uint32)
    return MaskRuns(image_id, w, h, np.array([m for m, _ in masks], np.uint32), runs.astype(np.uint32), offs)


def save_maskset_runs(mr: MaskRuns, path: str) -> None:
    """providers.hpp:113-127"""
    parts = [struct.pack("<4I", MASK_MAGIC, mr.width, mr.height, mr.n_masks)]
    for j in range(mr.n_masks):
        r = mr.runs[int(mr.offsets[j]):int(mr.offsets[j + 1])].astype("<u4")
        parts.append(struct.pack("<IQ", int(mr.mask_ids[j]), r.shape[0]))
        parts.append(r.tobytes())
    Path(path).write_bytes(b"".join(parts))


def load_mask_embeddings(path: str, expected_dim: int, expected_count=None) -> np.ndarray:
    """providers.hpp:178-204"""
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise IoError(f"cannot open embedding file: {path}")
    if len(data) < 12:
        raise FormatError("unexpected end of stream")
    magic, dim, count = struct.unpack_from("<3I", data, 0)
    if magic != EMB_MAGIC:
        raise FormatError(f"bad embedding file magic: {path}")
    if dim != expected_dim:
        raise DataError(f"embedding dimension mismatch: file has {dim}, manifest expects {expected_dim}")
    if expected_count is not None and count != expected_count:
        raise DataError(f"embedding count mismatch: file has {count}, mask set has {expected_count}")
    if len(data) < 12 + 4 * dim * count:
        raise FormatError("unexpected end of stream")
    e = np.frombuffer(data, np.float32, dim * count, 12).reshape(count, dim).copy()
    bad = ~np.isfinite(e).all(axis=1)
    if bad.any():
        raise DataError(f"non-finite embedding value in record {int(np.argmax(bad))}: {path}")
    return e


def save_mask_embeddings(vectors: np.ndarray, path: str) -> None:
    """providers.hpp:158-169"""
    v = np.ascontiguousarray(vectors, "<f4")
    Path(path).write_bytes(struct.pack("<3I", EMB_MAGIC, v.shape[1], v.shape[0]) + v.tobytes())


def _parse_ply_header(f):
    """scene_io.hpp:68-128"""
    first = f.readline().rstrip(b"\r\n")
    if first != b"ply":
        raise FormatError("scene PLY: missing 'ply' magic")
    props, count, fmt_ok, in_vertex, rec = [], 0, False, False, 0
    sizes = {"float": 4, "float32": 4, "double": 8, "float64": 8, "uchar": 1, "uint8": 1, "char": 1, "int8": 1,
             "short": 2, "ushort": 2, "int16": 2, "uint16": 2, "int": 4, "uint": 4, "int32": 4, "uint32": 4}
    while True:
        line = f.readline()
        if not line:
            raise FormatError("scene PLY: truncated header")
        toks = line.decode("ascii", "replace").split()
        if not toks or toks[0] == "comment":
            continue
        if toks[0] == "format":
            if toks[1] != "binary_little_endian":
                raise FormatError(f"scene PLY: unsupported format '{toks[1]}'")
            fmt_ok = True
        elif toks[0] == "element":
            in_vertex = toks[1] == "vertex"
            if in_vertex:
                count = int(toks[2])
            elif count == 0:
                raise FormatError("scene PLY: first element must be 'vertex'")
        elif toks[0] == "property":
            if not in_vertex:
                continue
            if toks[1] not in sizes:
                raise FormatError(f"scene PLY: unsupported property type '{toks[1]}'")
            props.append((toks[2], toks[1] in ("float", "float32"), rec))
            rec += sizes[toks[1]]
        elif toks[0] == "end_header":
            break
        else:
            raise FormatError(f"scene PLY: unexpected header keyword '{toks[0]}'")
    if not fmt_ok:
        raise FormatError("scene PLY: missing format line")
    return count, rec, {n: (isf, off) for n, isf, off in props}


def load_scene_arrays(path: str):
    """scene_io.hpp:132-180 load_scene -> (mean, scale, quat_xyzw, opacity, color) arrays.

    Activation arithmetic follows the reference: scale = (float)exp((double)s),
    opacity = (float)sigmoid((double)o), color = clamp(0.5f + (float)C0 * f, 0, 1),
    quaternion divided by its float norm."""
    try:
        f = open(path, "rb")
    except OSError:
        raise IoError(f"cannot open scene file: {path}")
    with f:
        count, rec, props = _parse_ply_header(f)
        need = ["x", "y", "z", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3", "f_dc_0",
                "f_dc_1", "f_dc_2", "opacity"]
        for n in need:
            if n not in props:
                raise FormatError(f"scene PLY is missing required property '{n}'")
            if not props[n][0]:
                raise FormatError(f"scene PLY property '{n}' must be float32")
        raw = f.read(count * rec)
        if len(raw) < count * rec:
            raise FormatError(f"scene PLY: truncated at record {len(raw) // max(rec, 1)}")
    buf = np.frombuffer(raw, np.uint8).reshape(count, rec)

    def col(name):
        off = props[name][1]
        return np.ascontiguousarray(buf[:, off:off + 4]).view("<f4").reshape(count)

    mean = np.stack([col("x"), col("y"), col("z")], 1)
    # glibc exp via math.exp (numpy's vectorised exp may differ by an ulp)
    gexp = np.frompyfunc(math.exp, 1, 1)
    sraw = np.stack([col("scale_0"), col("scale_1"), col("scale_2")], 1).astype(np.float64)
    scale = gexp(sraw).astype(np.float64).astype(np.float32)
    w, x, y, z = col("rot_0"), col("rot_1"), col("rot_2"), col("rot_3")
    o = col("opacity").astype(np.float64)
    opacity = (1.0 / (1.0 + gexp(-o).astype(np.float64))).astype(np.float32)
    c0 = np.float32(SH_C0)
    color = np.clip(np.float32(0.5) + c0 * np.stack([col("f_dc_0"), col("f_dc_1"), col("f_dc_2")], 1),
                    np.float32(0), np.float32(1)).astype(np.float32)
    q = np.stack([x, y, z, w], 1).astype(np.float32)
    finite = (np.isfinite(mean).all(1) & np.isfinite(scale).all(1) & np.isfinite(color).all(1) & np.isfinite(opacity)
              & np.isfinite(q).all(1))
    if not finite.all():
        raise DataError(f"scene PLY: non-finite value at record {int(np.argmin(finite))}")
    # Quaternionf::norm(): sqrt of the 4-lane float redux (x*x + z*z) + (y*y + w*w)
    n2 = (q[:, 0] * q[:, 0] + q[:, 2] * q[:, 2]) + (q[:, 1] * q[:, 1] + q[:, 3] * q[:, 3])
    qn = np.sqrt(n2.astype(np.float32))
    if not (qn > 0).all():
        raise DataError(f"scene PLY: zero quaternion at record {int(np.argmin(qn > 0))}")
    q = (q / qn[:, None]).astype(np.float32)
    return mean.astype(np.float32), scale, q, opacity, color


def save_scene_arrays(path: str, mean, scale, quat_xyzw, opacity, color=None) -> None:
    """scene_io.hpp:184-212 save_scene (inverse activations)."""
    n = mean.shape[0]
    props = ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1",
             "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    hdr = "ply\nformat binary_little_endian 1.0\nelement vertex %d\n" % n
    hdr += "".join(f"property float {p}\n" for p in props) + "end_header\n"
    rec = np.zeros((n, 17), np.float32)
    rec[:, 0:3] = mean
    col = np.zeros((n, 3), np.float32) if color is None else np.asarray(color, np.float32)
    rec[:, 6:9] = ((col.astype(np.float32) - 0.5) / SH_C0).astype(np.float32)
    p = np.asarray(opacity, np.float64)
    with np.errstate(divide="ignore"):
        lg = np.clip(np.log(p / (1.0 - p)), -LOGIT_CLAMP, LOGIT_CLAMP)
    lg = np.where(p <= 0, -LOGIT_CLAMP, np.where(p >= 1, LOGIT_CLAMP, lg))
    rec[:, 9] = lg.astype(np.float32)
    rec[:, 10:13] = np.log(np.asarray(scale, np.float32).astype(np.float64)).astype(np.float32)
    q = np.asarray(quat_xyzw, np.float32)
    rec[:, 13] = q[:, 3]
    rec[:, 14:17] = q[:, 0:3]
    with open(path, "wb") as f:
        f.write(hdr.encode("ascii"))
        f.write(rec.astype("<f4").tobytes())


def rle_runs_from_bitmap(bits: np.ndarray) -> np.ndarray:
    """providers.hpp:77-93 rle_encode of a 0/1 bitmap (row-major), zeros first."""
    b = (np.asarray(bits).reshape(-1) != 0).astype(np.int8)
    if b.size == 0:
        return np.zeros(1, np.uint32)
    change = np.flatnonzero(np.diff(b)) + 1
    bounds = np.concatenate([[0], change, [b.size]])
    lens = np.diff(bounds).astype(np.uint32)
    if b[0] == 1:
        lens = np.concatenate([[0], lens]).astype(np.uint32)
    return lens


def ensure_dir(path: str) -> None:
    os.makedirs(path, exist_ok=True)
