"""Test helpers: the reference test suite's fixtures (tests/helpers.hpp) in Python."""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np

_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (pure Python; for small test scenes only)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64


def urand(rng: MT19937_64, lo: float, hi: float) -> float:
    """helpers.hpp:12-14"""
    return lo + (hi - lo) * ((float(rng() >> 11) + 0.5) * 2.0 ** -53)


def random_scene(n: int, seed: int, extent: float = 2.0):
    """helpers.hpp:16-37 random_scene.  Argument evaluation inside the
    reference's Eigen constructors is compiler-ordered; here draws are taken
    in source order (the scene only needs to be identical for both paths)."""
    rng = MT19937_64(seed)
    mean = np.zeros((n, 3), np.float32)
    scale = np.zeros((n, 3), np.float32)
    quat = np.zeros((n, 4), np.float32)
    op = np.zeros(n, np.float32)
    color = np.zeros((n, 3), np.float32)
    for k in range(n):
        mean[k] = [urand(rng, -extent, extent) for _ in range(3)]
        scale[k] = [urand(rng, 0.05, 0.4) for _ in range(3)]
        w, x, y, z = (urand(rng, -1, 1) for _ in range(4))
        n2 = (x * x + z * z) + (y * y + w * w)
        s = n2 ** 0.5
        quat[k] = [x / s, y / s, z / s, w / s]
        op[k] = urand(rng, 0.05, 0.95)
        color[k] = [urand(rng, 0, 1) for _ in range(3)]
    return SimpleNamespace(mean=mean, scale=scale, quat_xyzw=quat, opacity=op, color=color)


def scene_ns(mean, scale, quat, opacity, color=None):
    return SimpleNamespace(mean=np.asarray(mean, np.float32), scale=np.asarray(scale, np.float32),
                           quat_xyzw=np.asarray(quat, np.float32), opacity=np.asarray(opacity, np.float32),
                           color=None if color is None else np.asarray(color, np.float32))


def plain_camera(fx, fy, cx, cy, w, h, image_id=0):
    return SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, rotation=np.eye(3), translation=np.zeros(3), width=w,
                           height=h, image_id=image_id)


def look_at(eye, target, w, h, focal, image_id=0):
    """fixture.hpp:65-84 with the shim's vector arithmetic (same as ss_synth_look_at)."""
    def norm(v):
        n = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]
        s = n ** 0.5
        return [v[0] / s, v[1] / s, v[2] / s] if n > 0 else v

    def cross(a, b):
        return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]

    fwd = norm([target[i] - eye[i] for i in range(3)])
    up = [0.0, 1.0, 0.0]
    if abs((fwd[0] * up[0] + fwd[1] * up[1]) + fwd[2] * up[2]) > 0.99:
        up = [1.0, 0.0, 0.0]
    right = norm(cross(fwd, up))
    down = cross(fwd, right)
    R = np.array([right, down, fwd], np.float64)
    t = np.array([-(R[i, 0] * eye[0] + (R[i, 1] * eye[1] + R[i, 2] * eye[2])) for i in range(3)], np.float64)
    return SimpleNamespace(fx=focal, fy=focal, cx=w / 2.0, cy=h / 2.0, rotation=R, translation=t, width=w, height=h,
                           image_id=image_id)


def make_test_camera(w, h, distance=8.0, focal=0.0, image_id=0):
    """helpers.hpp:40-47"""
    if focal <= 0:
        focal = 0.9 * w
    return look_at([0.0, 0.0, -distance], [0.0, 0.0, 0.0], w, h, focal, image_id)


def rect_mask_runs(w, h, rects):
    """RLE runs (zeros first) of the union of axis-aligned inclusive rectangles."""
    from paper_2505_08124_b200.formats import rle_runs_from_bitmap
    bits = np.zeros((h, w), np.uint8)
    for (x0, y0, x1, y1) in rects:
        bits[y0:y1 + 1, x0:x1 + 1] = 1
    return rle_runs_from_bitmap(bits), bits.reshape(-1)
