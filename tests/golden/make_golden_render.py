"""Generates tests/golden/golden_render.npz from the REFERENCE's own
rasterize (rasterizer.hpp:261-264, RenderResult: image, weights, alpha) via
oracle/_ref/libssref.so.  Run in the build container:
    python tests/golden/make_golden_render.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.bindings import Ref  # noqa: E402
from tests.golden.make_golden import cam_arrays, scene_arrays  # noqa: E402
from tests.util import make_test_camera, random_scene  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    R = Ref()
    cases = [(11, 400, 64, 48, 7.0, 0), (12, 300, 80, 56, 6.0, 1), (13, 900, 96, 96, 9.0, 0)]
    out = {}
    for i, (seed, n, w, h, dist, mode) in enumerate(cases):
        s = random_scene(n, seed)
        cam = make_test_camera(w, h, dist)
        r = R.rasterize(s, cam, mode, full_render=True)
        for k, v in scene_arrays(s).items():
            out[f"{k}_{i}"] = v
        out[f"color_{i}"] = s.color
        for k, v in cam_arrays([cam]).items():
            out[f"{k}_{i}"] = v
        out[f"mode_{i}"] = np.int32(mode)
        out[f"image_{i}"] = r["image"]
        out[f"alpha_{i}"] = r["alpha"]
        out[f"ppt_{i}"] = r["per_pixel_total"]
        out[f"entries_{i}"] = r["entries"]
    np.savez_compressed(OUT / "golden_render.npz", n=len(cases), **out)


if __name__ == "__main__":
    main()
