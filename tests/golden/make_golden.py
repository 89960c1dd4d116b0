"""Generates tests/golden/*.npz from the REFERENCE's own code (oracle/_ref/libssref.so:
the unmodified /root/reference headers compiled here against oracle/eigen_shim).

Run in the build container (the only place /root/reference exists):
    python tests/golden/make_golden.py
The fixtures are committed; tests/ compare the oracle and the device path to them.
"""
from __future__ import annotations

import struct
import sys
import tempfile
from decimal import Decimal, getcontext
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.bindings import Ref  # noqa: E402
from paper_2505_08124_b200 import formats  # noqa: E402
from paper_2505_08124_b200.semsplat import camera_scaled_to  # noqa: E402
from tests.util import MT19937_64, look_at, random_scene, make_test_camera, urand  # noqa: E402

OUT = Path(__file__).resolve().parent


def cam_arrays(cams):
    return {
        "cam_f": np.array([[c.fx, c.fy, c.cx, c.cy] for c in cams], np.float64),
        "cam_R": np.array([np.asarray(c.rotation, np.float64).reshape(9) for c in cams]),
        "cam_t": np.array([np.asarray(c.translation, np.float64).reshape(3) for c in cams]),
        "cam_wh": np.array([[c.width, c.height, c.image_id] for c in cams], np.uint32),
    }


def scene_arrays(s):
    return {"mean": s.mean, "scale": s.scale, "quat": s.quat_xyzw, "opacity": s.opacity}


def exp_table():
    """glibc e_exp_data.c __exp_data.tab re-derived with 80-digit arithmetic."""
    getcontext().prec = 80
    tab = []
    for k in range(128):
        v = Decimal(2) ** (Decimal(k) / Decimal(128))
        H = float(v)
        T = float(v / Decimal(H) - 1)
        hb = struct.unpack("<Q", struct.pack("<d", H))[0]
        tb = struct.unpack("<Q", struct.pack("<d", T))[0]
        tab += [tb, (hb - (k << 45)) & ((1 << 64) - 1)]
    return np.array(tab, np.uint64)


def main():
    R = Ref()

    # --- exp: table + glibc samples on the compositor's domain [-4.5, 0]
    rng = np.random.default_rng(7)
    xs = np.concatenate([-4.5 * rng.random(20000), -0.5 * np.linspace(0, 9, 5001), [0.0, -0.0, -1e-300]])
    import math
    np.savez_compressed(OUT / "golden_exp.npz", table=exp_table(), x=xs, y=np.array([math.exp(v) for v in xs]))

    # --- projection (test_projection.cpp style scenes/cameras)
    cases = [(random_scene(64, 303), make_test_camera(96, 80, 7.0, 90.0)),
             (random_scene(128, 17), make_test_camera(64, 64, 6.0)),
             (random_scene(200, 5, 3.0), look_at([2.0, 1.0, -9.0], [0.0, 0.0, 0.0], 72, 56, 60.0))]
    proj = {}
    for i, (s, c) in enumerate(cases):
        for k, v in {**scene_arrays(s), **cam_arrays([c])}.items():
            proj[f"{k}_{i}"] = v
        proj[f"projected_{i}"] = R.project(s, c)
    np.savez_compressed(OUT / "golden_project.npz", n=len(cases), **proj)

    # --- rasterizer (test_rasterizer.cpp:254-270 seeds and sizes, plus odd sizes / falloff)
    rcases = [(101, 50, (32, 32, 7.0), 0), (202, 50, (32, 32, 7.0), 0), (303, 50, (32, 32, 7.0), 0),
              (77, 64, (48, 48, 7.0), 0), (55, 70, (64, 48, 7.5), 0), (13, 40, (37, 29, 6.5), 0),
              (8, 60, (40, 56, 8.0), 1)]
    ras = {"n": len(rcases)}
    for i, (seed, n, (w, h, dist), mode) in enumerate(rcases):
        s = random_scene(n, seed)
        c = make_test_camera(w, h, dist)
        out = R.rasterize(s, c, mode=mode, full_render=True)
        for k, v in {**scene_arrays(s), **cam_arrays([c])}.items():
            ras[f"{k}_{i}"] = v
        ras[f"mode_{i}"] = np.int32(mode)
        ras[f"entries_{i}"] = out["entries"]
        ras[f"ppt_{i}"] = out["per_pixel_total"]
        ras[f"alpha_{i}"] = out["alpha"]
        ras[f"order_{i}"] = R.depth_order(s, c)
    np.savez_compressed(OUT / "golden_raster.npz", **ras)

    # --- encode: the reference's own synthetic fixtures (fixture.hpp) incl. dual resolution
    enc = {}
    fixtures = [dict(objects=3, per_object=12, views=4, resolution=32, mask_scale=1, dim=16, seed=5),
                dict(objects=2, per_object=10, views=3, resolution=24, mask_scale=2, dim=8, seed=21),
                dict(objects=5, per_object=40, views=6, resolution=64, mask_scale=1, dim=512, seed=3)]
    for i, spec in enumerate(fixtures):
        d = tempfile.mkdtemp()
        mp = R.write_fixture(d, **spec)
        man = formats.load_manifest(mp)
        mean, scale, quat, op, color = R.load_scene(man.resolve("scene.ply"))
        from types import SimpleNamespace
        sc = SimpleNamespace(mean=mean, scale=scale, quat_xyzw=quat, opacity=op)
        rows, cov, _ = R.encode(sc, mp, 1, 0)
        cams = {c.image_id: c for c in formats.load_cameras(man.resolve(man.camera_file))}
        rcams, runs, offs, nmask, clip = [], [], [0], [], []
        for e in man.images:
            c = camera_scaled_to(cams[e.camera_id], man.raster_width, man.raster_height)
            c.image_id = e.image_id
            rcams.append(c)
            mr = formats.load_maskset_runs(man.resolve(e.mask_path), e.image_id)
            emb = formats.load_mask_embeddings(man.resolve(e.embedding_path), man.embedding_dim, mr.n_masks)
            nmask.append(mr.n_masks)
            for j in range(mr.n_masks):
                r = mr.runs[int(mr.offsets[j]):int(mr.offsets[j + 1])]
                runs.append(r)
                offs.append(offs[-1] + r.shape[0])
            clip.append(emb)
        enc.update({f"{k}_{i}": v for k, v in {**scene_arrays(sc), **cam_arrays(rcams)}.items()})
        enc[f"mask_wh_{i}"] = np.array([man.mask_width, man.mask_height], np.uint32)
        enc[f"n_masks_{i}"] = np.array(nmask, np.uint32)
        enc[f"runs_{i}"] = np.concatenate(runs).astype(np.uint32)
        enc[f"run_offsets_{i}"] = np.array(offs, np.uint64)
        enc[f"clip_{i}"] = np.concatenate(clip).astype(np.float32)
        enc[f"rows_{i}"] = rows
        enc[f"coverage_{i}"] = cov
    np.savez_compressed(OUT / "golden_encode.npz", n=len(fixtures), **enc)

    # --- query (test_vecstore.cpp:144-183): 10k x 64 store, 20 queries, k = 37, tau = 0.05
    rng64 = MT19937_64(1234)
    dim, count = 64, 10000
    raw = np.array([[urand(rng64, -1, 1) for _ in range(dim)] for _ in range(count)], np.float32)
    rows = np.stack([R.normalized_copy(v) for v in raw])
    ids = np.arange(count, dtype=np.uint32)
    qr = MT19937_64(4321)
    qs = np.array([[urand(qr, -1, 1) for _ in range(dim)] for _ in range(20)], np.float32)
    tid, tsim, _ = R.query_topk(ids, rows, qs, 37)
    thr = [R.query_threshold(ids, rows, q, 0.05) for q in qs[:5]]
    np.savez_compressed(OUT / "golden_query.npz", raw=raw[:500], rows=rows, ids=ids, queries=qs, topk_ids=tid,
                        topk_sims=tsim, **{f"thr_ids_{i}": t[0] for i, t in enumerate(thr)},
                        **{f"thr_sims_{i}": t[1] for i, t in enumerate(thr)})

    # --- synth_embedding labels
    labels = ["object_0", "object_1", "bench_0_0", "bench_999_63"]
    np.savez_compressed(OUT / "golden_synth.npz", labels=np.array(labels),
                        vectors=np.stack([R.synth_embedding(l, 512) for l in labels]))
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
