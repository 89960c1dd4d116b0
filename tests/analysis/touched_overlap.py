"""Dev experiment: overlap of the touched-Gaussian sets (nonzero masked weight)
of nearby c4 views -- what batching views in the contraction would save."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle.bindings import Oracle  # noqa: E402  (decoder for the experiment only)
from paper_2505_08124_b200._lib import Context  # noqa: E402
from harness.workload import CONFIGS, make_bench_workload  # noqa: E402

cfg = CONFIGS["c4"]
views = list(range(8))
wl = make_bench_workload(n_gaussians=cfg["n_gaussians"], n_views=cfg["n_views"], width=cfg["width"],
                         height=cfg["height"], masks_per_view=cfg["masks_per_view"], dim=8, seed=2505, views=views)
O = Oracle()
ctx = Context(0)
ctx.set_scene(wl.scene.mean, wl.scene.scale, wl.scene.quat_xyzw, wl.scene.opacity)
sets = []
for v, cam in enumerate(wl.cams):
    m = wl.masks[v]
    n_masks, mw, mh, runs, offs = m[0], m[1], m[2], m[3], m[4]
    covered = np.zeros(mw * mh, bool)
    for j in range(n_masks):
        covered |= O.rle_decode(runs[offs[j]:offs[j + 1]], mw, mh).reshape(-1).astype(bool)
    e = ctx.raster_capture(cam)["entries"]
    sel = covered[e["pixel"]]
    s = np.unique(e["gaussian_id"][sel])
    sets.append(s)
    print(f"view {v}: entries {len(e)}, touched {len(s)}", flush=True)
for K in (2, 4, 8):
    tot = sum(len(sets[i]) for i in range(K))
    uni = len(np.unique(np.concatenate(sets[:K])))
    print(f"K={K}: sum {tot}, union {uni}, union/sum {uni / tot:.3f}")
for gap in (1, 4):
    inter = [len(np.intersect1d(sets[i], sets[i + gap])) / len(sets[i]) for i in range(len(sets) - gap)]
    print(f"gap {gap}: mean |A&B|/|A| = {np.mean(inter):.3f}")
