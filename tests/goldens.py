"""Golden-vector loaders (tests/golden/*.npz from tests/golden/make_golden.py)."""
from pathlib import Path
from types import SimpleNamespace

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden(name):
    return np.load(GOLDEN / f"golden_{name}.npz", allow_pickle=False)


def g_scene(z, i):
    return SimpleNamespace(mean=z[f"mean_{i}"], scale=z[f"scale_{i}"], quat_xyzw=z[f"quat_{i}"],
                           opacity=z[f"opacity_{i}"], color=None)


def g_cams(z, i):
    f, R, t, wh = z[f"cam_f_{i}"], z[f"cam_R_{i}"], z[f"cam_t_{i}"], z[f"cam_wh_{i}"]
    return [SimpleNamespace(fx=f[k, 0], fy=f[k, 1], cx=f[k, 2], cy=f[k, 3], rotation=R[k].reshape(3, 3),
                            translation=t[k], width=int(wh[k, 0]), height=int(wh[k, 1]), image_id=int(wh[k, 2]))
            for k in range(f.shape[0])]


def g_masks(z, i):
    """Per view (n_masks, mw, mh, runs, run_offsets, clip) from golden_encode."""
    nm = z[f"n_masks_{i}"]
    runs, offs, clip = z[f"runs_{i}"], z[f"run_offsets_{i}"], z[f"clip_{i}"]
    mw, mh = (int(x) for x in z[f"mask_wh_{i}"])
    out, m0 = [], 0
    for n in nm:
        n = int(n)
        o = offs[m0:m0 + n + 1]
        out.append((n, mw, mh, runs, o.astype(np.uint64), clip[m0:m0 + n]))
        m0 += n
    return out


