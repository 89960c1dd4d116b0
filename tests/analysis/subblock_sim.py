"""Compositor scheduling model (analysis only; DESIGN.md §7 item 1).

Counts, for sampled c4 tiles, how many warp steps the compositor's warp
schedule takes: a warp owns an 8x4 pixel block and steps through every splat
whose padded box touches the block (in depth order) while any of its pixels
is live, stopping when all 32 have saturated (T < 1e-4).  It compares that
with warps whose GWxGH sub-blocks walk their own hit lists, either fully
independently or synchronised at every 32-entry staging chunk.

The per-pixel arithmetic is a float64 numpy model of rasterizer.hpp:112-133
(exact enough to place early termination); the projection comes from the
CPU oracle.  Usage: python tests/analysis/subblock_sim.py [--tiles 40] [--view 0]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle.bindings import Oracle  # noqa: E402
from harness.workload import orbit_camera, synth_scene  # noqa: E402

W, H = 1152, 864


def splats(view):
    s = synth_scene(2_000_000, 1, 5.0)
    p = Oracle().project(s, orbit_camera(view, 1000, W, H))
    vis = p["visible"].astype(bool)
    mx, my, cxx, cxy, cyy, z = (p[k][vis] for k in ("mu_x", "mu_y", "cov_xx", "cov_xy", "cov_yy", "depth"))
    det = cxx * cyy - cxy * cxy
    rx, ry = 3 * np.sqrt(cxx) + 1, 3 * np.sqrt(cyy) + 1
    box = (np.maximum(np.ceil(mx - rx), 0), np.minimum(np.floor(mx + rx), W - 1),
           np.maximum(np.ceil(my - ry), 0), np.minimum(np.floor(my + ry), H - 1))
    keep = (box[0] <= box[1]) & (box[2] <= box[3])
    order = np.lexsort((np.nonzero(vis)[0], z))
    return dict(mx=mx, my=my, a=cyy / det, b2=-2 * cxy / det, c=cxx / det, op=s.opacity[vis].astype(np.float64),
                box=box, order=order[keep[order]])


def simulate(sp, tiles, shapes):
    x0, x1, y0, y1 = sp["box"]
    order = sp["order"]
    lanes = np.arange(32)
    cur = 0
    ind = {s: 0 for s in shapes}
    chk = {s: 0 for s in shapes}
    for t in tiles:
        X0, Y0 = (t % 72) * 16, (t // 72) * 16
        sel = order[(x1[order] >= X0) & (x0[order] <= X0 + 15) & (y1[order] >= Y0) & (y0[order] <= Y0 + 15)]
        for w in range(8):
            px = X0 + 8 * (w & 1) + (lanes & 7)
            py = Y0 + 4 * (w >> 1) + (lanes >> 3)
            grp = {(gw, gh): (lanes & 7) // gw + (8 // gw) * ((lanes >> 3) // gh) for gw, gh in shapes}
            tot = {s: np.zeros(32 // (s[0] * s[1]), int) for s in shapes}
            chunk = {s: np.zeros(32 // (s[0] * s[1]), int) for s in shapes}
            T = np.ones(32)
            done = np.zeros(32, bool)
            for idx, g in enumerate(sel):
                if idx % 32 == 0:
                    for s in shapes:
                        chk[s] += chunk[s].max()
                        chunk[s][:] = 0
                m = (px >= x0[g]) & (px <= x1[g]) & (py >= y0[g]) & (py <= y1[g]) & ~done
                if not m.any():
                    continue
                cur += 1
                for s in shapes:
                    hit = np.bincount(grp[s][m], minlength=len(tot[s])) > 0
                    tot[s] += hit
                    chunk[s] += hit
                dx, dy = px - sp["mx"][g], py - sp["my"][g]
                d2 = sp["a"][g] * dx * dx + sp["b2"][g] * dx * dy + sp["c"][g] * dy * dy
                al = np.minimum(0.99, sp["op"][g] * np.exp(-0.5 * d2))
                ok = m & (d2 <= 9) & (al >= 1 / 255)
                T = np.where(ok, T * (1 - al), T)
                done |= ok & (T < 1e-4)
                if done.all():
                    break
            for s in shapes:
                ind[s] += tot[s].max()
                chk[s] += chunk[s].max()
    return cur, ind, chk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=40)
    ap.add_argument("--view", type=int, default=0)
    a = ap.parse_args()
    sp = splats(a.view)
    tiles = np.random.default_rng(0).choice(72 * 54, a.tiles, replace=False)
    shapes = [(8, 2), (4, 4), (4, 2), (2, 2), (1, 1)]
    cur, ind, chk = simulate(sp, tiles, shapes)
    print(f"8x4-block warp steps: {cur}")
    for s in shapes:
        print(f"{s[0]}x{s[1]} sub-blocks: independent {ind[s] / cur:.3f}x, chunk-synchronous {chk[s] / cur:.3f}x")


if __name__ == "__main__":
    main()
