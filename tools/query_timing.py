"""Dev tool: time the c5 query (1024 queries x N store rows x 512, k = 10)
on the exact scan and on the tensor-core path, and check they agree bitwise."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_08124_b200._lib import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=2_000_000)
    ap.add_argument("--queries", type=int, default=1024)
    ap.add_argument("--dim", type=int, default=512)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--skip-exact", action="store_true")
    a = ap.parse_args()
    g = torch.Generator().manual_seed(5)
    raw = torch.randn(a.rows, a.dim, generator=g).numpy()
    q = torch.randn(a.queries, a.dim, generator=g).numpy()
    ctx = Context(0)
    t0 = time.time()
    cnt = ctx.store_build(raw, np.ones(a.rows, np.float32))
    print(f"store_build {cnt} rows {time.time() - t0:.2f}s", flush=True)
    res = {}
    for path in ([2] if a.skip_exact else [2, 1]):
        ctx.set_query_path(path)
        ctx.query_topk(q[:8], a.k)  # warm
        ts = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            out = ctx.query_topk(q, a.k)
            ts.append(time.perf_counter() - t)
        res[path] = out
        best = min(ts)
        print(f"path {path}: best {best * 1e3:.2f} ms  {a.queries / best:.1f} queries/s  "
              f"{2.0 * a.queries * a.rows * a.dim / best / 1e12:.1f} TFLOP/s-equivalent", flush=True)
    ctx.profile(True)
    ctx.set_query_path(2)
    ctx.profile_reset()
    ctx.query_topk(q, a.k)
    print("profile", ctx.profile_read(), flush=True)
    print("query stats", ctx.query_stats(), flush=True)
    if 1 in res:
        same = np.array_equal(res[1][0], res[2][0]) and res[1][1].tobytes() == res[2][1].tobytes()
        print("paths agree bitwise:", same, flush=True)
        if not same:
            bad = np.flatnonzero((res[1][0] != res[2][0]).any(axis=1))
            print("mismatching queries", bad[:20], len(bad))
            sys.exit(1)


if __name__ == "__main__":
    main()
