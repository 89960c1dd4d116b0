#!/usr/bin/env python3
"""Throughput of the B200 embedding pass (BASELINE.json metric: views/sec and
Gaussians embedded/sec; end-to-end embed time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl b200|reference]

One step = one full embedding pass over the config's views: every rank
encodes its round-robin share of the views into its own N x 512 fp32 partial
sums, a single NCCL reduce-scatter combines them (N > 1), and each rank
normalises its shard (pipeline.hpp:280-470 + the paper's Fig. 4 combine).
`value` times that pass with all inputs resident in HBM; `e2e` times the same
pass through the C ABI with pinned host inputs (RLE mask runs, CLIP vectors,
f64 cameras) copied in every step and the finished table shard copied back.

--impl reference times the reference's own CPU encode_scene (oracle/_ref, the
unmodified headers compiled here) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
DROPIN_BENCH = ROOT / "tests" / "cpp" / "_build" / "bench_dropin"  # built where the reference headers exist
sys.path.insert(0, str(ROOT))

from harness.workload import CONFIGS, make_bench_workload, write_reference_dataset  # noqa: E402

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0


DEFAULT_LANES = 5


def ncu_traffic(kernel, field="bytes_per_launch"):
    """DRAM bytes (or another per-launch count) of `kernel` from the committed ncu capture, or None."""
    try:
        t = json.loads((Path(__file__).resolve().parent / "profiles" / "ncu_traffic.json").read_text())
        return t[kernel][field]
    except Exception:
        return None


def peaks():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--views", type=int, default=0, help="limit the view count (debug only)")
    ap.add_argument("--seed", type=int, default=2505)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-views", type=int, default=0)
    ap.add_argument("--no-query", action="store_true", help="skip the c5 vector-DB query leg")
    ap.add_argument("--lanes", type=int, default=0, help="pipeline lanes (0 = library default)")
    ap.add_argument("--group", type=int, default=0, help="views per contraction group (0 = library default)")
    ap.add_argument("--bin", type=int, default=0, help="tile binning: 0 auto, 1 key sort, 2 direct")
    ap.add_argument("--raster", type=int, default=-1, help="compositor: 2 per-step on work-stealing warps (library default), 1 per-step CTA per tile, 0 staged")
    ap.add_argument("--sort-prefix", type=int, default=-1,
                    help="SS_OPT_SORT_PREFIX (-1 = library default, 0 = full tile sorts)")
    ap.add_argument("--deterministic", action="store_true",
                    help="SS_OPT_DETERMINISTIC: fixed-point per-(Gaussian, mask) scalars (bitwise run-to-run)")
    ap.add_argument("--combine-rows", type=int, default=0,
                    help="rows per block of the block-cyclic combine (0 = contiguous shards)")
    ap.add_argument("--cpu-sample-queries", type=int, default=32)
    return ap.parse_args()


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            sm.append(s)
            mx = max(mx, m)
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------- reference arm
def cpu_reference_sample(cfg_name, seed, views, threads=None):
    """Times the reference's encode_scene (oracle/_ref) -- or, where the
    reference build is absent, the oracle port -- on `views` views of the
    config.  Returns (seconds, kind, cores, sample description, workload,
    (rows, coverage) of the reference's table for the sample)."""
    cfg = CONFIGS[cfg_name]
    threads = threads or os.cpu_count() or 1
    wl = make_bench_workload(n_gaussians=cfg["n_gaussians"], n_views=cfg["n_views"], width=cfg["width"],
                             height=cfg["height"], masks_per_view=cfg["masks_per_view"], dim=cfg["dim"], seed=seed,
                             views=list(range(views)))
    from oracle.bindings import REF_SO
    n = cfg["n_gaussians"]
    if REF_SO.exists():
        from oracle.bindings import Ref
        R = Ref()
        tmp = tempfile.mkdtemp(prefix="ssref_")
        mp = write_reference_dataset(wl, tmp)
        workers = max(1, min(threads, views))
        # phase-2 partials are workers x chunk x D f64 (pipeline.hpp:417): bound them to ~8 GB
        chunk = int(max(4096, min(n, (8 << 30) // (workers * cfg["dim"] * 8))))
        t0 = time.perf_counter()
        rows, cov, _ = R.encode(wl.scene, mp, workers, chunk)
        dt = time.perf_counter() - t0
        return dt, "reference", workers, (f"{views} of {cfg['n_views']} views of {cfg_name} through the reference "
                                          f"encode_scene (workers={workers}, chunk_rows={chunk})"), wl, (rows, cov)
    from oracle.bindings import Oracle
    O = Oracle()
    t0 = time.perf_counter()
    rows, cov = O.encode(wl.scene, wl.cams, wl.masks, cfg["dim"])
    dt = time.perf_counter() - t0
    return (dt, "port", 1, f"{views} of {cfg['n_views']} views of {cfg_name} through the C oracle (1 thread)", wl,
            (rows, cov))


PARITY_REL, PARITY_COS = 1e-4, 0.9999  # BASELINE.json north_star tolerance (per-row relative L2, cosine)


def table_parity(rows, cov, ref_rows, ref_cov):
    """Per-row relative L2 and cosine of the device table against the
    reference's (oracles.hpp:129-160 definitions), over covered rows; the
    covered sets must be identical."""
    cg, ce = cov > np.float32(1e-8), ref_cov > np.float32(1e-8)
    out = {"max_row_rel": 0.0, "min_cos": 1.0, "covered_equal": bool(np.array_equal(cg, ce)),
           "covered_rows": int(ce.sum()), "uncovered_rows_zero": bool(not rows[~cg].any())}
    for lo in range(0, rows.shape[0], 1 << 18):
        sl = slice(lo, lo + (1 << 18))
        m = ce[sl]
        if not m.any():
            continue
        e = ref_rows[sl][m].astype(np.float64)
        g = rows[sl][m].astype(np.float64)
        den = np.sqrt((e * e).sum(1))
        rel = np.sqrt(((e - g) ** 2).sum(1)) / np.where(den > 0, den, 1.0)
        cos = (e * g).sum(1) / np.maximum(np.sqrt((e * e).sum(1) * (g * g).sum(1)), 1e-300)
        out["max_row_rel"] = max(out["max_row_rel"], float(rel.max()))
        out["min_cos"] = min(out["min_cos"], float(cos.min()))
    out["ok"] = bool(out["covered_equal"] and out["uncovered_rows_zero"] and out["max_row_rel"] <= PARITY_REL
                     and out["min_cos"] >= PARITY_COS)
    out["tolerance"] = {"max_row_rel": PARITY_REL, "min_cos": PARITY_COS}
    return out


def query_leg(ctx, args, dev, stream, want_cpu):
    """configs[4]: 1024 queries x 2M 512-d unit rows, top-10, through the
    public query call (host queries in, host ids/sims out).  Device-side
    kernel times come from CUDA events on the call's stream."""
    import torch
    from harness.workload import QUERY_CONFIG as QC
    n, nq, d, k = QC["n_rows"], QC["n_queries"], QC["dim"], QC["k"]
    from harness.workload import query_workload
    t_gen = time.perf_counter()
    raw, qraw = query_workload(args.seed, n, nq, d)  # cmd_bench's store + queries (main.cpp:440-450)
    gen_s = time.perf_counter() - t_gen
    queries = torch.from_numpy(qraw.copy())
    q_pinned = queries.pin_memory().numpy()
    cnt = ctx.store_build(raw, np.ones(n, np.float32))  # normalized_copy per row on the device
    del raw
    ctx.query_topk(q_pinned[:8], k)  # warm: fp16 copy of the store, kernel attributes
    for _ in range(args.warmup):
        ctx.query_topk(q_pinned, k)
    times = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ids, sims, _ = ctx.query_topk(q_pinned, k)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.median(times))
    ctx.profile_reset()
    ctx.profile(True)
    ctx.query_topk(q_pinned, k)
    ctx.profile(False)
    prof = ctx.profile_read()
    gemm, sel, tot = prof["query_gemm"], prof["query_select"], prof["query"]
    try:
        p = json.loads(PEAKS_FILE.read_text())
        tpeak, src = float(p["bf16_tflops"]), "bf16_tflops burst (MEASURED_PEAKS.json; fp16 runs at the bf16 rate)"
    except Exception:
        tpeak, src = 2250.0, "nominal dense fp16 (fallback)"
    achieved = gemm["bytes"] / (gemm["ms"] / 1e3) / 1e12 if gemm["ms"] > 0 else None
    # threshold mode of cmd_bench: tau so that a random query returns about k rows
    frac = min(0.5, k / float(cnt))
    z = 1.0
    for _ in range(40):
        z -= (math.erfc(z) - 2.0 * frac) / (-2.0 / math.sqrt(math.pi) * math.exp(-z * z))
    tau = float(np.float32(math.sqrt(2.0) * z / math.sqrt(float(d))))
    n_thr = min(nq, 64)
    ctx.query_threshold(q_pinned[0], tau)
    t0 = time.perf_counter()
    returned = 0
    thr_results = []
    for i in range(n_thr):
        ti, ts = ctx.query_threshold(q_pinned[i], tau)
        returned += len(ti)
        thr_results.append((ti, ts))
    thr_ms = 1e3 * (time.perf_counter() - t0) / n_thr
    out = {
        "workload": f"{QC['name']}: {nq} queries x {cnt} unit rows x {d}, top-{k} "
                    f"(cmd_bench generator, seed {args.seed} ^ 0xbe9c)",
        "dataset_gen_seconds": gen_s,
        "threshold": {"tau": tau, "ms_per_query_e2e": thr_ms, "queries": n_thr,
                      "avg_returned": returned / n_thr},
        "metric": "queries_per_sec", "unit": "queries/s", "value_e2e": nq / (ms / 1e3), "ms_per_batch_e2e": ms,
        "ms_device_query": tot["ms"], "value_device": nq / (tot["ms"] / 1e3) if tot["ms"] > 0 else None,
        "h2d_bytes_per_batch": int(nq * d * 4), "d2h_bytes_per_batch": int(nq * k * 8),
        "kernels": {"query_gemm_ms": gemm["ms"], "query_select_ms": sel["ms"],
                    "other_ms": tot["ms"] - gemm["ms"] - sel["ms"]},
        "roofline": {"bound": "tensor", "kernel": "coarse_scores_kernel (tcgen05 kind::f16)", "achieved": achieved,
                     "peak": tpeak, "unit": "TFLOP/s", "frac": achieved / tpeak if achieved else None,
                     "traffic": ncu_traffic("query_gemm"), "peak_source": src, "flops_per_launch": gemm["bytes"]},
        "data": "synthetic: U(-0.5,0.5)^512 rows and queries from std::mt19937_64 as in cmd_bench, normalised "
                "by store_build / prepare_query",
    }
    if want_cpu:
        try:
            from oracle.bindings import REF_SO
            ns = max(1, args.cpu_sample_queries)
            store_ids, store_rows = ctx.store_fetch()
            qs = queries[:ns].numpy()
            cores = os.cpu_count() or 1
            if REF_SO.exists():
                from oracle.bindings import Ref
                R, kind = Ref(), "reference"
            else:
                from oracle.bindings import Oracle
                R, kind = Oracle(), "port"
            t0 = time.perf_counter()
            ri, rs, _ = R.query_topk(store_ids, store_rows, qs, k, threads=cores)
            dt = time.perf_counter() - t0
            # threshold mode on the reference (single-threaded, as the reference API is)
            nt = min(4, n_thr)
            t1 = time.perf_counter()
            thr_ok = True
            for i in range(nt):
                rti, rts = R.query_threshold(store_ids, store_rows, qs[i] if i < ns else queries[i].numpy(), tau)
                gi, gs = thr_results[i]
                thr_ok = thr_ok and np.array_equal(rti, gi) and rts.tobytes() == gs.tobytes()
            out["threshold"]["cpu_baseline"] = {"value": 1e3 * (time.perf_counter() - t1) / nt,
                                                "unit": "ms/query", "cores": 1, "kind": kind,
                                                "sample": f"{nt} threshold queries over the full store"}
            out["threshold"]["parity_sample"] = bool(thr_ok)
            out["cpu_baseline"] = {"value": ns / dt, "unit": "queries/s", "cores": cores, "kind": kind,
                                   "sample": f"{ns} of the {nq} queries over the full store, threads={cores}",
                                   "seconds": dt}
            out["parity_sample"] = bool(np.array_equal(ri, ids[:ns]) and rs.tobytes() == sims[:ns].tobytes())
        except Exception as ex:
            out["cpu_baseline"] = {"value": None, "unit": "queries/s", "cores": None, "kind": "unavailable",
                                   "sample": str(ex)}
    return out


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    # inputs from the oracle-side build of the harness generator: this process
    # maps oracle/ libraries only, never libsemsplat_b200.so
    from harness import workload
    from oracle.build_oracle import GEN_SO
    workload.use_generator(GEN_SO)
    cfg = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    views = args.cpu_sample_views or max(1, min(cores, 16))
    times = []
    for i in range(args.warmup + args.steps):
        dt, kind, used, sample, _, _ = cpu_reference_sample(args.config, args.seed, views, cores)
        if i >= args.warmup:
            times.append(dt)
    sec = float(np.mean(times))
    v = views / sec
    print(json.dumps({
        "impl": "reference", "metric": "views_per_sec", "value": v, "unit": "views/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "gaussians_embedded_per_sec": cfg["n_gaussians"] * v / cfg["n_views"],
        "config": {"workload": f"{args.config}: {cfg['n_gaussians']} Gaussians, {cfg['n_views']} views "
                               f"{cfg['width']}x{cfg['height']}, {cfg['masks_per_view']} masks/view, D={cfg['dim']}",
                   "sample_views": views},
        "cpu_baseline": {"value": v, "unit": "views/s", "cores": used, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- B200 arm
def relaunch_under_torchrun(n: int) -> None:
    """`bench.py --gpus N` (N > 1) outside a launcher: re-exec as N ranks, one
    process per GPU, exactly as the driver launches it."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)", file=sys.stderr)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2505_08124_b200._lib import Context

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    n_views = args.views or cfg["n_views"]
    mine = [v for v in range(n_views) if v % world == rank]
    t_gen = time.perf_counter()
    wl = make_bench_workload(n_gaussians=cfg["n_gaussians"], n_views=cfg["n_views"], width=cfg["width"],
                             height=cfg["height"], masks_per_view=cfg["masks_per_view"], dim=cfg["dim"],
                             seed=args.seed, views=mine)
    gen_s = time.perf_counter() - t_gen
    N, D = cfg["n_gaussians"], cfg["dim"]

    ctx = Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    ctx.set_scene(wl.scene.mean, wl.scene.scale, wl.scene.quat_xyzw, wl.scene.opacity)
    if world > 1:
        # the library's own NCCL communicator (the combine is one grouped
        # reduce-scatter issued by libsemsplat_b200, not by torch)
        uid = [Context.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(world, rank, uid[0])
    ctx.set_combine_rows(args.combine_rows)
    lanes = args.lanes or DEFAULT_LANES
    ctx.set_lanes(lanes)
    if args.group:
        ctx.set_contract_group(args.group)
    if args.bin:
        ctx.set_bin_path(args.bin)
    if args.raster >= 0:
        ctx.set_raster_algo(args.raster)
    if args.deterministic:
        ctx.set_deterministic(True)
    if args.sort_prefix >= 0:
        ctx.set_sort_prefix(args.sort_prefix)

    # device-resident inputs for `value`
    dev = torch.device("cuda", local)
    runs_all = np.concatenate([m[3] for m in wl.masks]).astype(np.uint32)
    offs_abs, base = [], 0
    for m in wl.masks:
        offs_abs.append(m[4].astype(np.int64) + base)
        base += int(m[4][-1])
    d_runs = torch.from_numpy(runs_all.view(np.int32)).to(dev)
    d_offs = [torch.from_numpy(o).to(dev) for o in offs_abs]
    d_clip = [torch.from_numpy(np.ascontiguousarray(m[5], np.float32)).to(dev) for m in wl.masks]
    dev_masks = [(m[0], m[1], m[2], d_runs.data_ptr(), o.data_ptr(), c.data_ptr(), int(m[4][-1] - m[4][0]))
                 for m, o, c in zip(wl.masks, d_offs, d_clip)]
    lay = ctx.combine_layout()
    shard = lay["rank_rows"]  # rows this rank receives (block-cyclic rounds; padding included)
    sums = torch.zeros((lay["rows_alloc"], D), dtype=torch.float32, device=dev)
    totals = torch.zeros((lay["rows_alloc"],), dtype=torch.float32, device=dev)
    rows_out = torch.empty((shard, D), dtype=torch.float32, device=dev)
    cov_out = torch.empty((shard,), dtype=torch.float32, device=dev)
    held = ctx.combine_rows_of(lay)
    n_local = int((held < N).sum())  # real table rows this rank finalises

    def combine_and_normalize():
        # combine_partials + finalize_into: one grouped NCCL reduce-scatter per
        # round (sums and totals), then the shard's normalisation
        ctx.combine_device(rows_out.data_ptr(), cov_out.data_ptr())

    def step_device():
        ctx.encode_begin(D, sums.data_ptr(), totals.data_ptr())
        ctx.encode_views_device(wl.cams, dev_masks)
        combine_and_normalize()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def timed(fn, k):
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = torch.tensor([a.elapsed_time(b)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item()) / k

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    ctx.profile_reset()  # zeroes the launch and geometry counters too
    with ClockSampler(local) as clk:
        ms_step = timed(step_device, args.steps)
    counters = ctx.counters()
    own, cub = ctx.launch_count()

    # ---- e2e: pinned host inputs through the C ABI, table shard back to host
    e2e = None
    if not args.no_e2e:
        pin_masks, h2d = [], 0
        for m in wl.masks:
            r = torch.from_numpy(m[3].view(np.int32)).pin_memory().numpy().view(np.uint32)
            o = torch.from_numpy(m[4].view(np.int64)).pin_memory().numpy().view(np.uint64)
            c = torch.from_numpy(np.ascontiguousarray(m[5], np.float32)).pin_memory().numpy()
            pin_masks.append((m[0], m[1], m[2], r, o, c))
            h2d += r.nbytes + o.nbytes + c.nbytes + 128
        host_rows = torch.empty((shard, D), dtype=torch.float32).pin_memory()
        host_cov = torch.empty((shard,), dtype=torch.float32).pin_memory()

        def step_e2e():
            ctx.encode_begin(D, sums.data_ptr(), totals.data_ptr())
            ctx.encode_views(wl.cams, pin_masks)
            combine_and_normalize()
            host_rows.copy_(rows_out, non_blocking=True)
            host_cov.copy_(cov_out, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        step_e2e()
        e2e_ms = timed(step_e2e, args.steps)
        e2e = {"value": n_views / (e2e_ms / 1e3), "unit": "views/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(host_rows.numel() * 4 + host_cov.numel() * 4), "ms_per_step": e2e_ms}

    # ---- per-kernel attribution: one extra pass with the two lanes serialised
    # so every kernel class is timed exclusively (CUDA events on its stream)
    ctx.set_lanes(1)
    ctx.profile_reset()
    ctx.profile(True)
    ms_prof = timed(step_device, 1)
    ctx.profile(False)
    prof = ctx.profile_read()
    ctx.set_lanes(lanes)
    hbm, peak_kind = peaks()
    kernels = {}
    for k, v in prof.items():
        if v["launches"] and v["ms"] > 0 and not k.startswith("query"):
            kernels[k] = {"ms_per_step": v["ms"], "launches_per_step": v["launches"], "gb_per_step": v["bytes"] / 1e9,
                          "achieved_gbs": v["bytes"] / (v["ms"] / 1e3) / 1e9 if k != "h2d" else None,
                          "share_of_serial_step": v["ms"] / ms_prof}
            # measured DRAM traffic of the class per view (committed ncu capture, c4) beside the algorithmic bytes
            dv = ncu_traffic(k, "bytes_per_view") if args.config == "c4" else None
            if dv:
                kernels[k]["dram_gb_per_view_ncu"] = dv / 1e9
                kernels[k]["algorithmic_gb_per_view"] = v["bytes"] / 1e9 / n_views
    dom = max((k for k in kernels if k not in ("h2d",)), key=lambda k: kernels[k]["ms_per_step"])
    dk = kernels[dom]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": dk["achieved_gbs"], "peak": hbm, "unit": "GB/s",
                "frac": dk["achieved_gbs"] / hbm, "traffic": ncu_traffic(dom),
                "algorithmic_bytes_per_launch": dk["gb_per_step"] * 1e9 / max(dk["launches_per_step"], 1), "peak_source": f"{peak_kind} (MEASURED_PEAKS.json)",
                "share_of_step": dk["share_of_serial_step"],
                "timing": "CUDA events around each launch on its stream, one extra pass with lanes serialised"}
    # the compositor is bound by the fp64 pipe, not HBM; its fp64
    # operation count per c4 launch comes from the committed ncu capture, the
    # peak from a DFMA probe run here
    roofline_fp64 = None
    ops = ncu_traffic(dom, "fp64_ops_per_launch") if args.config == "c4" else None
    if ops:
        t_launch = dk["ms_per_step"] / max(dk["launches_per_step"], 1) / 1e3
        peak64 = ctx.probe_fp64_rate()
        roofline_fp64 = {"bound": "fp64", "kernel": dom, "achieved": ops / t_launch / 1e12, "peak": peak64 / 1e12,
                         "unit": "T fp64 lane-ops/s (DADD, DMUL, DFMA: one each)",
                         "frac": ops / t_launch / peak64, "ops_per_launch": ops,
                         "ops_source": "profiles/ncu_traffic.json (smsp__sass_thread_inst_executed_op_d{add,mul,fma})",
                         "peak_source": "ss_probe_fp64_rate: eight DFMA chains per thread on every SM, this run"}
    # the compositor's binding resource is instruction issue (ncu: IPC ~2.5-2.9
    # of 4, fp64 pipe ~34 % busy): warp instructions per launch from the
    # committed capture over the launch time, against 4 issue slots per SM per
    # clock at the sampled SM clock
    roofline_issue = None
    winst = ncu_traffic(dom, "warp_inst_per_launch") if args.config == "c4" else None
    if winst:
        t_launch = dk["ms_per_step"] / max(dk["launches_per_step"], 1) / 1e3
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        mhz = (clk.summary() or {}).get("sm_mhz") or 1965.0
        peak_issue = 4.0 * sms * mhz * 1e6
        roofline_issue = {"bound": "issue", "kernel": dom, "achieved": winst / t_launch / 1e12,
                          "peak": peak_issue / 1e12, "unit": "T warp-instructions/s", "frac": winst / t_launch / peak_issue,
                          "inst_per_launch": winst,
                          "inst_source": "profiles/ncu_traffic.json (smsp__inst_executed.sum of the committed capture)",
                          "peak_source": f"4 issue slots x {sms} SMs x {mhz:.0f} MHz (sampled SM clock)"}
    steps = 1
    pass_bytes = sum(v["bytes"] for k, v in prof.items() if k not in ("h2d", "query"))

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sample = args.cpu_sample_views or max(1, min(os.cpu_count() or 1, 16))
            dt, kind, cores, desc, swl, (er, ec) = cpu_reference_sample(args.config, args.seed, sample)
            cpu = {"value": sample / dt, "unit": "views/s", "cores": cores, "kind": kind, "sample": desc,
                   "seconds": dt}
            # parity at the benchmarked configuration: the same sample views
            # through the device pass (context-owned accumulators, same C ABI)
            ctx.encode_begin(D)
            ctx.encode_views(swl.cams, swl.masks)
            prow, pcov = ctx.encode_finalize()
            parity = table_parity(prow, pcov, er, ec)
            parity["sample"] = f"views 0..{sample - 1} of {args.config} vs the {kind} encode_scene table"
            del prow, pcov, er, ec
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": "views/s", "cores": None, "kind": "unavailable", "sample": str(ex)}

    # drop-in e2e leg: the whole c4 dataset in the reference's on-disk formats
    # (scene PLY, manifest, cameras, per-view RLE masks and CLIP files), run by
    # tests/cpp/_build/bench_dropin through b200::encode_scene -- the call a
    # reference user makes -- with file parsing and the host table included
    e2e_dropin = None
    if rank == 0 and world == 1 and not args.no_e2e and DROPIN_BENCH.exists():
        try:
            from paper_2505_08124_b200 import formats
            tmp = tempfile.mkdtemp(prefix="ss_dropin_")
            mp = write_reference_dataset(wl, tmp)
            sp = os.path.join(tmp, "scene.ply")
            s_ = wl.scene
            formats.save_scene_arrays(sp, s_.mean, s_.scale, s_.quat_xyzw, s_.opacity, s_.color)
            env = dict(os.environ, CUDA_VISIBLE_DEVICES=str(local))
            r = subprocess.run([str(DROPIN_BENCH), sp, mp, "1", "0", "3"], capture_output=True, text=True,
                               timeout=900, env=env)
            if r.returncode == 0:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                e2e_dropin = {"value": d["views"] / d["seconds"], "unit": "views/s",
                              "value_without_parse": d["views"] / d["encode_seconds"], **d,
                              "path": "b200::encode_scene (C++ drop-in) on the on-disk dataset: load_scene + "
                                      "load_manifest, per-view mask/CLIP files read inside encode_scene, "
                                      "table in host memory; best of 3 runs"}
            else:
                e2e_dropin = {"error": (r.stdout + r.stderr)[-400:]}
            shutil.rmtree(tmp, ignore_errors=True)
        except Exception as ex:  # reported, not fatal
            e2e_dropin = {"error": f"{type(ex).__name__}: {ex}"}

    # eval leg (eval.hpp:122-158): arg-max class per covered row of the table
    # shard just produced (device-resident), 16 synthetic class embeddings
    evl = None
    if rank == 0 and not args.no_query:
        try:
            from harness.workload import synth_embedding
            lab_ids = np.arange(16, dtype=np.int32)
            lab_vecs = np.stack([synth_embedding(f"class_{i}", D) for i in range(16)])
            ctx.assign_classes_device(rows_out.data_ptr(), cov_out.data_ptr(), n_local, D, lab_ids, lab_vecs)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cls = ctx.assign_classes_device(rows_out.data_ptr(), cov_out.data_ptr(), n_local, D, lab_ids, lab_vecs)
            dt = time.perf_counter() - t0
            evl = {"function": "assign_classes (eval.hpp:122-158)", "rows": int(n_local), "labels": 16,
                   "covered": int((cls >= 0).sum()), "ms": 1e3 * dt, "rows_per_sec": n_local / dt}
            if world == 1 and not args.no_cpu_baseline:
                from oracle.bindings import REF_SO
                if REF_SO.exists():
                    from oracle.bindings import Ref
                    ns = 20000
                    hr = rows_out[:ns].cpu().numpy()
                    hc = cov_out[:ns].cpu().numpy()
                    t1 = time.perf_counter()
                    rc = Ref().assign_classes(hr, hc, lab_ids, lab_vecs)
                    dt1 = time.perf_counter() - t1
                    evl["cpu_baseline"] = {"value": ns / dt1, "unit": "rows/s", "cores": 1, "kind": "reference",
                                           "sample": f"first {ns} rows of the table"}
                    evl["parity_sample"] = bool(np.array_equal(rc, cls[:ns]))
        except Exception as ex:  # reported, not fatal
            evl = {"error": f"{type(ex).__name__}: {ex}"}

    query = None
    if rank == 0 and not args.no_query:
        try:
            query = query_leg(ctx, args, dev, stream, want_cpu=world == 1 and not args.no_cpu_baseline)
        except Exception as ex:  # reported, not fatal
            query = {"error": f"{type(ex).__name__}: {ex}"}

    value = n_views / (ms_step / 1e3)
    if rank == 0:
        line = {
            "metric": "views_per_sec", "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic (bench-style scene, orbit cameras, random "
                                                              "rectangle RLE masks, synth_embedding CLIP)",
            "gaussians_embedded_per_sec": N * value / n_views,
            "gaussian_views_per_sec": N * value,
            "embed_seconds": ms_step / 1e3,
            "config": {"workload": f"{args.config}: {N} Gaussians, {n_views} views {cfg['width']}x{cfg['height']}, "
                                   f"{cfg['masks_per_view']} masks/view, D={D}",
                       "parallelism": f"views round-robin over {world} GPU(s); combine = the library's NCCL "
                                      f"reduce-scatter of the N x D sums and N totals (one group per round, "
                                      f"{lay['rounds']} round(s) of {lay['block_rows']} rows per rank), then "
                                      f"per-rank normalisation of {n_local} rows",
                       "nccl": {"nranks": world, "communicator": "libsemsplat_b200 (ss_comm_init)"} if world > 1
                       else None,
                       "l2": "inputs larger than L2 (N x 512 fp32 sums = %.1f GB RMW per pass)" % (N * D * 4 / 1e9),
                       "dataset_gen_seconds": gen_s,
                       "scalars": "u64 fixed point (SS_OPT_DETERMINISTIC: bitwise run-to-run)" if args.deterministic
                       else "f32 atomics (library default)"},
            "roofline": roofline,
            "roofline_fp64": roofline_fp64,
            "roofline_issue": roofline_issue,
            "pass_algorithmic_gb": pass_bytes / 1e9,
            "pass_hbm_frac": pass_bytes / (ms_step / 1e3) / 1e9 / hbm,
            "kernels": kernels,
            "geometry_per_view": {k: counters[k] / max(counters["views"], 1) for k in
                                  ("n_vis", "instances", "touched", "pairs")},
            "e2e": e2e,
            "e2e_dropin": e2e_dropin,
            "cpu_baseline": cpu,
            "parity": parity,
            "clocks": clk.summary(),
            "gpu_launches": int((own + cub) / max(args.steps, 1)),
            "gpu_launches_detail": {"own_per_step": own / max(args.steps, 1), "cub_per_step": cub / max(args.steps, 1)},
            "serial_profile_ms_per_step": ms_prof,
            "query": query,
            "eval": evl,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    if parity is not None and not parity["ok"]:
        # loud: the bench configuration does not match the reference
        print(f"PARITY FAILURE at {args.config}: {json.dumps(parity)}", file=sys.stderr, flush=True)
        sys.exit(3)


if __name__ == "__main__":
    main()
