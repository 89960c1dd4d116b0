"""Builds libsemsplat_b200.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

Exact fp64 kernels (projection + compositor) are compiled with -fmad=false on
top of their explicit __dmul_rn/__dadd_rn arithmetic; everything else with the
default contraction.  Objects are rebuilt when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
BUILD = PKG / "_build"
LIB = PKG / "libsemsplat_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include")]
UNITS = [
    ("ss_exact.cu", ["-fmad=false"]),
    ("ss_kernels.cu", []),
    ("ss_api.cu", []),
    ("ss_query_tc.cu", []),
    ("ss_contract_tc.cu", []),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def _newest_header() -> float:
    hdrs = list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hdrs), default=0.0)


def build(verbose: bool = False, force: bool = False, defines=(), out: Path | None = None) -> Path:
    """defines/out: a variant build (extra -D flags) into out/ (its own objects and .so), for A/B timing."""
    build_dir = BUILD if out is None else Path(out)
    lib = LIB if out is None else Path(out) / LIB.name
    build_dir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    hdr_time = _newest_header()
    objs = []
    relink = force or not lib.exists()
    for src, extra in UNITS:
        s = CSRC / src
        o = build_dir / (src + ".o")
        objs.append(o)
        if force or not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, hdr_time):
            if src.endswith(".cpp"):
                cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)]
            else:
                cmd = [nvcc, *ARCH, *COMMON, *extra, *[f"-D{d}" for d in defines], "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            relink = True
    if relink or lib.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
    print(LIB)
