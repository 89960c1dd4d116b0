"""Builds tests/cpp/_build/dropin_test (TEST INFRASTRUCTURE): the C++ drop-in
layer include/semsplat_b200/semsplat_b200.hpp exercised against the
reference's own headers (present only in the build container, compiled with
oracle/eigen_shim) and linked to libsemsplat_b200.so.  The binary travels to
the GPU box with the repo; tests/test_gpu_dropin.py runs it there."""
from __future__ import annotations

import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF_INCLUDE = Path("/root/reference/proj/include")
OUT = HERE / "_build" / "dropin_test"
BENCH = HERE / "_build" / "bench_dropin"  # bench.py's drop-in e2e leg (b200::encode_scene from disk)


def _one(src: Path, out: Path, verbose: bool) -> Path:
    hdr = ROOT / "include" / "semsplat_b200" / "semsplat_b200.hpp"
    lib = ROOT / "paper_2505_08124_b200" / "libsemsplat_b200.so"
    if out.exists() and all(p.stat().st_mtime < out.stat().st_mtime for p in (src, hdr, lib)):
        return out
    out.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-I", str(ROOT / "oracle" / "eigen_shim"), "-I", str(REF_INCLUDE), "-I",
           str(ROOT / "include"), str(src), "-o", str(out), "-L", str(lib.parent), "-lsemsplat_b200",
           "-Wl,-rpath,$ORIGIN/../../../paper_2505_08124_b200", "-lz", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return out


def build(verbose: bool = False) -> Path | None:
    if not REF_INCLUDE.exists():
        return None
    _one(HERE / "bench_dropin.cpp", BENCH, verbose)
    return _one(HERE / "dropin_test.cpp", OUT, verbose)


if __name__ == "__main__":
    print(build(verbose=True))
