"""Builds the parity checkers -- TEST INFRASTRUCTURE ONLY.

  oracle/libssoracle.so   the C restatement (oracle/ssoracle.c)
  oracle/libssgen.so      the synthetic-input generator (harness/ss_synth.cpp),
                          a second build used only by bench.py's reference
                          arm so that process never maps the product library
  oracle/_ref/libssref.so the UNMODIFIED reference headers
                          (/root/reference/proj/include, only present in the
                          build container) + oracle/eigen_shim + ref_capi.cpp

Both are built with the reference's own flags (-O3, baseline x86-64, no FMA:
proj/CMakeLists.txt:11).  On the GPU box /root/reference is absent and the
prebuilt .so files that travelled with the repo are used as-is.
"""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_INCLUDE = Path("/root/reference/proj/include")
ORACLE_SO = HERE / "libssoracle.so"
GEN_SO = HERE / "libssgen.so"
REF_SO = HERE / "_ref" / "libssref.so"


def _stale(out: Path, srcs) -> bool:
    return not out.exists() or any(s.stat().st_mtime > out.stat().st_mtime for s in srcs)


def build(verbose: bool = False) -> None:
    src = HERE / "ssoracle.c"
    if _stale(ORACLE_SO, [src]):
        cmd = ["gcc", "-O3", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", str(src), "-o", str(ORACLE_SO),
               "-lm", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    sys.path.insert(0, str(HERE.parent))
    from harness.build import compile_generator
    compile_generator(GEN_SO, verbose)
    if REF_INCLUDE.exists():
        REF_SO.parent.mkdir(exist_ok=True)
        deps = [HERE / "ref_capi.cpp", HERE / "eigen_shim" / "Eigen" / "Dense", HERE / "eigen_shim" / "Eigen" / "Geometry",
                *REF_INCLUDE.glob("semsplat/*.hpp")]
        if _stale(REF_SO, deps):
            cmd = ["g++", "-std=c++20", "-O3", "-fPIC", "-shared", "-I", str(HERE / "eigen_shim"), "-I",
                   str(REF_INCLUDE), str(HERE / "ref_capi.cpp"), "-o", str(REF_SO), "-lz", "-lpthread"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)


if __name__ == "__main__":
    build(verbose=True)
    print(ORACLE_SO, REF_SO if REF_SO.exists() else "(reference headers absent; _ref not built)", file=sys.stderr)
