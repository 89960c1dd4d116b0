"""Builds harness/libss_synth.so, the synthetic-input generator of the bench
and the tests (BENCH/TEST HARNESS: not part of the product library)."""
from __future__ import annotations

import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "ss_synth.cpp"
LIB = HERE / "libss_synth.so"


def compile_generator(out: Path, verbose: bool = False) -> Path:
    deps = [SRC, HERE / "ss_synth.h"]
    if out.exists() and all(d.stat().st_mtime <= out.stat().st_mtime for d in deps):
        return out
    cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-shared", str(SRC), "-o", str(out)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return out


def build(verbose: bool = False) -> Path:
    return compile_generator(LIB, verbose)


if __name__ == "__main__":
    print(build(verbose=True))
