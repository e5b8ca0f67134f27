"""Build recipe for liboffsim_b200.so (sm_100a, in-tree).

`python -m paper_1806_10113_b200._build` or __graft_entry__.build().  The
library is linked against the static CUDA runtime, so it needs only the
driver at run time.  -fmad=false forbids FMA contraction (the reference
rounds every multiply and add separately); the kernels additionally use
explicit round-to-nearest intrinsics on every operation of the event loop.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liboffsim_b200.so")
SOURCES = [os.path.join(CSRC, "osim_capi.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("osim_sim.cuh", "osim_kernels.cuh")] + [
    os.path.join(ROOT, "include", "offsim_b200.h")
]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
