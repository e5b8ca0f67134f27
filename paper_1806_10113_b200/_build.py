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
SOURCES = [os.path.join(CSRC, f) for f in (
    "osim_capi.cu", "osim_exh_d2s1.cu", "osim_exh_d2s0.cu", "osim_exh_d1.cu",
    "osim_batch_d2.cu", "osim_batch_d1.cu", "osim_heur.cu", "osim_null.cu", "osim_wide.cu",
    "osim_big.cu")]
HEADERS = [os.path.join(CSRC, f) for f in (
    "osim_sim.cuh", "osim_kernels.cuh", "osim_launch.cuh", "osim_deps.cuh", "osim_micro.cuh", "osim_harness.cuh", "osim_exh_impl.cuh", "osim_batch_impl.cuh", "osim_suftab.h", "osim_null.cuh", "osim_wide.cuh", "osim_heur_null.cuh", "osim_big.cuh", "osim_heur_lane.cuh")] + [
    os.path.join(ROOT, "include", "offsim_b200.h")
]
OBJDIR = os.path.join(PKG, "build")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC",
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


def _compile(src: str, objdir: str, verbose: bool) -> str:
    obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
    extra = os.environ.get("OSIM_NVCC_EXTRA", "").split()  # tuning only, e.g. -DOSIM_PFX_MINB=3
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", obj, src]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False, verbose: bool = False, jobs: int = 0) -> str:
    """Compile the translation units in parallel, link the shared library."""
    if not force and not stale():
        return LIB
    return _build_to(LIB, OBJDIR, verbose, jobs)


def build_variant(name: str, extra: list, verbose: bool = False) -> str:
    """A/B tuning build: liboffsim_b200_<name>.so with extra nvcc flags
    (e.g. -DOSIM_HSPLIT=0); load it with OSIM_LIB=<path>."""
    out = os.path.join(PKG, f"liboffsim_b200_{name}.so")
    os.environ["OSIM_NVCC_EXTRA"] = " ".join(extra)
    return _build_to(out, OBJDIR + "_" + name, verbose, 0)


def _build_to(lib: str, objdir: str, verbose: bool, jobs: int) -> str:
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(objdir, exist_ok=True)
    jobs = jobs or min(len(SOURCES), os.cpu_count() or 1)
    with ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, objdir, verbose), SOURCES))
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib + ".tmp", *objs]
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:], verbose=True))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
