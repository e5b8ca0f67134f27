"""Short single-GPU workloads for ncu captures (one launch of each kernel).

    python tools/profile_run.py c4|c3|c2|c5|f1|all
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def main(which):
    _capi.set_device(0)
    if which in ("c4", "all"):
        s, _ = _capi.exhaustive(synth.c4_group(), 2, 0.5, 0, 479001600)
        print("c4", s)
    if which in ("c3", "all"):
        s, _ = _capi.exhaustive(synth.c3_group(), 2, 0.5, 0, 3628800)
        print("c3", s)
    if which in ("c2", "all"):
        out = _capi.exhaustive_batch(synth.c2_batch(20000), 2, 0.5)
        print("c2", out[0])
    if which in ("c5", "all"):
        d, r = synth.c5_batch_fast("nvidia", 200_000)
        o, m, n = _capi.heuristic_batch(d, r, 2, 0.5, 1)
        print("c5", o[0], m[0], n[0])
    if which in ("f1", "all"):
        d = synth.real_group("K20", 16, 41)[1]
        for dma, sigma in ((2, 0.5), (1, 1.0)):
            s, _, _ = _capi.interleavings(d, 4, 4, dma, sigma, 0, 63_063_000)
            print("f1", dma, s)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
