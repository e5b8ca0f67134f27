"""Lane-slot utilization of the C5 heuristic kernel's candidate replays.

Needs a build with the counters compiled in:
    OSIM_NVCC_EXTRA=-DOSIM_HSTATS python -m paper_1806_10113_b200._build --force
    python tools/heur_lanes.py

slots = 32 lanes x warp replay length summed over item iterations; useful =
steps a lane's own candidate needs; empty = lanes without an item (partial
fill); full-step slots = slots spent in the full-step phase (while any lane
of the warp still has its candidate's HtD running) vs the steps in which a
lane's own HtD is actually running.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def main():
    L = _capi.load()
    L.osim_hstats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    for prof in ("nvidia", "amd", "phi"):
        _, dma, sigma = synth.PROFILES[prof]
        d, r = synth.c5_batch_fast(prof, 100_000)
        buf = (C.c_ulonglong * 8)()
        L.osim_hstats(buf, 1)
        _capi.heuristic_batch(d, r, dma, sigma, 1)
        L.osim_hstats(buf, 1)
        a = list(buf)
        print(f"{prof}: useful/slots {a[1] / a[0]:.3f}, empty lanes {a[4] / a[0]:.3f}, "
              f"full-step slots {a[2] / a[0]:.3f} (own HtD running {a[3] / a[0]:.3f}), "
              f"mean warp replay {a[6] / a[5]:.2f} steps, mean full-step phase {a[7] / a[5]:.2f}")


if __name__ == "__main__":
    main()
