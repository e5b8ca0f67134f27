"""Lane-slot utilization of the exhaustive prefix kernel's phase-B replays
(C4, C3 and a C2 slice, 2-DMA, sigma 0.5).  Needs the counters compiled in:
    OSIM_NVCC_EXTRA=-DOSIM_HSTATS python -m paper_1806_10113_b200._build --force
"""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def main():
    L = _capi.load()
    L.osim_hstats_exh.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    L.osim_hstats_batch.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * 8)()
    runs = (("C4", L.osim_hstats_exh, lambda: _capi.exhaustive(synth.c4_group(), 2, 0.5, 0, math.factorial(12) // 8)),
            ("C3", L.osim_hstats_exh, lambda: _capi.exhaustive(synth.c3_group(), 2, 0.5, 0, math.factorial(10))),
            ("C2", L.osim_hstats_batch, lambda: _capi.exhaustive_batch(synth.c2_batch(2000), 2, 0.5)))
    for name, rd, f in runs:
        rd(buf, 1)
        f()
        rd(buf, 1)
        a = list(buf)
        print(f"{name}: useful/slots {a[1] / a[0]:.3f}, empty lanes {a[4] / a[0]:.3f}, "
              f"full-step slots {a[2] / a[0]:.3f} (own HtD running {a[3] / a[0]:.3f}), "
              f"mean warp replay {a[6] / a[5]:.2f} steps, mean full-step phase {a[7] / a[5]:.2f}")


if __name__ == "__main__":
    main()
