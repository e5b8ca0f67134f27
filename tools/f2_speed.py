"""Row f2: exact median + below-threshold count over all 12! orderings of the
C4 group (osim_exhaustive_stats), host API wall clock."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def main():
    d = synth.c4_group()
    tot = math.factorial(12)
    _capi.exhaustive_stats(d, 2, 0.5, 0, tot, threshold=60.0)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        s, below, med = _capi.exhaustive_stats(d, 2, 0.5, 0, tot, threshold=60.0)
        ts.append(time.perf_counter() - t)
    print(f"12! + exact median + count below 60: {min(ts) * 1e3:.1f} ms (median {med!r}, below {below})")


if __name__ == "__main__":
    main()
