"""General-path speed probe: the C4 group with one null stage, and scaled out
of the fast range (both run k_exhaustive_gen: one thread per ordering from
time 0, IEEE division)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def rate(d, count=20_000_000):
    _capi.exhaustive(d, 2, 0.5, 0, 1_000_000)
    t = time.perf_counter()
    _capi.exhaustive(d, 2, 0.5, 0, count)
    return count / (time.perf_counter() - t)


def main():
    d = synth.c4_group().copy()
    d[3, 0] = 0.0  # one null HtD
    assert not _capi.fast_eligible(d, 0.5)
    print(f"general path, C4 with a null stage: {rate(d) / 1e9:.2f} G orderings/s")
    d2 = synth.c4_group() * 1e23  # out of the fast range
    print(f"general path, C4 scaled by 1e23: {rate(d2) / 1e9:.2f} G orderings/s")


if __name__ == "__main__":
    main()
