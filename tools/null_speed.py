"""Batch and heuristic throughput with null stages (general kernels) next to
the all-non-null fast kernels, same shapes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def best(f, k=3):
    f()
    ts = []
    for _ in range(k):
        t = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t)
    return min(ts)


def main():
    d2 = synth.c2_batch(20_000)
    dn = d2.copy()
    dn[:, 3, 0] = 0.0  # task 3 of every group: no HtD
    for name, d in (("c2 batch", d2), ("c2 batch, null HtD", dn)):
        t = best(lambda: _capi.exhaustive_batch(d, 2, 0.5))
        print(f"{name}: {20_000 * 40320 / t / 1e9:.2f} G orderings/s")
    h, r = synth.c5_batch_fast("nvidia", 200_000)
    hn = h.copy()
    hn[:, 5, 2] = 0.0  # task 5: no DtH
    for name, d in (("c5 heuristic", h), ("c5 heuristic, null DtH", hn)):
        t = best(lambda: _capi.heuristic_batch(d, r, 2, 0.5, 1))
        print(f"{name}: {200_000 / t / 1e6:.1f} M decisions/s (host API)")


if __name__ == "__main__":
    main()
