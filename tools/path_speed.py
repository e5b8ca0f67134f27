"""Throughput of the secondary (non-benchmark) paths through the host API."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

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
    h, r = synth.c5_batch_fast("nvidia", 100_000)
    hn = h.copy()
    hn[:, 5, 2] = 0.0
    t = best(lambda: _capi.heuristic_batch(hn, r, 2, 0.5, 1))
    print(f"heuristic, null stages (general kernel): {1e5 / t / 1e6:.1f} M decisions/s")
    t = best(lambda: _capi.heuristic_batch(h, r, 2, 0.5, 1))
    print(f"heuristic, fast kernel (same batch): {1e5 / t / 1e6:.1f} M decisions/s")
    d1 = synth.real_group("K20", 12, 41)[1]
    t = best(lambda: _capi.interleavings(d1, 4, 3, 1, 1.0, 0, 369600))
    print(f"f1 1-DMA waves (k_interleave_pfx1): {369600 / t / 1e9:.3f} G interleavings/s")
    t = best(lambda: _capi.interleavings(d1, 4, 3, 2, 0.5, 0, 369600))
    print(f"f1 2-DMA (k_interleave_pfx): {369600 / t / 1e9:.3f} G interleavings/s")
    d4 = synth.c4_group()
    perms = np.stack([np.random.default_rng(i).permutation(12) for i in range(200_000)]).astype(np.uint8)
    t = best(lambda: _capi.eval_perms(d4, 2, 0.5, perms))
    print(f"sampled mode eval_perms: {2e5 / t / 1e6:.1f} M orderings/s (host API, 2.4 MB H2D)")


if __name__ == "__main__":
    main()
