"""Wall-clock C4 / C3 / C2 / C5 under the current environment (used with
OSIM_CTAS_PER_SM / OSIM_PFX_L sweeps; one line per config)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def best_of(f, k=5):
    f()
    ts = []
    for _ in range(k):
        t = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t)
    return min(ts)


def main():
    d4, d3 = synth.c4_group(), synth.c3_group()
    c2 = synth.c2_batch(100_000)
    h, r = synth.c5_batch_fast("nvidia", 1_000_000)
    t4 = best_of(lambda: _capi.exhaustive(d4, 2, 0.5, 0, 479001600))
    t48 = best_of(lambda: _capi.exhaustive(d4, 2, 0.5, 0, 479001600 // 8))
    t3 = best_of(lambda: _capi.exhaustive(d3, 2, 0.5, 0, 3628800), 20)
    t2 = best_of(lambda: _capi.exhaustive_batch(c2, 2, 0.5), 3)
    t5 = best_of(lambda: _capi.heuristic_batch(h, r, 2, 0.5, 1), 3)
    print(f"env={os.environ.get('OSIM_CTAS_PER_SM', '-')} c4 {479001600 / t4 / 1e9:.2f}G/s ({t4 * 1e3:.2f} ms) "
          f"c4/8-shard {479001600 / 8 / t48 / 1e9:.2f}G/s c3 {3628800 / t3 / 1e9:.2f}G/s c2 {4.032e9 / t2 / 1e9:.2f}G/s c5 {1e6 / t5 / 1e6:.1f}M/s", flush=True)


if __name__ == "__main__":
    main()
