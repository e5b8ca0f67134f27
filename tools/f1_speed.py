"""f1 (NoReorder interleavings) throughput vs the prefix-sharing run length.

Runs itself once per OSIM_F1_RUN value (the library reads it at first use).
"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one():
    from paper_1806_10113_b200 import _capi, synth
    d = synth.real_group("K20", 16, 41)[1]
    tot = 63_063_000
    res = {}
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        _capi.interleavings(d, 4, 4, dma, sigma, 0, tot)
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            _capi.interleavings(d, 4, 4, dma, sigma, 0, tot)
            ts.append(time.perf_counter() - t)
        res[(dma, sigma)] = tot / min(ts) / 1e9
    print(os.environ.get("OSIM_F1_RUN", "default"),
          "  ".join(f"dma{k[0]} s{k[1]}: {v:.2f} G/s" for k, v in res.items()), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        for k in (sys.argv[1:] or ["4", "8", "12", "16", "24", "32", "64"]):
            subprocess.run([sys.executable, __file__, "one"], env={**os.environ, "OSIM_F1_RUN": k}, check=True)
