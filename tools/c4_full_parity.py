"""Every makespan of the C4 headline space (all 12! = 479,001,600 orderings)
bit-exact against the pinned CPU oracle, for 2-DMA sigma 0.5 / 0.375 and
1-DMA, compared window by window (10^7 ranks at a time); plus the summary
fields.  Writes a JSON summary (argv[1])."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def main(out_path):
    d = synth.c4_group()
    total = math.factorial(12)
    W = 10_000_000
    threads = os.cpu_count() or 1
    res = {"orderings": total, "window": W, "host_threads": threads, "configs": {}}
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        t0 = time.perf_counter()
        mism = 0
        for lo in range(0, total, W):
            hi = min(lo + W, total)
            _, g = _capi.exhaustive(d, dma, sigma, lo, hi, want_makespans=True)
            _, o = O.exhaustive(d, dma, sigma, lo, hi, threads=threads, makespans=True)
            mism += int(np.count_nonzero(g.view(np.uint64) != o.view(np.uint64)))
        s, _ = _capi.exhaustive(d, dma, sigma, 0, total)
        res["configs"][f"{dma}dma_sigma{sigma}"] = {
            "mismatching_makespans": mism, "best": s["best"], "best_rank": s["best_rank"], "worst": s["worst"],
            "seconds": time.perf_counter() - t0}
        print(dma, sigma, res["configs"][f"{dma}dma_sigma{sigma}"], flush=True)
        assert mism == 0
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c4_full_parity.json")
