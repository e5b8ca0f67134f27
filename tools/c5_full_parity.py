"""Whole config-5 batch parity: all 10^6 16-task groups per device profile
through the GPU heuristic vs the pinned CPU oracle (order, makespan and
simulation count bit-exact).  Writes a JSON summary (argv[1])."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1806_10113_b200 import _capi, synth  # noqa: E402
from paper_1806_10113_b200.heuristic import SUM_MODE  # noqa: E402


def main(out_path):
    B = 1_000_000
    threads = os.cpu_count() or 1
    res = {"groups_per_profile": B, "host_threads": threads, "sum_mode": SUM_MODE,
           "inputs": "config 5 exactly: group b = sample_real_tasks(dev, 16, seed=b), b in [0, 10^6) (synth.c5_batch)",
           "profiles": {}}
    for prof, (_, dma, sigma) in synth.PROFILES.items():
        d, r = synth.c5_batch(prof, B, start=0, workers=min(threads, 32))
        t = time.perf_counter()
        order, ms, sims = _capi.heuristic_batch(d, r, dma, sigma, SUM_MODE)
        tg = time.perf_counter() - t
        t = time.perf_counter()
        oo, om, osims = O.reorder_batch(d, r, dma, sigma, SUM_MODE, threads=threads)
        tc = time.perf_counter() - t
        bad = int(np.count_nonzero((order != oo).any(axis=1) | (ms != om) | (sims != osims)))
        res["profiles"][prof] = {"mismatching_groups": bad, "gpu_host_api_s": tg, "cpu_oracle_s": tc}
        print(prof, res["profiles"][prof], flush=True)
        assert bad == 0
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c5_full_parity.json")
