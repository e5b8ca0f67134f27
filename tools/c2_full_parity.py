"""Whole config-2 batch parity: all 10^5 8-task groups x 8! orderings on the
GPU (osim_exhaustive_batch) vs the pinned CPU oracle per group (best,
argmin, worst, count bit-exact; sum and sum of logs within 1e-12 relative).
~6 min of oracle time on 16 host threads.  Writes a JSON summary (argv[1])."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


from oracle import oracle as O  # noqa: E402
from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def main(out_path):
    B = 100_000
    threads = os.cpu_count() or 1
    d = synth.c2_batch(B)
    res = {"groups": B, "orderings_per_group": 40320, "host_threads": threads, "modes": {}}
    for dma, sigma in ((2, 0.5), (1, 1.0)):
        t = time.perf_counter()
        out = _capi.exhaustive_batch(d, dma, sigma)
        tg = time.perf_counter() - t
        t = time.perf_counter()
        bad, worst_rel = 0, 0.0
        for b in range(B):
            o, _ = O.exhaustive(d[b], dma, sigma, threads=threads)
            g = out[b]
            ok = (g["best"] == o["best"] and g["best_rank"] == o["best_rank"] and g["worst"] == o["worst"]
                  and g["count"] == o["count"])
            rel = max(abs(g["sum"] - o["sum"]) / abs(o["sum"]), abs(g["sum_log"] - o["sum_log"]) / abs(o["sum_log"]))
            worst_rel = max(worst_rel, float(rel))
            bad += 0 if (ok and rel <= 1e-12) else 1
        tc = time.perf_counter() - t
        res["modes"][f"{dma}dma_sigma{sigma}"] = {"mismatching_groups": bad, "max_rel_sum_diff": worst_rel,
                                                  "gpu_host_api_s": tg, "cpu_oracle_s": tc}
        print(dma, sigma, res["modes"][f"{dma}dma_sigma{sigma}"], flush=True)
        assert bad == 0
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c2_full_parity.json")
