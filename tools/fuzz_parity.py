"""Randomized GPU-vs-oracle parity sweep over the input space the fixtures do
not enumerate: group sizes 1..12 (exhaustive, every ordering) and 1..40
(heuristic, timelines), integer / mixed / real / wide-range durations with
null stages and ties, sigma in {1, 1/2, 3/8, 0.8, 2^-k}, both DMA modes.
Every makespan, argmin, order and simulation count must match bit for bit
(sums within 1e-12).  Runs for --seconds; writes a JSON summary.

    python tools/fuzz_parity.py [--seconds 600] [--seed 1] [--out fuzz.json]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1806_10113_b200 import _capi  # noqa: E402
from paper_1806_10113_b200.heuristic import SUM_MODE  # noqa: E402

SIGMAS = (1.0, 0.5, 0.375, 0.8, 0.25, 0.125, 0.9999999999999999)


def durations(rng, n, nulls=True):
    """Random stage durations in four regimes; nulls=False keeps every stage
    non-null (the all-non-null kernels: k_exhaustive_pfx, k_heuristic_lane)."""
    mode = rng.integers(4)
    if mode == 0:
        d = rng.integers(0 if nulls else 1, 5, (n, 3)).astype(np.float64)
    elif mode == 1:
        d = np.where(rng.random((n, 3)) < 0.5, rng.integers(1, 4, (n, 3)).astype(np.float64),
                     rng.uniform(0.1, 5.0, (n, 3)))
    elif mode == 2:
        d = rng.uniform(0.01, 10.0, (n, 3))
    else:
        d = np.exp(rng.uniform(np.log(1e-6), np.log(1e8), (n, 3)))  # wide range (above 2^22 ms: general path)
    if nulls:
        d[rng.random((n, 3)) < (0.15 if mode else 0.0)] = 0.0
    empty = d.sum(axis=1) == 0.0
    d[empty, 1] = 1.0  # every task keeps a command (the reference rejects empty tasks)
    return d


def close(a, b):
    return abs(a - b) <= 1e-12 * max(abs(a), abs(b), 1e-300)


def rows_step(rng, dma, sigma, threads, stats):
    """f1: an interleaving window (T*N <= 16) and sampled label sequences (up
    to 48 tasks); f3: a batch of proxy-thread scenarios (up to 48 tasks)."""
    import ctypes as C

    T, N = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    d = durations(rng, T * N)
    total = math.factorial(T * N) // math.factorial(N) ** T
    lo = int(rng.integers(0, max(1, total - 50_000)))
    hi = min(total, lo + 50_000)
    g, _, gm = _capi.interleavings(d, T, N, dma, sigma, lo, hi, want_makespans=True)
    o, om = O.interleavings(d, T, N, dma, sigma, lo, hi, threads=threads, makespans=True)
    stats["interleavings"] += hi - lo
    if not (np.array_equal(gm.view(np.uint64), om.view(np.uint64)) and g["best_rank"] == o["best_rank"]):
        stats["mismatches"].append({"kind": "interleavings", "T": T, "N": N, "dma": dma, "sigma": sigma, "lo": lo,
                                    "durs": d.tolist()})
    T, N = int(rng.integers(1, 9)), int(rng.integers(1, 7))
    d = durations(rng, T * N)
    lab = np.stack([rng.permutation(np.repeat(np.arange(T), N)) for _ in range(256)]).astype(np.uint8)
    _, gm = _capi.eval_sequences(d, T, N, dma, sigma, lab)
    _, om = O.eval_sequences(d, T, N, dma, sigma, lab, threads=threads)
    stats["sequences"] += len(lab)
    if not np.array_equal(gm.view(np.uint64), om.view(np.uint64)):
        stats["mismatches"].append({"kind": "sequences", "T": T, "N": N, "dma": dma, "sigma": sigma,
                                    "durs": d.tolist()})
    T, N = int(rng.integers(1, 9)), int(rng.integers(1, 7))
    S = 64
    dd = np.stack([durations(rng, T * N) for _ in range(S)])
    rr = np.stack([rng.permutation(T * N) for _ in range(S)]).astype(np.uint8)
    ms, ng, sz, _, _ = _capi.harness_batch(dd, rr, T, N, dma, sigma, SUM_MODE)
    L = O.lib()
    L.oracle_harness.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int,
                                 C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    for s_ in range(S):
        om_, ong, osz = C.c_double(), C.c_int(), np.zeros(64, dtype=np.int32)
        x = np.ascontiguousarray(dd[s_])
        y = np.ascontiguousarray(rr[s_])
        rc = L.oracle_harness(x.ctypes.data_as(C.POINTER(C.c_double)), y.ctypes.data_as(C.POINTER(C.c_uint8)), T, N,
                              dma, sigma, SUM_MODE, C.byref(om_), C.byref(ong), osz.ctypes.data_as(C.POINTER(C.c_int)))
        stats["scenarios"] += 1
        if rc != 0 or ms[s_] != om_.value or sz[s_, : ng[s_]].tolist() != osz[: ong.value].tolist():
            stats["mismatches"].append({"kind": "harness", "T": T, "N": N, "dma": dma, "sigma": sigma,
                                        "durs": x.tolist(), "id_rank": y.tolist()})
            break


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default="fuzz_parity.json")
    ap.add_argument("--rows", action="store_true", help="also the f1 (interleavings, sequences) and f3 (harness) paths")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    threads = os.cpu_count() or 1
    stats = {"exhaustive_groups": 0, "exhaustive_orderings": 0, "heuristic_groups": 0, "timelines": 0,
             "interleavings": 0, "sequences": 0, "scenarios": 0, "mismatches": []}
    t_end = time.perf_counter() + a.seconds
    it = 0
    while time.perf_counter() < t_end:
        it += 1
        dma = int(rng.integers(1, 3))
        sigma = 1.0 if dma == 1 else float(SIGMAS[rng.integers(len(SIGMAS))])
        # exhaustive summary (every ordering, or a window for n >= 10)
        n = int(rng.integers(1, 13))
        d = durations(rng, n, rng.random() < 0.5)
        total = math.factorial(n)
        lo, hi = 0, total
        if n >= 10:
            lo = int(rng.integers(0, total - 200_000))
            hi = lo + 200_000
        g, gm = _capi.exhaustive(d, dma, sigma, lo, hi, want_makespans=True)
        o, om = O.exhaustive(d, dma, sigma, lo, hi, threads=threads, makespans=True)
        ok = (np.array_equal(gm.view(np.uint64), om.view(np.uint64)) and g["best"] == o["best"]
              and g["best_rank"] == o["best_rank"] and g["worst"] == o["worst"] and g["count"] == o["count"]
              and close(g["sum"], o["sum"]) and close(g["sum_log"], o["sum_log"]))
        stats["exhaustive_groups"] += 1
        stats["exhaustive_orderings"] += hi - lo
        if not ok:
            stats["mismatches"].append({"kind": "exhaustive", "n": n, "dma": dma, "sigma": sigma, "lo": lo,
                                        "durs": d.tolist()})
        # heuristic batch of one group size: up to 16 tasks (half of the batches
        # without null stages: the lane kernel), 17..40 (wide path), 65..90 (any-size path)
        u = rng.random()
        n = int(rng.integers(65, 91)) if u < 0.05 else (int(rng.integers(1, 41)) if u < 0.3 else int(rng.integers(1, 17)))
        B = 8 if n > 64 else 64
        nulls = rng.random() < 0.5
        dd = np.stack([durations(rng, n, nulls) for _ in range(B)])
        rr = np.stack([rng.permutation(n) for _ in range(B)]).astype(np.uint8)
        go, gms, gs = _capi.heuristic_batch(dd, rr.astype(np.uint32) if n > 64 else rr, dma, sigma, SUM_MODE)
        oo, oms, osims = O.reorder_batch(dd, rr, dma, sigma, SUM_MODE, threads=threads)
        stats["heuristic_groups"] += B
        if not (np.array_equal(go, oo) and np.array_equal(gms.view(np.uint64), oms.view(np.uint64))
                and np.array_equal(gs, osims)):
            bad = int(np.nonzero((go != oo).any(axis=1) | (gms != oms) | (gs != osims))[0][0])
            stats["mismatches"].append({"kind": "heuristic", "n": n, "dma": dma, "sigma": sigma,
                                        "durs": dd[bad].tolist(), "id_rank": rr[bad].tolist()})
        # one timeline (up to 300 tasks: the any-size path above 64)
        u = rng.random()
        n = int(rng.integers(65, 301)) if u < 0.05 else (int(rng.integers(1, 65)) if u < 0.25 else int(rng.integers(1, 17)))
        d = durations(rng, n)
        order = [int(x) for x in rng.permutation(n)]
        st, en, ms, idle = _capi.timeline(d, dma, sigma, order)
        r = O.simulate(d, order, dma, sigma)
        stats["timelines"] += 1
        if not (ms == r.makespan and np.array_equal(st, r.start) and np.array_equal(en, r.end)
                and idle.tolist() == r.idle.tolist()):
            stats["mismatches"].append({"kind": "timeline", "n": n, "dma": dma, "sigma": sigma, "order": order,
                                        "durs": d.tolist()})
        if a.rows:
            rows_step(rng, dma, sigma, threads, stats)
        if it % 20 == 0:
            print(it, {k: v for k, v in stats.items() if k != "mismatches"}, "mismatches", len(stats["mismatches"]),
                  flush=True)
    stats["iterations"] = it
    stats["host_threads"] = threads
    with open(a.out, "w") as fh:
        json.dump(stats, fh, indent=1)
    print("done", {k: v for k, v in stats.items() if k != "mismatches"}, "mismatches", len(stats["mismatches"]))
    sys.exit(1 if stats["mismatches"] else 0)


if __name__ == "__main__":
    main()
