"""Synthetic task groups for the benchmark configs (BASELINE.json configs 1-5).

Restates the reference's input generators as float64 arrays instead of
TaskSpec lists (workload.py:35-179): the Table-2 synthetic tasks, the five
BK compositions, and the per-device kernel envelopes that
`sample_real_tasks` draws from with numpy's default_rng -- so a group
generated here is bit-identical to the reference's for the same seed
(tests/test_host.py pins this against the reference-generated fixtures).
"""

from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

TIME_UNIT_MS = 10.0

# Table 2 of the paper: (htd, k, dth) as fractions of 10 ms (workload.py:38-47)
TABLE2: Dict[str, Tuple[float, float, float]] = {
    "T0": (0.1, 0.8, 0.1),
    "T1": (0.2, 0.7, 0.1),
    "T2": (0.3, 0.6, 0.1),
    "T3": (0.1, 0.7, 0.2),
    "T4": (0.6, 0.2, 0.2),
    "T5": (0.2, 0.2, 0.6),
    "T6": (0.4, 0.2, 0.4),
    "T7": (0.8, 0.1, 0.1),
}

BK: Dict[str, Tuple[str, ...]] = {  # workload.py:49-55
    "BK0": ("T6", "T7", "T4", "T5"),
    "BK25": ("T0", "T4", "T6", "T7"),
    "BK50": ("T0", "T1", "T4", "T5"),
    "BK75": ("T0", "T1", "T2", "T4"),
    "BK100": ("T0", "T1", "T2", "T3"),
}

# Measured (min, max) ms envelopes per device and kernel, (htd, k, dth)
# (workload.py:61-92; Table 4 of the paper).
REAL_TASK_RANGES: Dict[str, Dict[str, Tuple[Tuple[float, float], ...]]] = {
    "AMD": {
        "MM": ((0.97, 2.57), (1.80, 9.02), (0.14, 1.18)),
        "BS": ((0.08, 1.29), (2.98, 5.57), (0.16, 2.17)),
        "FWT": ((1.29, 2.57), (2.59, 5.47), (1.18, 2.35)),
        "FLW": ((0.05, 0.07), (7.77, 10.08), (0.09, 0.16)),
        "CONV": ((0.09, 0.37), (1.51, 14.58), (0.09, 0.37)),
        "VA": ((0.65, 3.86), (0.05, 0.30), (0.30, 1.81)),
        "TM": ((2.57, 5.15), (0.29, 3.59), (2.36, 4.70)),
        "DCT": ((2.57, 5.15), (0.95, 1.89), (2.35, 4.71)),
    },
    "PHI": {
        "MM": ((0.36, 0.90), (4.98, 5.03), (0.09, 0.16)),
        "BS": ((0.17, 0.63), (5.25, 12.03), (0.33, 1.24)),
        "FWT": ((0.67, 1.26), (4.59, 6.39), (0.61, 1.21)),
        "FLW": ((0.03, 0.06), (1.12, 9.05), (0.06, 0.12)),
        "CONV": ((0.06, 0.17), (0.56, 10.09), (0.17, 10.09)),
        "VA": ((1.27, 7.46), (0.18, 1.18), (0.61, 3.68)),
        "TM": ((2.58, 4.98), (1.09, 2.36), (2.54, 4.93)),
        "DCT": ((1.71, 2.25), (6.97, 9.41), (1.67, 2.18)),
    },
    "K20": {
        "MM": ((2.51, 3.77), (3.99, 7.95), (1.24, 2.49)),
        "BS": ((0.31, 1.25), (1.25, 9.26), (0.62, 2.50)),
        "FWT": ((1.25, 5.01), (1.20, 4.94), (1.25, 4.98)),
        "FLW": ((0.01, 0.31), (1.32, 9.25), (0.03, 0.63)),
        "CONV": ((0.63, 2.53), (1.47, 9.20), (0.62, 2.50)),
        "VA": ((2.51, 12.54), (0.09, 0.44), (1.25, 6.19)),
        "TM": ((2.60, 5.01), (0.41, 2.61), (2.60, 4.96)),
        "DCT": ((2.51, 5.01), (1.55, 3.08), (2.48, 4.96)),
    },
}

# Device-style profiles of config 5: (envelope device, dma engines, sigma)
PROFILES = {
    "nvidia": ("K20", 2, 0.5),
    "amd": ("AMD", 2, 0.375),
    "phi": ("PHI", 1, 1.0),
}


def table2_durations() -> np.ndarray:
    return np.array([[f * TIME_UNIT_MS for f in TABLE2[k]] for k in sorted(TABLE2)], dtype=np.float64)


def bk_group(name: str) -> Tuple[List[str], np.ndarray]:
    ids = list(BK[name])
    return ids, np.array([[f * TIME_UNIT_MS for f in TABLE2[i]] for i in ids], dtype=np.float64)


def real_group(device: str, count: int, seed: int) -> Tuple[List[str], np.ndarray]:
    """Same draws as workload.sample_real_tasks(device, count, seed)
    (workload.py:152-179): per task a kernel uniformly, then each stage
    uniformly in its envelope; ids "<KERNEL>-i"."""
    ranges = REAL_TASK_RANGES[device]
    kernels = sorted(ranges)
    gen = np.random.default_rng(seed)
    ids, rows = [], []
    for i in range(count):
        name = kernels[int(gen.integers(len(kernels)))]
        (h0, h1), (k0, k1), (d0, d1) = ranges[name]
        rows.append((float(gen.uniform(h0, h1)), float(gen.uniform(k0, k1)), float(gen.uniform(d0, d1))))
        ids.append(f"{name}-{i}")
    return ids, np.array(rows, dtype=np.float64)


def id_rank_of(ids: List[str]) -> np.ndarray:
    order = sorted(range(len(ids)), key=lambda i: ids[i])
    r = np.empty(len(ids), dtype=np.uint8)
    r[order] = np.arange(len(ids), dtype=np.uint8)
    return r


C2_SEED = 18061011302


def c2_batch(count: int = 100_000) -> np.ndarray:
    """Config 2: Table-2 tasks x U(0.5, 1.5) per stage, [count][8][3]
    (BASELINE.md, C2 row)."""
    base = table2_durations()
    gen = np.random.default_rng(C2_SEED)
    return np.ascontiguousarray((base[None] * gen.uniform(0.5, 1.5, (100_000, 8, 3)))[:count])


def c3_group() -> np.ndarray:
    return real_group("K20", 10, 10)[1]


def c4_group() -> np.ndarray:
    return real_group("AMD", 12, 12)[1]


def c5_batch(profile: str, count: int, start: int = 0, workers: int = 1) -> Tuple[np.ndarray, np.ndarray]:
    """Config 5: group b = sample_real_tasks(dev, 16, seed=b).  One
    generator per group (~0.2 ms each), so large batches can be drawn by
    `workers` processes over contiguous seed ranges."""
    if workers > 1 and count >= 4 * workers:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor

        cuts = [count * i // workers for i in range(workers + 1)]
        with ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn")) as ex:
            parts = list(ex.map(c5_batch, [profile] * workers, [cuts[i + 1] - cuts[i] for i in range(workers)],
                                [start + cuts[i] for i in range(workers)]))
        return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])
    dev = PROFILES[profile][0]
    d = np.empty((count, 16, 3))
    r = np.empty((count, 16), dtype=np.uint8)
    for j in range(count):
        ids, rows = real_group(dev, 16, start + j)
        d[j] = rows
        r[j] = id_rank_of(ids)
    return d, r


_STR_RANK = {s: r for r, s in enumerate(sorted(str(i) for i in range(16)))}


def c5_batch_fast(profile: str, count: int, seed: int = 1806) -> Tuple[np.ndarray, np.ndarray]:
    """Config-5-shaped batch for the benchmark: the same envelopes, kernel
    mix and "<KERNEL>-i" id order as c5_batch, drawn from ONE generator
    stream (vectorized) instead of one default_rng(b) per group, so 10^6
    groups take a fraction of a second to synthesize.  Parity tests use
    c5_batch's exact per-seed groups."""
    dev = PROFILES[profile][0]
    ranges = REAL_TASK_RANGES[dev]
    kernels = sorted(ranges)
    lo = np.array([[ranges[k][s][0] for s in range(3)] for k in kernels])
    hi = np.array([[ranges[k][s][1] for s in range(3)] for k in kernels])
    gen = np.random.default_rng(seed)
    kid = gen.integers(len(kernels), size=(count, 16))
    u = gen.random((count, 16, 3))
    d = lo[kid] + u * (hi[kid] - lo[kid])
    # id "<KERNEL>-i" string order: kernel name first, then str(i)
    pos = np.array([_STR_RANK[str(i)] for i in range(16)])
    key = kid * 16 + pos[None, :]
    order = np.argsort(key, axis=1, kind="stable")
    r = np.empty((count, 16), dtype=np.uint8)
    np.put_along_axis(r, order, np.arange(16, dtype=np.uint8)[None, :].repeat(count, 0), axis=1)
    return np.ascontiguousarray(d), r
