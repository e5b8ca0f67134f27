"""Permutation search drop-in (offsim.oracle's exhaustive_search / make_report).

`exhaustive_search(tasks, profile, cap, seed)` (oracle.py:111-136):
  * n! <= cap: every ordering, in itertools.permutations order, which is
    lexicographic Lehmer-rank order -> the GPU evaluates ranks [0, n!)
    with no permutation list at all (osim_exhaustive);
  * otherwise the reference's seeded sample (oracle.py:98-108) is drawn on
    the host with the same numpy generator and the GPU evaluates that
    explicit list (osim_eval_perms).
best / argmin / worst come from the device reduction; median and geomean
are make_report's numpy expressions over the returned makespans.

The summary APIs (`exhaustive_summary*`) keep everything on the device and
return only the 48-byte reduction, for spaces too large to materialize
(12! = 479,001,600 orderings).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from itertools import permutations
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from .model import MAX_ENUM_TASKS, WIDE_MAX_TASKS, DeviceProfile, TaskSpec, resolve_group

DEFAULT_CAP = 10_000  # oracle.py:24
DEFAULT_DT = 0.001


@dataclass
class PermutationReport:
    """Makespan distribution over evaluated orderings (oracle.py:27-38)."""

    orderings: List[Tuple[str, ...]]
    makespans: List[float]
    best_ordering: Tuple[str, ...]
    best: float
    worst: float
    median: float
    geomean: float
    exhaustive: bool


def make_report(orderings: Sequence[Tuple[str, ...]], makespans: Sequence[float],
                exhaustive: bool) -> PermutationReport:
    """Reference reduction over host lists (oracle.py:41-57)."""
    ms = np.asarray(makespans, dtype=float)
    i = int(np.argmin(ms))
    return PermutationReport(
        orderings=list(orderings),
        makespans=[float(m) for m in ms],
        best_ordering=tuple(orderings[i]),
        best=float(ms.min()),
        worst=float(ms.max()),
        median=float(np.median(ms)),
        geomean=float(np.exp(np.log(ms).mean())),
        exhaustive=exhaustive,
    )


def sample_permutations(n: int, cap: int, seed: int) -> np.ndarray:
    """`cap` distinct permutations of range(n) in first-drawn order from
    numpy's default_rng(seed) (oracle.py:98-108) -> uint8 [cap][n] (uint32 above
    64 tasks, the *_u32 entry points)."""
    gen = np.random.default_rng(seed)
    kept = {}
    while len(kept) < cap:
        p = gen.permutation(n)
        key = p.tobytes()
        if key not in kept:
            kept[key] = p
    out = np.empty((cap, n), dtype=np.uint8 if n <= WIDE_MAX_TASKS else np.uint32)
    for row, p in enumerate(kept.values()):  # dicts keep insertion order
        out[row] = p
    return out


def exhaustive_search(tasks: Sequence[TaskSpec], profile: DeviceProfile, cap: int = DEFAULT_CAP,
                      seed: int = 0) -> PermutationReport:
    """Makespan distribution over all (or `cap` sampled) orderings."""
    if not tasks:
        raise ValueError("task set must be non-empty")
    if cap < 1:
        raise ValueError("cap must be at least 1")
    n = len(tasks)
    durs = resolve_group(tasks, profile)
    ids = [t.id for t in tasks]
    total = math.factorial(n)
    dma, sigma = profile.dma_engines, profile.overlap_sigma
    if total <= cap:
        if n > MAX_ENUM_TASKS:  # n! >= 3.6e14 orderings: infeasible for the reference as well
            raise NotImplementedError(f"enumerating all orderings of more than {MAX_ENUM_TASKS} tasks")
        summ, ms = _capi.exhaustive(durs, dma, sigma, 0, total, want_makespans=True)
        orderings = [tuple(ids[i] for i in p) for p in permutations(range(n))]
        exhaustive = True
    else:
        perms = sample_permutations(n, cap, seed)
        summ, ms = _capi.eval_perms(durs, dma, sigma, perms)
        orderings = [tuple(ids[i] for i in p) for p in perms.tolist()]
        exhaustive = False
    return PermutationReport(
        orderings=orderings,
        makespans=ms.tolist(),
        best_ordering=orderings[int(summ["best_rank"])],
        best=float(summ["best"]),
        worst=float(summ["worst"]),
        median=float(np.median(ms)),
        geomean=float(np.exp(np.log(ms).mean())),
        exhaustive=exhaustive,
    )


# ---- summary mode ------------------------------------------------------

@dataclass
class OrderingSummary:
    """Device-side reduction over a rank range (no per-ordering lists)."""

    best: float
    best_rank: int
    best_ordering: Tuple[int, ...]  # task indices
    worst: float
    mean: float
    geomean: float
    count: int
    sum: float
    sum_log: float


def unrank(rank: int, n: int) -> Tuple[int, ...]:
    """Lexicographic permutation of range(n) with index `rank` in
    itertools.permutations order."""
    avail = list(range(n))
    out = []
    for i in range(n - 1, -1, -1):
        f = math.factorial(i)
        d, rank = divmod(rank, f)
        out.append(avail.pop(d))
    return tuple(out)


def summary_from_dict(s: dict, n: int) -> OrderingSummary:
    c = int(s["count"])
    return OrderingSummary(
        best=float(s["best"]), best_rank=int(s["best_rank"]),
        best_ordering=unrank(int(s["best_rank"]), n) if c else (),
        worst=float(s["worst"]), mean=float(s["sum"]) / c if c else float("nan"),
        geomean=math.exp(float(s["sum_log"]) / c) if c else float("nan"), count=c,
        sum=float(s["sum"]), sum_log=float(s["sum_log"]))


def exhaustive_summary_durs(durs, dma: int, sigma: float, rank_lo: int = 0, rank_hi: Optional[int] = None,
                            n_dev: int = 1) -> OrderingSummary:
    d = np.asarray(durs, dtype=np.float64).reshape(-1, 3)
    n = d.shape[0]
    if rank_hi is None:
        rank_hi = math.factorial(n)
    s, _ = _capi.exhaustive(d, dma, sigma, rank_lo, rank_hi, n_dev=n_dev)
    return summary_from_dict(s, n)


def exhaustive_summary(tasks: Sequence[TaskSpec], profile: DeviceProfile, rank_lo: int = 0,
                       rank_hi: Optional[int] = None, n_dev: int = 1) -> OrderingSummary:
    """best / argmin / worst / mean / geomean over ranks [rank_lo, rank_hi)."""
    if not tasks:
        raise ValueError("task set must be non-empty")
    return exhaustive_summary_durs(resolve_group(tasks, profile), profile.dma_engines, profile.overlap_sigma,
                                   rank_lo, rank_hi, n_dev)


def exhaustive_summary_batch(groups, profile: DeviceProfile, n_dev: int = 1) -> np.ndarray:
    """One full-space summary per group.  `groups`: a float64 array
    [B][n][3] of stage times, or a sequence of task lists of equal size.
    Returns a structured array with _capi.SUMMARY_DTYPE fields."""
    if isinstance(groups, np.ndarray):
        d = np.ascontiguousarray(groups, dtype=np.float64)
    else:
        d = np.stack([resolve_group(g, profile) for g in groups])
    return _capi.exhaustive_batch(d, profile.dma_engines, profile.overlap_sigma, n_dev=n_dev)


# ---- full-distribution statistics ----------------

@dataclass
class OrderingStats:
    """OrderingSummary plus the exact median and the below-threshold count."""

    summary: OrderingSummary
    median: float
    below: int
    threshold: float

    @property
    def percentile(self) -> float:
        """100 * below / count, as `offsim permute` reports it (cli.py:102-103)."""
        return 100.0 * self.below / self.summary.count if self.summary.count else float("nan")


def exhaustive_stats_durs(durs, dma: int, sigma: float, threshold: float = float("-inf"), rank_lo: int = 0,
                          rank_hi: Optional[int] = None, n_dev: int = 1) -> OrderingStats:
    d = np.asarray(durs, dtype=np.float64).reshape(-1, 3)
    n = d.shape[0]
    if rank_hi is None:
        rank_hi = math.factorial(n)
    s, below, med = _capi.exhaustive_stats(d, dma, sigma, rank_lo, rank_hi, threshold, n_dev=n_dev)
    return OrderingStats(summary_from_dict(s, n), med, below, threshold)


def exhaustive_stats(tasks: Sequence[TaskSpec], profile: DeviceProfile, threshold: Optional[float] = None,
                     rank_lo: int = 0, rank_hi: Optional[int] = None, n_dev: int = 1) -> OrderingStats:
    """Median / percentile of the makespan distribution over every ordering
    without materializing it on the host (12! works)."""
    if not tasks:
        raise ValueError("task set must be non-empty")
    thr = float("-inf") if threshold is None else float(threshold)
    return exhaustive_stats_durs(resolve_group(tasks, profile), profile.dma_engines, profile.overlap_sigma, thr,
                                 rank_lo, rank_hi, n_dev)


def heuristic_percentile(tasks: Sequence[TaskSpec], profile: DeviceProfile, n_dev: int = 1):
    """The `offsim permute` figure (cli.py:96-103) over the full ordering
    space: (heuristic makespan, percentile of orderings strictly faster)."""
    from .heuristic import reorder_batch_many

    _, ms = reorder_batch_many([list(tasks)], profile, return_makespans=True)
    st = exhaustive_stats(tasks, profile, threshold=float(ms[0]), n_dev=n_dev)
    return float(ms[0]), st.percentile, st
