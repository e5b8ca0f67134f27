"""Batch Reordering heuristic drop-in (offsim.heuristic, Algorithm 1).

`reorder_batch` / `reorder_batch_many` run the whole algorithm
(heuristic.py:105-125) on the GPU: the first pick, every greedy round's
candidate simulations and completion estimates, the final-pair rule and
the makespan of the result (osim_heuristic_batch).  Ties are broken
exactly like the reference: by Python string order of task ids, by
builtin sum()'s rounding (Neumaier on CPython >= 3.12, naive before; the
mode follows the running interpreter) and by the rt iteration order.

The step functions `select_first_task`, `select_next_task` and
`select_last_tasks` keep the reference's signatures; their candidate
simulations go through the GPU `simulate`.
"""

from __future__ import annotations

import sys
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from .engine import KIND_K, Timeline, simulate
from .model import DeviceProfile, TaskSpec, id_ranks, resolve_group, stage_times

SUM_MODE = 1 if sys.version_info >= (3, 12) else 0


def _pysum(values) -> float:
    return sum(values)  # the interpreter's own builtin, as in heuristic.py:47


def select_first_task(rt: Sequence[TaskSpec], profile: DeviceProfile) -> TaskSpec:
    """Largest t_K - t_HtD, then longer DtH, then smaller id (heuristic.py:22-31)."""
    if not rt:
        raise ValueError("remaining task set is empty")

    def key(t):
        h, k, d = stage_times(t, profile)
        return (-(k - h), -d, t.id)

    return min(rt, key=key)


def _completion_estimate(partial: Timeline, rest: Sequence[TaskSpec], profile: DeviceProfile) -> float:
    """max(makespan, last K end + remaining kernel work + shortest DtH)
    (heuristic.py:34-49)."""
    k_end = max((c.end for c in partial.commands if c.kind == KIND_K), default=0.0)
    rest_k = _pysum(stage_times(r, profile)[1] for r in rest)
    tail = min(stage_times(r, profile)[2] for r in rest)
    return max(partial.makespan, k_end + rest_k + tail)


def select_next_task(rt: Sequence[TaskSpec], ot: Sequence[TaskSpec], profile: DeviceProfile) -> TaskSpec:
    """Candidate with the smallest (estimate, idle_K, id) (heuristic.py:52-78)."""
    if not rt:
        raise ValueError("remaining task set is empty")
    if not ot:
        raise ValueError("ordered task list is empty")
    if len(rt) == 1:
        return rt[0]
    best = None
    best_task = None
    for cand in sorted(rt, key=lambda t: t.id):
        tl = simulate(list(ot) + [cand], profile)
        rest = [r for r in rt if r is not cand]
        key = (_completion_estimate(tl, rest, profile), tl.idle[KIND_K], cand.id)
        if best is None or key < best:
            best, best_task = key, cand
    return best_task


def select_last_tasks(rt: Sequence[TaskSpec], ot: Sequence[TaskSpec],
                      profile: DeviceProfile) -> Tuple[TaskSpec, TaskSpec]:
    """Both completions simulated; tie -> shorter DtH last (heuristic.py:81-102)."""
    if len(rt) != 2:
        raise ValueError("select_last_tasks needs exactly two remaining tasks")
    a, b = sorted(rt, key=lambda t: t.id)
    m_ab = simulate(list(ot) + [a, b], profile).makespan
    m_ba = simulate(list(ot) + [b, a], profile).makespan
    if m_ab < m_ba:
        return a, b
    if m_ba < m_ab:
        return b, a
    return (b, a) if stage_times(a, profile)[2] <= stage_times(b, profile)[2] else (a, b)


def reorder_batch(tg: Sequence[TaskSpec], profile: DeviceProfile) -> List[TaskSpec]:
    """Near-optimal submission order for one task group (on the GPU)."""
    if not tg:
        raise ValueError("task group is empty")
    if len(tg) == 1:  # heuristic.py:113-114: returned as is, durations never resolved
        return [tg[0]]
    return reorder_batch_many([tg], profile)[0]


def reorder_batch_many(groups: Sequence[Sequence[TaskSpec]], profile: DeviceProfile,
                       n_dev: int = 1, return_makespans: bool = False):
    """reorder_batch over many independent groups of equal size in one launch."""
    if not groups:
        return ([], np.empty(0)) if return_makespans else []
    n = len(groups[0])
    if n == 0:
        raise ValueError("task group is empty")
    if any(len(g) != n for g in groups):
        raise ValueError("all groups of one batch must have the same size")
    if n == 1 and not return_makespans:  # heuristic.py:113-114 (no stage_times, no simulation)
        return [[g[0]] for g in groups]
    durs = np.stack([resolve_group(g, profile) for g in groups])
    ranks = np.stack([id_ranks(g) for g in groups])
    order, ms, _ = reorder_durs(durs, ranks, profile.dma_engines, profile.overlap_sigma, n_dev=n_dev)
    out = [[g[i] for i in row] for g, row in zip(groups, order.tolist())]
    return (out, ms) if return_makespans else out


def reorder_durs(durs, id_rank, dma: int, sigma: float, sum_mode: Optional[int] = None, n_dev: int = 1):
    """Array form: durs float64 [B][n][3], id_rank uint8 [B][n] ->
    (order uint8 [B][n], makespan float64 [B], n_sims uint32 [B])."""
    mode = SUM_MODE if sum_mode is None else int(sum_mode)
    return _capi.heuristic_batch(durs, id_rank, dma, sigma, mode, n_dev=n_dev)
