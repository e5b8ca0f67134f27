"""NoReorder baseline distribution on the GPU.

Drop-ins for workload.simulate_sequence / noreorder_distribution
(/root/reference/pkg/src/offsim/workload.py:259-327): T workers each submit N
dependent tasks in order; the paper's NoReorder baseline is the makespan
distribution over every interleaving of the workers' task sequences that
keeps each worker's own order.  The GPU enumerates the interleavings by
multinomial rank (the order of `sorted(set(permutations(labels)))`), gates
each task on its predecessor's completion, and on a 1-DMA device splits the
sequence into submit waves exactly as simulate_sequence does.
"""

from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from .engine import Timeline, _simulate
from .model import MAX_ENUM_TASKS, MAX_TASKS, DeviceProfile, TaskSpec, resolve_group
from .search import PermutationReport


def simulate_sequence(seq: Sequence[TaskSpec], profile: DeviceProfile,
                      deps: Optional[Dict[str, str]] = None) -> Timeline:
    """workload.simulate_sequence (workload.py:277-304) on the GPU."""
    if not seq:
        raise ValueError("task group must be non-empty")
    deps = deps or {}
    return _simulate(list(seq), profile, deps or None, waves=profile.dma_engines == 1 and bool(deps))


def interleaving_count(T: int, N: int) -> int:
    return math.factorial(T * N) // math.factorial(N) ** T


def unrank_labels(rank: int, T: int, N: int) -> Tuple[int, ...]:
    """Index into sorted(set(permutations(labels))) -> label sequence."""
    c = [N] * T
    rem = T * N
    m = interleaving_count(T, N)
    out = []
    for _ in range(T * N):
        for w in range(T):
            if not c[w]:
                continue
            mw = m * c[w] // rem
            if rank < mw:
                out.append(w)
                c[w] -= 1
                rem -= 1
                m = mw
                break
            rank -= mw
    return tuple(out)


def sample_interleavings(T: int, N: int, cap: int, seed: int) -> np.ndarray:
    """`cap` distinct label sequences in first-drawn order from
    default_rng(seed).permutation(labels) (workload.py:266-274)."""
    labels = np.array([w for w in range(T) for _ in range(N)])
    gen = np.random.default_rng(seed)
    kept = {}
    while len(kept) < cap:
        p = gen.permutation(labels)
        key = p.tobytes()
        if key not in kept:
            kept[key] = p
    return np.array(list(kept.values()), dtype=np.uint8).reshape(cap, T * N)


def distribution_durs(durs, dma: int, sigma: float, cap: int = 10_000, seed: int = 0):
    """Array form: durs float64 [T][N][3] -> (labels uint8 [count][T*N],
    makespans float64 [count], summary dict, exhaustive flag)."""
    d = np.ascontiguousarray(np.asarray(durs, dtype=np.float64))
    T, N = d.shape[0], d.shape[1]
    if T * N > MAX_TASKS:
        raise NotImplementedError(f"more than {MAX_TASKS} tasks are not supported on the B200 path")
    total = interleaving_count(T, N)
    flat = d.reshape(-1, 3)
    if total <= cap:
        if T * N > MAX_ENUM_TASKS:
            raise NotImplementedError(f"enumerating the interleavings of more than {MAX_ENUM_TASKS} tasks")
        summ, _, ms = _capi.interleavings(flat, T, N, dma, sigma, 0, total, want_makespans=True)
        labels = None
        exhaustive = True
    else:
        labels = sample_interleavings(T, N, cap, seed)
        summ, ms = _capi.eval_sequences(flat, T, N, dma, sigma, labels)
        exhaustive = False
    return labels, ms, summ, exhaustive


def noreorder_distribution(scenario, worker_tasks: List[List[TaskSpec]], cap: int = 10_000) -> PermutationReport:
    """workload.noreorder_distribution (workload.py:307-327) on the GPU.
    `scenario` needs .workers, .batch_depth, .seed and .profile."""
    T, N = scenario.workers, scenario.batch_depth
    profile = scenario.profile
    d = np.stack([resolve_group(worker_tasks[w], profile) for w in range(T)])
    labels, ms, summ, exhaustive = distribution_durs(d, profile.dma_engines, profile.overlap_sigma, cap,
                                                     scenario.seed)
    count = len(ms)

    def ordering(lab):
        cnt = [0] * T
        ids = []
        for w in lab:
            ids.append(worker_tasks[w][cnt[w]].id)
            cnt[w] += 1
        return tuple(ids)

    if labels is None:
        orderings = [ordering(unrank_labels(r, T, N)) for r in range(count)]
    else:
        orderings = [ordering(row) for row in labels.tolist()]
    return PermutationReport(
        orderings=orderings, makespans=ms.tolist(), best_ordering=orderings[int(summ["best_rank"])],
        best=float(summ["best"]), worst=float(summ["worst"]), median=float(np.median(ms)),
        geomean=float(np.exp(np.log(ms).mean())), exhaustive=exhaustive)
