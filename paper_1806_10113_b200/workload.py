"""Scenario harness drop-ins and the input generators
they need, mirroring /root/reference/pkg/src/offsim/workload.py.

`run_scenario` replays the proxy-thread protocol (workers feed dependent
tasks, the proxy groups what is available, reorders each group and submits
it behind the commands still in flight) on the GPU, plus the NoReorder
distribution (row f1) for the speedup figures.  `run_heuristic_schedule_batch`
runs many independent scenarios in one launch (one GPU thread each).
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, replace
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi, synth
from .engine import KINDS, Command, Timeline, idle_report
from .heuristic import SUM_MODE
from .model import DeviceProfile, OffsimError, TaskDominance, TaskSpec, classify_task, resolve_group
from .noreorder import noreorder_distribution
from .search import DEFAULT_CAP, PermutationReport


class UnknownBenchmark(OffsimError):
    pass


class CapExceeded(UserWarning):
    """Ordering space larger than the cap; distribution is sampled."""


@dataclass(frozen=True)
class Benchmark:
    name: str
    tasks: Tuple[TaskSpec, ...]
    dk_fraction: float


@dataclass(frozen=True)
class Scenario:
    """T workers, each submitting a batch of N dependent tasks (workload.py:102-114)."""

    workers: int
    batch_depth: int
    pool: Benchmark
    seed: int
    profile: DeviceProfile

    def __post_init__(self):
        if self.workers < 1 or self.batch_depth < 1:
            raise ValueError("workers and batch_depth must be at least 1")


@dataclass
class ScenarioResult:
    heuristic_makespan: float
    timeline: Timeline
    tg_sizes: List[int]
    scheduling_overhead_ms: float
    noreorder: Optional[PermutationReport]
    speedup_heuristic: Optional[float]
    speedup_median: Optional[float]
    speedup_best: Optional[float]


BK_NAMES = tuple(synth.BK)


def load_table2_tasks() -> List[TaskSpec]:
    return [TaskSpec(id=k, fixed_durations=tuple(f * synth.TIME_UNIT_MS for f in synth.TABLE2[k]))
            for k in synth.TABLE2]


def make_benchmark(name: str, tasks: Sequence[TaskSpec]) -> Benchmark:
    dk = sum(1 for t in tasks if classify_task(t) is TaskDominance.DOMINANT_KERNEL)
    return Benchmark(name=name, tasks=tuple(tasks), dk_fraction=dk / len(tasks))


def load_bk_benchmark(name: str) -> Benchmark:
    if name not in synth.BK:
        raise UnknownBenchmark(f"unknown benchmark {name!r}; expected one of {BK_NAMES}")
    by_id = {t.id: t for t in load_table2_tasks()}
    return make_benchmark(name, [by_id[i] for i in synth.BK[name]])


def sample_real_tasks(device: str, count: int, seed: int) -> List[TaskSpec]:
    if device not in synth.REAL_TASK_RANGES:
        raise ValueError(f"unknown device {device!r}; expected one of {tuple(synth.REAL_TASK_RANGES)}")
    if count < 1:
        raise ValueError("count must be at least 1")
    ids, d = synth.real_group(device, count, seed)
    return [TaskSpec(id=i, fixed_durations=tuple(float(x) for x in r)) for i, r in zip(ids, d)]


def draw_worker_tasks(scenario: Scenario) -> List[List[TaskSpec]]:
    """_draw_worker_tasks (workload.py:185-194): pool picks, ids "w{w}.{j}"."""
    gen = np.random.default_rng(scenario.seed)
    pool = scenario.pool.tasks
    return [[replace(pool[int(gen.integers(len(pool)))], id=f"w{w}.{j}") for j in range(scenario.batch_depth)]
            for w in range(scenario.workers)]


def _flat(worker_tasks):
    return [t for row in worker_tasks for t in row]


def run_heuristic_schedule(scenario: Scenario, worker_tasks: List[List[TaskSpec]]):
    """(Timeline, tg_sizes, wall time per group in s) on the GPU.

    The third value is not the reference's per-group `reorder_batch` time
    (workload.py:227-229, a host-side measurement around each call): here the
    whole protocol -- every group's Algorithm 1 and the device simulation --
    runs inside one kernel, so it is the wall time of the whole harness call
    (H2D, kernel, D2H) divided by the number of groups."""
    T, N = scenario.workers, scenario.batch_depth
    flat = _flat(worker_tasks)
    d = resolve_group(flat, scenario.profile)
    order = sorted(range(len(flat)), key=lambda i: flat[i].id)
    rank = np.empty(len(flat), dtype=np.uint8 if len(flat) <= 64 else np.uint32)
    rank[order] = np.arange(len(flat))
    t0 = time.perf_counter()
    ms, ng, sz, st, en = _capi.harness_batch(d[None], rank[None], T, N, scenario.profile.dma_engines,
                                             scenario.profile.overlap_sigma, SUM_MODE, timeline=True)
    wall = time.perf_counter() - t0
    cmds = []
    for i, t in enumerate(flat):
        for k, kind in enumerate(KINDS):
            if st[0, i, k] >= 0.0:
                cmds.append(Command(t.id, kind, float(d[i, k]), float(st[0, i, k]), float(en[0, i, k]), 0.0))
    cmds.sort(key=lambda c: (c.start, c.end, KINDS.index(c.kind)))
    tl = Timeline(commands=cmds, makespan=float(ms[0]), idle=idle_report(cmds))
    sizes = [int(x) for x in sz[0, : int(ng[0])]]
    return tl, sizes, wall / max(len(sizes), 1)


def run_scenario(scenario: Scenario, evaluate_noreorder: bool = True, cap: int = DEFAULT_CAP) -> ScenarioResult:
    """workload.run_scenario (workload.py:330-362) on the GPU."""
    worker_tasks = draw_worker_tasks(scenario)
    timeline, tg_sizes, overhead = run_heuristic_schedule(scenario, worker_tasks)
    result = ScenarioResult(heuristic_makespan=timeline.makespan, timeline=timeline, tg_sizes=tg_sizes,
                            scheduling_overhead_ms=overhead * 1e3, noreorder=None, speedup_heuristic=None,
                            speedup_median=None, speedup_best=None)
    if evaluate_noreorder:
        report = noreorder_distribution(scenario, worker_tasks, cap)
        if not report.exhaustive:
            warnings.warn(f"ordering space exceeds cap={cap}; NoReorder distribution is sampled", CapExceeded,
                          stacklevel=2)
        result.noreorder = report
        result.speedup_heuristic = report.worst / timeline.makespan
        result.speedup_median = report.worst / report.median
        result.speedup_best = report.worst / report.best
    return result


def run_heuristic_schedule_batch(durs, id_rank, T: int, N: int, profile: DeviceProfile, n_dev: int = 1):
    """Many scenarios at once: durs [S][T*N][3], id_rank [S][T*N] ->
    (makespan [S], n_groups [S], tg_sizes [S][T*N])."""
    ms, ng, sz, _, _ = _capi.harness_batch(durs, id_rank, T, N, profile.dma_engines, profile.overlap_sigma,
                                           SUM_MODE, n_dev=n_dev)
    return ms, ng, sz
