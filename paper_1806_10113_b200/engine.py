"""Simulator drop-in (offsim.engine): `simulate` on the B200.

`simulate(tasks, profile)` (engine.py:252-263 in the reference) resolves
stage times on the host and runs the event loop in the CUDA library
(osim_timeline); the returned `Timeline` carries the same command records,
sort order, makespan and idle report as the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from . import _capi
from .model import DeviceProfile, TaskSpec, resolve_group

KIND_HTD = "HtD"
KIND_K = "K"
KIND_DTH = "DtH"
KINDS = (KIND_HTD, KIND_K, KIND_DTH)


@dataclass
class Command:
    """One queued command (engine.py:29-36)."""

    task_id: str
    kind: str
    nominal_duration: float
    start: Optional[float] = None
    end: Optional[float] = None
    remaining_work: float = 1.0


@dataclass
class Timeline:
    """Finalized commands plus makespan and per-kind idle (engine.py:39-48)."""

    commands: List[Command]
    makespan: float
    idle: Dict[str, float]

    def commands_of_kind(self, kind: str) -> List[Command]:
        return [c for c in self.commands if c.kind == kind]


def recompute_overlap(executing_htd: Command, executing_dth: Command, now: float,
                      profile: DeviceProfile) -> Tuple[float, float]:
    """Closed-form provisional ends of two overlapping transfers,
    now + rw*nd/sigma each (engine.py:51-65)."""
    s = profile.overlap_sigma
    return (now + executing_htd.remaining_work * executing_htd.nominal_duration / s,
            now + executing_dth.remaining_work * executing_dth.nominal_duration / s)


def idle_report(commands: Sequence[Command]) -> Dict[str, float]:
    """Per-kind sum of gaps between (start, end)-sorted spans (engine.py:68-80)."""
    out: Dict[str, float] = {}
    for kind in KINDS:
        spans = sorted((c.start, c.end) for c in commands if c.kind == kind and c.start is not None)
        gap = 0.0
        for i in range(1, len(spans)):
            if spans[i][0] > spans[i - 1][1]:
                gap += spans[i][0] - spans[i - 1][1]
        out[kind] = gap
    return out


def simulate(tasks: Sequence[TaskSpec], profile: DeviceProfile,
             deps: Optional[Dict[str, str]] = None) -> Timeline:
    """Simulate one ordered task group on the GPU and return its timeline."""
    if not tasks:
        raise ValueError("task group must be non-empty")
    return _simulate(tasks, profile, deps, waves=False)


def _simulate(tasks: Sequence[TaskSpec], profile: DeviceProfile, deps: Optional[Dict[str, str]],
              waves: bool) -> Timeline:
    """One ordered group on the GPU; deps -> osim_timeline_deps (waves: the
    1-DMA split of workload.simulate_sequence)."""
    durs = resolve_group(tasks, profile)
    n = len(tasks)
    if deps:
        index = {t.id: i for i, t in enumerate(tasks)}
        dep = [-1] * n
        for i, t in enumerate(tasks):
            d = deps.get(t.id)
            if d is not None:
                if d not in index:
                    # never finishes -> the task's commands never become ready
                    # (engine.py:169-171) -> DeviceSim.run stalls (:239-241)
                    raise RuntimeError("simulation stalled with commands pending")
                dep[i] = index[d]
        start, end, makespan, idle = _capi.timeline_deps(durs, profile.dma_engines, profile.overlap_sigma,
                                                         list(range(n)), dep, waves)
    else:
        start, end, makespan, idle = _capi.timeline(durs, profile.dma_engines, profile.overlap_sigma,
                                                    list(range(n)))
    cmds: List[Command] = []
    for i, t in enumerate(tasks):
        for k, kind in enumerate(KINDS):
            if start[i, k] >= 0.0:
                cmds.append(Command(t.id, kind, float(durs[i, k]), float(start[i, k]), float(end[i, k]), 0.0))
    cmds.sort(key=lambda c: (c.start, c.end, KINDS.index(c.kind)))
    return Timeline(commands=cmds, makespan=float(makespan),
                    idle={KIND_HTD: float(idle[0]), KIND_K: float(idle[1]), KIND_DTH: float(idle[2])})
