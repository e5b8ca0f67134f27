"""Micro-step validation oracle on the GPU.

`micro_simulate` is the drop-in for oracle.micro_simulate
(/root/reference/pkg/src/offsim/oracle.py:60-95, core _micro.py:19-143): a
fixed-dt tick simulator independent of the event engine.  `validate` is the
`offsim validate` sweep (cli.py:162-181): every ordering of each BK set on
both bundled profiles through the event engine and the tick oracle, with
the maximum deviation checked against 2*dt -- both simulators on the GPU.
"""

from __future__ import annotations

import math
from typing import Iterable, List, Sequence, Tuple

import numpy as np

from . import _capi, synth
from .engine import KINDS, Command, Timeline, idle_report
from .model import DeviceProfile, TaskSpec, resolve_group

DEFAULT_DT = 0.001  # ms, oracle.py:23


def micro_simulate(tasks: Sequence[TaskSpec], profile: DeviceProfile, dt: float = DEFAULT_DT) -> Timeline:
    """Fixed-step reference timeline (command times quantized to dt)."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    durs = resolve_group(tasks, profile, submit_checks=False)
    n = len(tasks)
    if n == 0:  # micro_core over empty arrays: no commands, makespan 0.0 (_micro.py:68-71)
        return Timeline(commands=[], makespan=0.0, idle=idle_report([]))
    st, en, ms = _capi.micro_timeline(durs, profile.dma_engines, profile.overlap_sigma, dt, list(range(n)))
    cmds: List[Command] = []
    for k, kind in enumerate(KINDS):  # oracle.py:80-93 builds HtD, then K, then DtH commands
        for i, t in enumerate(tasks):
            if st[i, k] >= 0.0:
                cmds.append(Command(t.id, kind, float(durs[i, k]), float(st[i, k]), float(en[i, k]), 0.0))
    cmds.sort(key=lambda c: (c.start, c.end, KINDS.index(c.kind)))
    return Timeline(commands=cmds, makespan=float(ms), idle=idle_report(cmds))


# bundled profiles (data/profiles/one_dma.json, two_dma.json): (dma, sigma)
BUNDLED = {"1dma": (1, 1.0), "2dma": (2, 0.5)}


def validate(benchmarks: Iterable[str] = tuple(synth.BK), dt: float = DEFAULT_DT) -> Tuple[int, float, bool]:
    """(orderings checked, max |engine - micro| ms, max <= 2*dt)."""
    names = [b for b in benchmarks]
    if not names:
        raise ValueError("empty benchmark selector")
    checked, max_dev = 0, 0.0
    for name in names:
        _, d = synth.bk_group(name)
        n = d.shape[0]
        total = math.factorial(n)
        for dma, sigma in BUNDLED.values():
            _, eng = _capi.exhaustive(d, dma, sigma, 0, total, want_makespans=True)
            mic = _capi.micro(d, dma, sigma, dt, 0, total)
            max_dev = max(max_dev, float(np.max(np.abs(eng - mic))))
            checked += total
    return checked, max_dev, max_dev <= 2.0 * dt
