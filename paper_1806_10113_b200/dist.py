"""Multi-GPU sharding over torch.distributed (one process per GPU).

Exhaustive search of one group (configs 3/4): rank r of W takes the
contiguous Lehmer-rank range [r*n!/W, (r+1)*n!/W) and reduces it on its
own GPU; the only exchange is one all_gather of the 48-byte summaries
(NCCL over NVLink on the GPU box, gloo in the CPU tests), combined on
every rank in rank order.  Because the ranges are ordered, "first rank
attaining the minimum" is the global lowest-rank argmin, so best / argmin /
worst / count are bit-exact and mean / geomean are fixed-order sums.

Batched groups and the heuristic (configs 2/5) shard the group index range
with no collective at all.
"""

from __future__ import annotations

import math
from typing import Callable, List, Optional, Tuple

import numpy as np

from .search import OrderingSummary, summary_from_dict

FIELDS = ("best", "best_rank", "worst", "sum", "sum_log", "count")


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    return total * rank // world, total * (rank + 1) // world


def pack(s: dict) -> np.ndarray:
    """Summary dict -> 6 float64 words (integers bit-cast, no rounding)."""
    out = np.empty(6, dtype=np.float64)
    out[0], out[2], out[3], out[4] = s["best"], s["worst"], s["sum"], s["sum_log"]
    out[1:2].view(np.uint64)[0] = np.uint64(s["best_rank"])
    out[5:6].view(np.uint64)[0] = np.uint64(s["count"])
    return out


def unpack(a: np.ndarray) -> dict:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return {"best": float(a[0]), "best_rank": int(a[1:2].view(np.uint64)[0]), "worst": float(a[2]),
            "sum": float(a[3]), "sum_log": float(a[4]), "count": int(a[5:6].view(np.uint64)[0])}


def combine(parts: List[dict]) -> dict:
    """Merge per-shard summaries in shard order (osim merge rules)."""
    acc = None
    for p in parts:
        if p["count"] == 0:
            continue
        if acc is None:
            acc = dict(p)
            continue
        if p["best"] < acc["best"] or (p["best"] == acc["best"] and p["best_rank"] < acc["best_rank"]):
            acc["best"], acc["best_rank"] = p["best"], p["best_rank"]
        if p["worst"] > acc["worst"]:
            acc["worst"] = p["worst"]
        acc["sum"] += p["sum"]
        acc["sum_log"] += p["sum_log"]
        acc["count"] += p["count"]
    if acc is None:
        acc = {"best": math.inf, "best_rank": 0, "worst": -math.inf, "sum": 0.0, "sum_log": 0.0, "count": 0}
    return acc


def _gpu_local(durs, dma, sigma, lo, hi) -> dict:
    from . import _capi
    s, _ = _capi.exhaustive(durs, dma, sigma, lo, hi)
    return s


def exhaustive_summary_distributed(durs, dma: int, sigma: float, group=None,
                                   local_fn: Optional[Callable] = None,
                                   device=None) -> OrderingSummary:
    """Whole-space summary of one group sharded over the process group."""
    import torch
    import torch.distributed as tdist

    d = np.asarray(durs, dtype=np.float64).reshape(-1, 3)
    n = d.shape[0]
    total = math.factorial(n)
    world = tdist.get_world_size(group)
    rank = tdist.get_rank(group)
    lo, hi = shard(total, rank, world)
    local = (local_fn or _gpu_local)(d, dma, sigma, lo, hi)
    backend = tdist.get_backend(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if backend == "nccl" else torch.device("cpu"))
    mine = torch.from_numpy(pack(local)).to(dev)
    bufs = [torch.empty_like(mine) for _ in range(world)]
    tdist.all_gather(bufs, mine, group=group)
    parts = [unpack(b.cpu().numpy()) for b in bufs]
    return summary_from_dict(combine(parts), n)
