"""Multi-GPU sharding over torch.distributed (one process per GPU).

Exhaustive search of one group (configs 3/4): rank r of W takes shard r
of the Lehmer-rank space -- on the GPU fast path the interleaved calls of
512 prefixes r, r + W, ... (osim_exhaustive_shard), otherwise (and with a
`local_fn`) the contiguous range [r*n!/W, (r+1)*n!/W) -- and reduces it on
its own GPU; the only exchange is one all_gather of the 48-byte summaries
(NCCL over NVLink on the GPU box, gloo in the CPU tests), combined on every
rank in rank order.  The merge keeps the lowest best and, on ties, the lower
best_rank, so best / argmin / worst / count are bit-exact for any partition
and mean / geomean are fixed-order sums.

Batched groups and the heuristic (configs 2/5) shard the group index range
with no collective in the compute (reorder_durs_distributed,
exhaustive_summary_batch_distributed; an optional all_gather assembles the
whole batch on every rank).
"""

from __future__ import annotations

import math
from typing import Callable, List, Optional, Tuple

import numpy as np

from .search import OrderingSummary, summary_from_dict

FIELDS = ("best", "best_rank", "worst", "sum", "sum_log", "count")


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    return total * rank // world, total * (rank + 1) // world


def default_suffix_len(n: int) -> int:
    """Default suffix length L of the prefix-sharing kernel (csrc/osim_launch.cuh
    default_pfx_l): one kernel call covers 512 prefixes x L! leaves."""
    return 1 if n <= 3 else (2 if n <= 5 else (3 if n <= 10 else 4))


def suffix_len(n: int) -> int:
    """The L the library actually uses for n (osim_pfx_suffix_len: the default,
    or the OSIM_PFX_L tuning override for n in {8, 10, 12}, read once per
    process), so the interleaved ranges below match its shards."""
    from . import _capi

    return int(_capi.load().osim_pfx_suffix_len(int(n)))


def shard_ranges(n: int, rank: int, world: int, fast: bool = True) -> List[Tuple[int, int]]:
    """The Lehmer-rank ranges osim_exhaustive_shard gives rank `rank` of
    `world`: on the fast path the interleaved 512-prefix calls rank,
    rank + world, ... (each 512 * L! consecutive ranks), otherwise the
    contiguous `shard` range.  Every ordering lies in exactly one rank's
    ranges."""
    total = math.factorial(n)
    if not fast:
        return [shard(total, rank, world)]
    chunk = 512 * math.factorial(suffix_len(n))
    calls = -(-total // chunk)
    return [(k * chunk, min(total, (k + 1) * chunk)) for k in range(rank, calls, world)]


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


def exhaustive_summary_distributed(durs, dma: int, sigma: float, group=None,
                                   local_fn: Optional[Callable] = None,
                                   device=None, interleaved: bool = False) -> OrderingSummary:
    """Whole-space summary of one group sharded over the process group.
    Without `local_fn` each rank runs its library shard on its GPU; with
    `local_fn(durs, dma, sigma, lo, hi) -> summary dict` (e.g. the oracle in
    the CPU tests) each rank evaluates its contiguous `shard` range, or with
    `interleaved=True` the library's interleaved ranges (`shard_ranges`)."""
    import torch
    import torch.distributed as tdist

    d = np.asarray(durs, dtype=np.float64).reshape(-1, 3)
    n = d.shape[0]
    world = tdist.get_world_size(group)
    rank = tdist.get_rank(group)
    if local_fn is None:
        # the library's shard: interleaved 512-prefix calls on the fast path
        # (every rank samples the whole rank space, so per-rank work evens
        # out), the contiguous range otherwise; combine() is order-free for
        # best / argmin (ties to the lower rank) / worst / count
        from . import _capi

        local = _capi.exhaustive_shard(d, dma, sigma, rank, world)
        part_l = suffix_len(n) if _capi.fast_eligible(d, sigma) == 1 else 0
    else:
        ranges = shard_ranges(n, rank, world, fast=interleaved)
        local = combine([local_fn(d, dma, sigma, lo, hi) for lo, hi in ranges])
        part_l = suffix_len(n) if interleaved else 0
    backend = tdist.get_backend(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if backend == "nccl" else torch.device("cpu"))
    # word 6: the partition this rank used (suffix length L of the interleaved
    # calls, 0 = contiguous); ranks whose environments disagree (OSIM_PFX_L)
    # would double-count or drop orderings, so every rank checks all of them
    mine = torch.from_numpy(np.append(pack(local), float(part_l))).to(dev)
    bufs = [torch.empty_like(mine) for _ in range(world)]
    tdist.all_gather(bufs, mine, group=group)
    rows = [b.cpu().numpy() for b in bufs]
    if len({float(r[6]) for r in rows}) != 1:
        raise ValueError("ranks partitioned the rank space differently (suffix lengths %s); "
                         "set OSIM_PFX_L identically on every rank" % [float(r[6]) for r in rows])
    return summary_from_dict(combine([unpack(r[:6]) for r in rows]), n)


# ---- batches of groups (configs 2 and 5): group-range shards, no collective
# in the compute; gather=True assembles the whole batch on every rank -------

def _gather_rows(local: np.ndarray, total: int, group, world: int, device) -> np.ndarray:
    """all_gather of this rank's contiguous rows of a [total][...] array
    (shards from `shard`, padded to the largest shard for the collective)."""
    import torch
    import torch.distributed as tdist

    width = max(shard(total, r, world)[1] - shard(total, r, world)[0] for r in range(world))
    row = local.shape[1:]
    # explicit row width: reshape(0, -1) is ambiguous for a rank whose shard is empty
    row_bytes = local.dtype.itemsize * int(np.prod(row, dtype=np.int64))
    raw = np.ascontiguousarray(local).view(np.uint8).reshape(local.shape[0], row_bytes)
    pad = np.zeros((width, raw.shape[1]), dtype=np.uint8)
    pad[: raw.shape[0]] = raw
    t = torch.from_numpy(pad).to(device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    tdist.all_gather(bufs, t, group=group)
    parts = []
    for r, b in enumerate(bufs):
        lo, hi = shard(total, r, world)
        parts.append(b.cpu().numpy()[: hi - lo])
    out = np.concatenate(parts).view(local.dtype)
    return out.reshape((total,) + row)


def _coll_device(group, device):
    import torch
    import torch.distributed as tdist

    if device is not None:
        return device
    return torch.device("cuda", torch.cuda.current_device()) if tdist.get_backend(group) == "nccl" else \
        torch.device("cpu")


def reorder_durs_distributed(durs, id_rank, dma: int, sigma: float, sum_mode: Optional[int] = None, group=None,
                             gather: bool = True, local_fn: Optional[Callable] = None, device=None):
    """reorder_batch over a batch sharded by group range over the process
    group (one GPU per rank, no collective in the compute).  Returns
    (order uint8 [B][n], makespan [B], n_sims [B]) for the whole batch on every
    rank (gather=True, one all_gather per output) or this rank's rows."""
    import torch.distributed as tdist

    from . import _capi
    from .heuristic import SUM_MODE

    d = np.ascontiguousarray(np.asarray(durs, dtype=np.float64))
    r = np.ascontiguousarray(np.asarray(id_rank, dtype=np.uint8))
    B = d.shape[0]
    world, rank = tdist.get_world_size(group), tdist.get_rank(group)
    lo, hi = shard(B, rank, world)
    mode = SUM_MODE if sum_mode is None else int(sum_mode)
    fn = local_fn or (lambda dd, rr: _capi.heuristic_batch(dd, rr, dma, sigma, mode))
    order, ms, sims = fn(d[lo:hi], r[lo:hi])
    if not gather:
        return order, ms, sims
    dev = _coll_device(group, device)
    return (_gather_rows(np.asarray(order, dtype=np.uint8), B, group, world, dev),
            _gather_rows(np.asarray(ms, dtype=np.float64), B, group, world, dev),
            _gather_rows(np.asarray(sims, dtype=np.uint32), B, group, world, dev))


def exhaustive_summary_batch_distributed(durs, dma: int, sigma: float, group=None, gather: bool = True,
                                         local_fn: Optional[Callable] = None, device=None) -> np.ndarray:
    """One full-space summary per group of a batch sharded by group range
    (config 2); _capi.SUMMARY_DTYPE records for the whole batch on every rank
    (gather=True) or this rank's rows."""
    import torch.distributed as tdist

    from . import _capi

    d = np.ascontiguousarray(np.asarray(durs, dtype=np.float64))
    B = d.shape[0]
    world, rank = tdist.get_world_size(group), tdist.get_rank(group)
    lo, hi = shard(B, rank, world)
    fn = local_fn or (lambda dd: _capi.exhaustive_batch(dd, dma, sigma))
    out = fn(d[lo:hi])
    if not gather:
        return out
    return _gather_rows(out, B, group, world, _coll_device(group, device))


# ---- order statistics of a sharded makespan set (row f2) -------------------

RADIX_BITS = 11


def _bits_to_double(b: int) -> float:
    return float(np.array([b], dtype=np.uint64).view(np.float64)[0])


def _double_bits(x: float) -> int:
    return int(np.array([x], dtype=np.float64).view(np.uint64)[0])


def common_prefix(vmin: float, vmax: float) -> Tuple[int, int]:
    """(prefix, bits): the leading bit-pattern bits shared by every positive
    double in [vmin, vmax] (the selection walk starts below them)."""
    if not (vmin > 0.0 and vmax >= vmin):
        return 0, 0
    a, b = _double_bits(vmin), _double_bits(vmax)
    bits = 64 - (a ^ b).bit_length()
    bits = min(bits, 63)
    return a >> (64 - bits) if bits else 0, bits


def select_kth_distributed(local_hist: Callable, k: int, group=None, device=None,
                           vmin: float = 0.0, vmax: float = 0.0) -> float:
    """k-th smallest (0-based) positive double of a set sharded over ranks.

    local_hist(prefix, prefix_bits, digit_bits) -> int64 histogram of this
    rank's values (2**digit_bits bins, MSB-first digits of the bit pattern,
    values whose top prefix_bits bits equal prefix).  One all_reduce(SUM)
    per pass combines the ranks (NCCL on GPUs); every rank gets the answer.
    vmin / vmax (the set's min and max, e.g. best / worst) skip the leading
    bits all values share.
    """
    import torch
    import torch.distributed as tdist

    backend = tdist.get_backend(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if backend == "nccl" else torch.device("cpu"))
    prefix, pbits = common_prefix(vmin, vmax)
    while pbits < 64:
        d = min(RADIX_BITS, 64 - pbits)
        h = torch.from_numpy(np.ascontiguousarray(local_hist(prefix, pbits, d), dtype=np.int64)).to(dev)
        tdist.all_reduce(h, group=group)
        tot = h.cpu().numpy()
        cum = np.cumsum(tot)
        b = int(np.searchsorted(cum, k, side="right"))
        if b >= len(tot):
            raise ValueError(f"rank {k} outside the value set")
        k -= int(cum[b - 1]) if b > 0 else 0
        prefix = (prefix << d) | b
        pbits += d
    return _bits_to_double(prefix)


def numpy_hist(vals: np.ndarray):
    """Host histogram of positive doubles (test double of osim_radix_hist_dev)."""
    u = np.ascontiguousarray(vals, dtype=np.float64).view(np.uint64)

    def hist(prefix, pbits, dbits):
        sel = u if pbits == 0 else u[(u >> np.uint64(64 - pbits)) == np.uint64(prefix)]
        dig = (sel >> np.uint64(64 - pbits - dbits)) & np.uint64((1 << dbits) - 1)
        return np.bincount(dig.astype(np.int64), minlength=1 << dbits)

    return hist


def median_distributed(local_hist: Callable, count: int, group=None, device=None,
                       vmin: float = 0.0, vmax: float = 0.0) -> float:
    """np.median of the sharded set: the middle value, or (a + b) / 2."""
    if count % 2:
        return select_kth_distributed(local_hist, count // 2, group, device, vmin, vmax)
    a = select_kth_distributed(local_hist, count // 2 - 1, group, device, vmin, vmax)
    b = select_kth_distributed(local_hist, count // 2, group, device, vmin, vmax)
    return float(np.float64(a) + np.float64(b)) / 2.0


def exhaustive_stats_distributed(durs, dma: int, sigma: float, threshold: float = float("-inf"), group=None):
    """Summary, below-threshold count and exact median of one group's whole
    ordering space, sharded over the process group (one GPU per rank): each
    rank keeps its shard's makespans in HBM (8 B per ordering), reductions and
    selection histograms are combined with NCCL all_gather / all_reduce."""
    import ctypes as C

    import torch
    import torch.distributed as tdist

    from . import _capi

    d = np.asarray(durs, dtype=np.float64).reshape(-1, 3)
    n = d.shape[0]
    total = math.factorial(n)
    world, rank = tdist.get_world_size(group), tdist.get_rank(group)
    lo, hi = shard(total, rank, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    L = _capi.load()
    # library work and torch's reads of its outputs must share one stream; the
    # legacy default stream (handle 0) would map to the library's own stream
    st = torch.cuda.Stream(device=dev)
    st.wait_stream(torch.cuda.current_stream())
    prev = torch.cuda.current_stream()
    torch.cuda.set_stream(st)
    try:
        return _stats_on_stream(L, C, torch, tdist, _capi, d, n, dma, sigma, threshold, group, lo, hi, world, dev, st)
    finally:
        torch.cuda.set_stream(prev)


def _stats_on_stream(L, C, torch, tdist, _capi, d, n, dma, sigma, threshold, group, lo, hi, world, dev, st):
    sp = C.c_void_p(st.cuda_stream)
    dd = torch.from_numpy(d).to(dev)
    out = torch.zeros(6, dtype=torch.float64, device=dev)
    below = torch.zeros(1, dtype=torch.int64, device=dev)
    ms = torch.empty(max(hi - lo, 1), dtype=torch.float64, device=dev)
    hist = torch.empty(1 << RADIX_BITS, dtype=torch.int64, device=dev)  # uint64 counts (< 2^63)
    fast = int(_capi.fast_eligible(d, sigma))
    _capi.check(L.osim_exhaustive_ex_dev(C.c_void_p(dd.data_ptr()), n, int(dma), float(sigma), lo, hi, fast,
                                         float(threshold), C.c_void_p(out.data_ptr()), C.c_void_p(below.data_ptr()),
                                         C.c_void_p(ms.data_ptr()), sp))
    bufs = [torch.empty_like(out) for _ in range(world)]
    tdist.all_gather(bufs, out, group=group)
    tdist.all_reduce(below, group=group)
    summ = summary_from_dict(combine([unpack(b.cpu().numpy()) for b in bufs]), n)

    def local_hist(prefix, pbits, dbits):
        _capi.check(L.osim_radix_hist_dev(C.c_void_p(ms.data_ptr()), hi - lo, prefix, pbits, dbits,
                                          C.c_void_p(hist.data_ptr()), sp))
        return hist[: 1 << dbits].cpu().numpy()

    med = median_distributed(local_hist, summ.count, group, vmin=summ.best, vmax=summ.worst)
    return summ, int(below.item()), med
