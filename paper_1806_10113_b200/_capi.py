"""ctypes binding of include/offsim_b200.h (liboffsim_b200.so).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every call raises.  ctypes releases the GIL for the duration of a
call; the library is reentrant (per-device mutex).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .model import UnresolvableDuration

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OSIM_LIB") or os.path.join(PKG, "liboffsim_b200.so")  # OSIM_LIB: A/B builds (tuning only)

OSIM_OK, OSIM_EINVAL, OSIM_ENODEV, OSIM_ECUDA, OSIM_ENCCL, OSIM_ESTALL = 0, -1, -2, -3, -4, -5

# Every symbol include/offsim_b200.h declares (tests check the export list).
EXPORTS = (
    "osim_version", "osim_last_error", "osim_init", "osim_shutdown", "osim_set_device",
    "osim_exhaustive", "osim_eval_perms", "osim_exhaustive_batch", "osim_heuristic_batch",
    "osim_timeline", "osim_fast_eligible", "osim_exhaustive_dev", "osim_exhaustive_batch_dev",
    "osim_heuristic_batch_dev", "osim_selftest_div", "osim_fp64_peak", "osim_exhaustive_stats",
    "osim_exhaustive_ex_dev", "osim_radix_hist_dev", "osim_interleavings", "osim_eval_sequences",
    "osim_timeline_deps", "osim_micro", "osim_micro_timeline", "osim_harness_batch",
    "osim_exhaustive_shard_dev", "osim_exhaustive_shard", "osim_select_kth_dev",
    "osim_pfx_suffix_len", "osim_timeline_u32", "osim_eval_perms_u32", "osim_eval_sequences_u32",
    "osim_heuristic_batch_u32", "osim_harness_batch_u32", "osim_micro_timeline_u32", "osim_selftest_div_mode",
)


class OsimSummary(C.Structure):
    _fields_ = [
        ("best", C.c_double),
        ("best_rank", C.c_uint64),
        ("worst", C.c_double),
        ("sum", C.c_double),
        ("sum_log", C.c_double),
        ("count", C.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


SUMMARY_DTYPE = np.dtype([("best", "<f8"), ("best_rank", "<u8"), ("worst", "<f8"), ("sum", "<f8"),
                          ("sum_log", "<f8"), ("count", "<u8")])
assert SUMMARY_DTYPE.itemsize == C.sizeof(OsimSummary) == 48


class OsimError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{msg} (osim code {code})")
        self.code = code


class StallError(RuntimeError):
    """engine.py:239-241: simulation stalled with commands pending (the
    reference raises RuntimeError; this is a subclass)."""


_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load the library (no build, no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_1806_10113_b200._build` "
                "(there is no CPU fallback)")
        L = C.CDLL(path)
        dp, u8p, u32p, vp = C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.c_void_p
        i32p = C.POINTER(C.c_int32)
        sp = C.POINTER(OsimSummary)
        i, d, u64 = C.c_int, C.c_double, C.c_uint64
        sig = {
            "osim_version": ([], C.c_char_p),
            "osim_last_error": ([], C.c_char_p),
            "osim_init": ([i, C.POINTER(i)], i),
            "osim_shutdown": ([], i),
            "osim_set_device": ([i], i),
            "osim_exhaustive": ([dp, i, i, d, u64, u64, i, sp, dp], i),
            "osim_eval_perms": ([dp, i, i, d, u8p, u64, i, dp, sp], i),
            "osim_exhaustive_batch": ([dp, u64, i, i, d, i, vp], i),
            "osim_heuristic_batch": ([dp, u8p, u64, i, i, d, i, i, u8p, dp, u32p], i),
            "osim_timeline": ([dp, i, i, d, u8p, dp, dp, dp, dp], i),
            "osim_fast_eligible": ([dp, u64, d], i),
            "osim_exhaustive_dev": ([vp, i, i, d, u64, u64, i, vp, vp, vp], i),
            "osim_exhaustive_shard_dev": ([vp, i, i, d, i, i, i, vp, vp], i),
            "osim_exhaustive_shard": ([dp, i, i, d, i, i, sp], i),
            "osim_exhaustive_batch_dev": ([vp, u64, i, i, d, i, vp, vp], i),
            "osim_heuristic_batch_dev": ([vp, vp, u64, i, i, d, i, i, vp, vp, vp, vp], i),
            "osim_selftest_div": ([u64, u64, C.POINTER(u64)], i),
            "osim_selftest_div_mode": ([u64, u64, i, C.POINTER(u64)], i),
            "osim_exhaustive_stats": ([dp, i, i, d, u64, u64, d, i, sp, C.POINTER(u64), dp], i),
            "osim_exhaustive_ex_dev": ([vp, i, i, d, u64, u64, i, d, vp, vp, vp, vp], i),
            "osim_radix_hist_dev": ([vp, u64, u64, i, i, vp, vp], i),
            "osim_select_kth_dev": ([vp, u64, u64, dp, vp], i),
            "osim_pfx_suffix_len": ([i], i),
            "osim_timeline_u32": ([dp, u64, i, d, u32p, i32p, i, dp, dp, dp, dp], i),
            "osim_eval_perms_u32": ([dp, u64, i, d, u32p, u64, i, dp, sp], i),
            "osim_eval_sequences_u32": ([dp, C.c_uint32, C.c_uint32, i, d, u32p, u64, i, dp, sp], i),
            "osim_heuristic_batch_u32": ([dp, u32p, u64, u64, i, d, i, i, u32p, dp, u32p], i),
            "osim_harness_batch_u32": ([dp, u32p, u64, C.c_uint32, C.c_uint32, i, d, i, i, dp, u32p, u32p, dp, dp],
                                       i),
            "osim_micro_timeline_u32": ([dp, u64, i, d, d, u32p, dp, dp, dp], i),
            "osim_interleavings": ([dp, i, i, i, d, u64, u64, d, i, sp, C.POINTER(u64), dp], i),
            "osim_eval_sequences": ([dp, i, i, i, d, u8p, u64, i, dp, sp], i),
            "osim_micro": ([dp, i, i, d, d, u64, u64, i, dp], i),
            "osim_harness_batch": ([dp, u8p, u64, i, i, i, d, i, i, dp, u8p, u8p, dp, dp], i),
            "osim_micro_timeline": ([dp, i, i, d, d, u8p, dp, dp, dp], i),
            "osim_timeline_deps": ([dp, i, i, d, u8p, C.POINTER(C.c_int8), i, dp, dp, dp, dp], i),
            "osim_fp64_peak": ([dp], i),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def check(rc: int):
    if rc == OSIM_OK:
        return
    msg = load().osim_last_error().decode(errors="replace")
    if rc == OSIM_EINVAL:
        if "no commands" in msg:
            raise UnresolvableDuration(msg)
        raise ValueError(msg)
    if rc == OSIM_ESTALL:
        raise StallError(msg)
    raise OsimError(rc, msg)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.reshape(shape) if shape is not None else a


def u8(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint8))
    return a.reshape(shape) if shape is not None else a


# ---- thin typed wrappers ------------------------------------------------

def init(want: int = 0) -> int:
    got = C.c_int()
    check(load().osim_init(want, C.byref(got)))
    return got.value


def set_device(dev: int):
    check(load().osim_set_device(int(dev)))


def exhaustive(durs, dma, sigma, lo, hi, n_dev=1, want_makespans=False):
    d = f64(durs, (-1, 3))
    n = d.shape[0]
    out = OsimSummary()
    ms = np.empty(hi - lo) if want_makespans else None
    check(load().osim_exhaustive(ptr(d, C.c_double), n, int(dma), float(sigma), int(lo), int(hi), int(n_dev),
                                 C.byref(out), ptr(ms, C.c_double) if ms is not None else None))
    return out.as_dict(), ms


def exhaustive_shard(durs, dma, sigma, shard, shards):
    """Summary dict of shard `shard` of `shards` of all n! orderings
    (osim_exhaustive_shard: interleaved prefix calls on the fast path)."""
    d = f64(durs, (-1, 3))
    out = OsimSummary()
    check(load().osim_exhaustive_shard(ptr(d, C.c_double), d.shape[0], int(dma), float(sigma), int(shard),
                                       int(shards), C.byref(out)))
    return out.as_dict()


def exhaustive_stats(durs, dma, sigma, lo, hi, threshold=float("-inf"), n_dev=1, median=True):
    """(summary dict, count strictly below threshold, exact median or None)."""
    d = f64(durs, (-1, 3))
    n = d.shape[0]
    out = OsimSummary()
    below = C.c_uint64()
    med = C.c_double()
    check(load().osim_exhaustive_stats(ptr(d, C.c_double), n, int(dma), float(sigma), int(lo), int(hi),
                                       float(threshold), int(n_dev), C.byref(out), C.byref(below),
                                       C.byref(med) if median else None))
    return out.as_dict(), below.value, (med.value if median else None)


def select_kth_dev(d_vals_ptr: int, count: int, k: int, stream: int = 0) -> float:
    """k-th smallest (0-based) of `count` non-negative doubles at device
    address d_vals_ptr (osim_select_kth_dev; waits for `stream` first)."""
    out = C.c_double()
    check(load().osim_select_kth_dev(C.c_void_p(d_vals_ptr), int(count), int(k), C.byref(out),
                                     C.c_void_p(stream) if stream else None))
    return out.value


WIDE_MAX = 64  # largest group of the uint8 entry points; above: the *_u32 general path (osim_big.cuh)


def u32(a, shape=None) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(a, dtype=np.uint32))
    return x.reshape(shape) if shape is not None else x


def eval_perms(durs, dma, sigma, perms, n_dev=1):
    d = f64(durs, (-1, 3))
    n = d.shape[0]
    if n > WIDE_MAX:
        p = u32(perms, (-1, n))
        ms = np.empty(p.shape[0])
        out = OsimSummary()
        check(load().osim_eval_perms_u32(ptr(d, C.c_double), n, int(dma), float(sigma), ptr(p, C.c_uint32),
                                         p.shape[0], int(n_dev), ptr(ms, C.c_double), C.byref(out)))
        return out.as_dict(), ms
    p = u8(perms, (-1, n))
    ms = np.empty(p.shape[0])
    out = OsimSummary()
    check(load().osim_eval_perms(ptr(d, C.c_double), n, int(dma), float(sigma), ptr(p, C.c_uint8), p.shape[0],
                                 int(n_dev), ptr(ms, C.c_double), C.byref(out)))
    return out.as_dict(), ms


def exhaustive_batch(durs, dma, sigma, n_dev=1, out=None):
    d = durs if isinstance(durs, np.ndarray) and durs.dtype == np.float64 and durs.flags.c_contiguous else f64(durs)
    B, n = d.shape[0], d.shape[1]
    if out is None:
        out = np.empty(B, dtype=SUMMARY_DTYPE)
    check(load().osim_exhaustive_batch(ptr(d, C.c_double), B, n, int(dma), float(sigma), int(n_dev),
                                       out.ctypes.data_as(C.c_void_p)))
    return out


def heuristic_batch(durs, id_rank, dma, sigma, sum_mode, n_dev=1, order=None, makespan=None, n_sims=None):
    """(order [B][n] (uint8; uint32 above 64 tasks), makespan [B], n_sims [B])."""
    d = durs if isinstance(durs, np.ndarray) and durs.dtype == np.float64 and durs.flags.c_contiguous else f64(durs)
    B, n = d.shape[0], d.shape[1]
    if n > WIDE_MAX:
        r = u32(id_rank, (B, n))
        order = np.empty((B, n), dtype=np.uint32) if order is None else order
        makespan = np.empty(B) if makespan is None else makespan
        n_sims = np.empty(B, dtype=np.uint32) if n_sims is None else n_sims
        check(load().osim_heuristic_batch_u32(ptr(d, C.c_double), ptr(r, C.c_uint32), B, n, int(dma), float(sigma),
                                              int(sum_mode), int(n_dev), ptr(order, C.c_uint32),
                                              ptr(makespan, C.c_double), ptr(n_sims, C.c_uint32)))
        return order, makespan, n_sims
    r = u8(id_rank, (B, n))
    order = np.empty((B, n), dtype=np.uint8) if order is None else order
    makespan = np.empty(B) if makespan is None else makespan
    n_sims = np.empty(B, dtype=np.uint32) if n_sims is None else n_sims
    check(load().osim_heuristic_batch(ptr(d, C.c_double), ptr(r, C.c_uint8), B, n, int(dma), float(sigma),
                                      int(sum_mode), int(n_dev), ptr(order, C.c_uint8),
                                      ptr(makespan, C.c_double), ptr(n_sims, C.c_uint32)))
    return order, makespan, n_sims


def timeline(durs, dma, sigma, order):
    d = f64(durs, (-1, 3))
    n = d.shape[0]
    if n > WIDE_MAX:
        return timeline_deps(d, dma, sigma, order)
    o = u8(order)
    st = np.empty((n, 3))
    en = np.empty((n, 3))
    ms = C.c_double()
    idle = np.empty(3)
    check(load().osim_timeline(ptr(d, C.c_double), n, int(dma), float(sigma), ptr(o, C.c_uint8),
                               ptr(st, C.c_double), ptr(en, C.c_double), C.byref(ms), ptr(idle, C.c_double)))
    return st, en, ms.value, idle


def fast_eligible(durs, sigma) -> bool:
    d = f64(durs)
    return bool(load().osim_fast_eligible(ptr(d, C.c_double), d.size // 3, float(sigma)))


def selftest_div(samples: int, seed: int = 1, mode: int = 0) -> int:
    """Mismatches of the fast-path division against IEEE division over
    `samples` operand pairs (mode 0 random, 1 adversarial)."""
    m = C.c_uint64()
    check(load().osim_selftest_div_mode(int(samples), int(seed), int(mode), C.byref(m)))
    return m.value


def fp64_peak_tflops() -> float:
    t = C.c_double()
    check(load().osim_fp64_peak(C.byref(t)))
    return t.value


def interleavings(durs, T, N, dma, sigma, lo, hi, threshold=float("-inf"), n_dev=1, want_makespans=False):
    d = f64(durs, (-1, 3))
    out = OsimSummary()
    below = C.c_uint64()
    ms = np.empty(hi - lo) if want_makespans else None
    check(load().osim_interleavings(ptr(d, C.c_double), int(T), int(N), int(dma), float(sigma), int(lo), int(hi),
                                    float(threshold), int(n_dev), C.byref(out), C.byref(below),
                                    ptr(ms, C.c_double) if ms is not None else None))
    return out.as_dict(), below.value, ms


def eval_sequences(durs, T, N, dma, sigma, labels, n_dev=1):
    d = f64(durs, (-1, 3))
    if T * N > WIDE_MAX:
        lab = u32(labels, (-1, T * N))
        ms = np.empty(lab.shape[0])
        out = OsimSummary()
        check(load().osim_eval_sequences_u32(ptr(d, C.c_double), int(T), int(N), int(dma), float(sigma),
                                             ptr(lab, C.c_uint32), lab.shape[0], int(n_dev), ptr(ms, C.c_double),
                                             C.byref(out)))
        return out.as_dict(), ms
    lab = u8(labels, (-1, T * N))
    ms = np.empty(lab.shape[0])
    out = OsimSummary()
    check(load().osim_eval_sequences(ptr(d, C.c_double), int(T), int(N), int(dma), float(sigma),
                                     ptr(lab, C.c_uint8), lab.shape[0], int(n_dev), ptr(ms, C.c_double),
                                     C.byref(out)))
    return out.as_dict(), ms


def timeline_deps(durs, dma, sigma, order, dep=None, waves=False):
    d = f64(durs, (-1, 3))
    n = d.shape[0]
    st, en, idle = np.empty((n, 3)), np.empty((n, 3)), np.empty(3)
    ms = C.c_double()
    if n > WIDE_MAX:
        o = u32(order)
        dp_ = None if dep is None else np.ascontiguousarray(np.asarray(dep, dtype=np.int32))
        check(load().osim_timeline_u32(ptr(d, C.c_double), n, int(dma), float(sigma), ptr(o, C.c_uint32),
                                       ptr(dp_, C.c_int32) if dp_ is not None else None, int(bool(waves)),
                                       ptr(st, C.c_double), ptr(en, C.c_double), C.byref(ms), ptr(idle, C.c_double)))
        return st, en, ms.value, idle
    o = u8(order)
    dp_ = None if dep is None else np.ascontiguousarray(np.asarray(dep, dtype=np.int8))
    check(load().osim_timeline_deps(ptr(d, C.c_double), n, int(dma), float(sigma), ptr(o, C.c_uint8),
                                    ptr(dp_, C.c_int8) if dp_ is not None else None, int(bool(waves)),
                                    ptr(st, C.c_double), ptr(en, C.c_double), C.byref(ms), ptr(idle, C.c_double)))
    return st, en, ms.value, idle


def micro(durs, dma, sigma, dt, lo, hi, n_dev=1):
    d = f64(durs, (-1, 3))
    ms = np.empty(hi - lo)
    check(load().osim_micro(ptr(d, C.c_double), d.shape[0], int(dma), float(sigma), float(dt), int(lo), int(hi),
                            int(n_dev), ptr(ms, C.c_double)))
    return ms


def micro_timeline(durs, dma, sigma, dt, order):
    d = f64(durs, (-1, 3))
    n = d.shape[0]
    if n > 16:  # above the 4-bit kernels: osim_micro_timeline_u32
        o = u32(order)
        st, en = np.empty((n, 3)), np.empty((n, 3))
        ms = C.c_double()
        check(load().osim_micro_timeline_u32(ptr(d, C.c_double), n, int(dma), float(sigma), float(dt),
                                             ptr(o, C.c_uint32), ptr(st, C.c_double), ptr(en, C.c_double),
                                             C.byref(ms)))
        return st, en, ms.value
    o = u8(order)
    st, en = np.empty((n, 3)), np.empty((n, 3))
    ms = C.c_double()
    check(load().osim_micro_timeline(ptr(d, C.c_double), n, int(dma), float(sigma), float(dt), ptr(o, C.c_uint8),
                                     ptr(st, C.c_double), ptr(en, C.c_double), C.byref(ms)))
    return st, en, ms.value


def harness_batch(durs, id_rank, T, N, dma, sigma, sum_mode, n_dev=1, timeline=False):
    """(makespan [S], n_groups [S], tg_sizes [S][T*N], start/end [S][T*N][3] or None);
    n_groups / tg_sizes are uint8, uint32 above 64 tasks."""
    d = f64(durs).reshape(-1, T * N, 3)
    S = d.shape[0]
    if T * N > WIDE_MAX:
        r = u32(id_rank, (S, T * N))
        ms = np.empty(S)
        ng = np.empty(S, dtype=np.uint32)
        sz = np.zeros((S, T * N), dtype=np.uint32)
        st = np.empty((S, T * N, 3)) if timeline else None
        en = np.empty((S, T * N, 3)) if timeline else None
        check(load().osim_harness_batch_u32(ptr(d, C.c_double), ptr(r, C.c_uint32), S, int(T), int(N), int(dma),
                                            float(sigma), int(sum_mode), int(n_dev), ptr(ms, C.c_double),
                                            ptr(ng, C.c_uint32), ptr(sz, C.c_uint32),
                                            ptr(st, C.c_double) if timeline else None,
                                            ptr(en, C.c_double) if timeline else None))
        return ms, ng, sz, st, en
    r = u8(id_rank, (S, T * N))
    ms = np.empty(S)
    ng = np.empty(S, dtype=np.uint8)
    sz = np.zeros((S, T * N), dtype=np.uint8)
    st = np.empty((S, T * N, 3)) if timeline else None
    en = np.empty((S, T * N, 3)) if timeline else None
    check(load().osim_harness_batch(ptr(d, C.c_double), ptr(r, C.c_uint8), S, int(T), int(N), int(dma),
                                    float(sigma), int(sum_mode), int(n_dev), ptr(ms, C.c_double),
                                    ptr(ng, C.c_uint8), ptr(sz, C.c_uint8),
                                    ptr(st, C.c_double) if timeline else None,
                                    ptr(en, C.c_double) if timeline else None))
    return ms, ng, sz, st, en
