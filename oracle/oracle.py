"""ctypes wrapper around the CPU oracle (oracle/osim_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / --impl reference leg, always as the checker or the
timed CPU baseline -- never by the product package paper_1806_10113_b200.

Parity pinned against the unmodified reference: tests/test_oracle_golden.py
checks this oracle bit-for-bit against tests/golden/*.json, which
tests/golden/make_golden.py produced by running /root/reference's offsim.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libosim_oracle.so")


class OracleSummary(C.Structure):
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


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "osim_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        dp, ip, u8p = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_uint8)
        L.oracle_simulate.argtypes = [dp, C.c_int, C.c_int, C.c_double, ip, C.c_int, ip, dp, dp, dp,
                                      dp, dp, ip]
        L.oracle_exhaustive.argtypes = [dp, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                        C.c_int, C.POINTER(OracleSummary), dp]
        L.oracle_eval_perms.argtypes = [dp, C.c_int, C.c_int, C.c_double, u8p, C.c_uint64, C.c_int,
                                        dp, C.POINTER(OracleSummary)]
        L.oracle_reorder.argtypes = [dp, u8p, C.c_int, C.c_int, C.c_double, C.c_int, u8p, dp,
                                     C.POINTER(C.c_uint32)]
        L.oracle_reorder_batch.argtypes = [dp, u8p, C.c_uint64, C.c_int, C.c_int, C.c_double,
                                           C.c_int, C.c_int, u8p, dp, C.POINTER(C.c_uint32)]
        L.oracle_pysum.argtypes = [dp, C.c_int, C.c_int]
        L.oracle_pysum.restype = C.c_double
        L.oracle_unrank.argtypes = [C.c_uint64, C.c_int, ip]
        L.oracle_stats_get.argtypes = [C.POINTER(C.c_int64)]
        L.oracle_micro.argtypes = [dp, C.c_int, C.c_int, C.c_double, C.c_double, ip, dp, dp, dp]
        L.oracle_simulate_seq.argtypes = [dp, C.c_int, C.c_int, C.c_double, ip, C.c_int, ip, dp, dp, dp, dp]
        L.oracle_unrank_labels.argtypes = [C.c_uint64, C.c_int, C.c_int, ip]
        L.oracle_interleavings.argtypes = [dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                           C.c_int, C.POINTER(OracleSummary), dp]
        L.oracle_eval_sequences.argtypes = [dp, C.c_int, C.c_int, C.c_int, C.c_double, u8p, C.c_uint64, C.c_int,
                                            dp, C.POINTER(OracleSummary)]
        L.oracle_op_stats.argtypes = [dp, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                      C.c_uint64, C.POINTER(C.c_int64)]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def _durs(durs):
    return np.ascontiguousarray(np.asarray(durs, dtype=np.float64).reshape(-1, 3))


@dataclass
class SimResult:
    makespan: float
    k_end: float
    idle: np.ndarray  # HtD, K, DtH
    start: np.ndarray  # [n][3], -1 = null stage
    end: np.ndarray
    steps: int


def simulate(durs, order, dma, sigma, dep=None) -> SimResult:
    d = _durs(durs)
    n = d.shape[0]
    o = np.ascontiguousarray(np.asarray(order, dtype=np.int32))
    dp_ = None if dep is None else np.ascontiguousarray(np.asarray(dep, dtype=np.int32))
    st = np.empty((n, 3))
    en = np.empty((n, 3))
    idle = np.empty(3)
    ms, ke, steps = C.c_double(), C.c_double(), C.c_int()
    rc = lib().oracle_simulate(_p(d, C.c_double), n, int(dma), float(sigma), _p(o, C.c_int), len(o),
                               _p(dp_, C.c_int), _p(st, C.c_double), _p(en, C.c_double), C.byref(ms),
                               _p(idle, C.c_double), C.byref(ke), C.byref(steps))
    if rc:
        raise RuntimeError(f"oracle_simulate rc={rc}")
    return SimResult(ms.value, ke.value, idle, st, en, steps.value)


def exhaustive(durs, dma, sigma, lo=0, hi=None, threads=1, makespans=False):
    d = _durs(durs)
    n = d.shape[0]
    if hi is None:
        hi = int(np.prod(np.arange(1, n + 1, dtype=np.uint64)))
    out = OracleSummary()
    ms = np.empty(hi - lo) if makespans else None
    rc = lib().oracle_exhaustive(_p(d, C.c_double), n, int(dma), float(sigma), lo, hi, threads,
                                 C.byref(out), _p(ms, C.c_double))
    if rc:
        raise RuntimeError(f"oracle_exhaustive rc={rc}")
    return out.as_dict(), ms


def eval_perms(durs, dma, sigma, perms, threads=1):
    d = _durs(durs)
    n = d.shape[0]
    p = np.ascontiguousarray(np.asarray(perms, dtype=np.uint8).reshape(-1, n))
    ms = np.empty(p.shape[0])
    out = OracleSummary()
    rc = lib().oracle_eval_perms(_p(d, C.c_double), n, int(dma), float(sigma), _p(p, C.c_uint8),
                                 p.shape[0], threads, _p(ms, C.c_double), C.byref(out))
    if rc:
        raise RuntimeError(f"oracle_eval_perms rc={rc}")
    return out.as_dict(), ms


def reorder(durs, id_rank, dma, sigma, sum_mode):
    d = _durs(durs)
    n = d.shape[0]
    r = np.ascontiguousarray(np.asarray(id_rank, dtype=np.uint8))
    order = np.empty(n, dtype=np.uint8)
    ms = C.c_double()
    sims = C.c_uint32()
    rc = lib().oracle_reorder(_p(d, C.c_double), _p(r, C.c_uint8), n, int(dma), float(sigma),
                              int(sum_mode), _p(order, C.c_uint8), C.byref(ms), C.byref(sims))
    if rc:
        raise RuntimeError(f"oracle_reorder rc={rc}")
    return order.tolist(), ms.value, sims.value


def reorder_batch(durs, id_rank, dma, sigma, sum_mode, threads=1):
    d = np.ascontiguousarray(np.asarray(durs, dtype=np.float64))
    B, n = d.shape[0], d.shape[1]
    r = np.ascontiguousarray(np.asarray(id_rank, dtype=np.uint8).reshape(B, n))
    order = np.empty((B, n), dtype=np.uint8)
    ms = np.empty(B)
    sims = np.empty(B, dtype=np.uint32)
    rc = lib().oracle_reorder_batch(_p(d, C.c_double), _p(r, C.c_uint8), B, n, int(dma), float(sigma),
                                    int(sum_mode), threads, _p(order, C.c_uint8), _p(ms, C.c_double),
                                    _p(sims, C.c_uint32))
    if rc:
        raise RuntimeError(f"oracle_reorder_batch rc={rc}")
    return order, ms, sims


def pysum(x, sum_mode):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return lib().oracle_pysum(_p(a, C.c_double), len(a), int(sum_mode))


def unrank(rank, n):
    p = np.empty(n, dtype=np.int32)
    lib().oracle_unrank(rank, n, _p(p, C.c_int))
    return p.tolist()


def op_stats(durs, dma, sigma, lo, hi, stride=1):
    """Summed (S, R, O) over ranks lo, lo+stride, ... < hi."""
    d = _durs(durs)
    out = np.zeros(3, dtype=np.int64)
    rc = lib().oracle_op_stats(_p(d, C.c_double), d.shape[0], int(dma), float(sigma), lo, hi, stride,
                               _p(out, C.c_int64))
    if rc:
        raise RuntimeError(f"oracle_op_stats rc={rc}")
    return out


def reorder_op_stats(durs, id_rank, dma, sigma, sum_mode):
    """(S, R, O, simulations) summed over one reorder_batch call's
    simulations, including the final makespan evaluation."""
    lib().oracle_stats_reset()
    reorder(durs, id_rank, dma, sigma, sum_mode)
    out = np.zeros(4, dtype=np.int64)
    lib().oracle_stats_get(_p(out, C.c_int64))
    return out


def simulate_seq(durs, order, dma, sigma, dep=None) -> SimResult:
    """workload.simulate_sequence: deps gate + 1-DMA wave split."""
    d = _durs(durs)
    n = d.shape[0]
    o = np.ascontiguousarray(np.asarray(order, dtype=np.int32))
    dp_ = None if dep is None else np.ascontiguousarray(np.asarray(dep, dtype=np.int32))
    st, en, idle = np.empty((n, 3)), np.empty((n, 3)), np.empty(3)
    ms = C.c_double()
    rc = lib().oracle_simulate_seq(_p(d, C.c_double), n, int(dma), float(sigma), _p(o, C.c_int), len(o),
                                   _p(dp_, C.c_int), _p(st, C.c_double), _p(en, C.c_double), C.byref(ms),
                                   _p(idle, C.c_double))
    if rc:
        raise RuntimeError(f"oracle_simulate_seq rc={rc}")
    return SimResult(ms.value, float("nan"), idle, st, en, -1)


def unrank_labels(rank, T, N):
    p = np.empty(T * N, dtype=np.int32)
    lib().oracle_unrank_labels(rank, T, N, _p(p, C.c_int))
    return p.tolist()


def interleavings(durs, T, N, dma, sigma, lo=0, hi=None, threads=1, makespans=False):
    import math

    d = np.ascontiguousarray(np.asarray(durs, dtype=np.float64).reshape(-1, 3))
    if hi is None:
        hi = math.factorial(T * N) // math.factorial(N) ** T
    out = OracleSummary()
    ms = np.empty(hi - lo) if makespans else None
    rc = lib().oracle_interleavings(_p(d, C.c_double), T, N, int(dma), float(sigma), lo, hi, threads,
                                    C.byref(out), _p(ms, C.c_double))
    if rc:
        raise RuntimeError(f"oracle_interleavings rc={rc}")
    return out.as_dict(), ms


def eval_sequences(durs, T, N, dma, sigma, labels, threads=1):
    d = np.ascontiguousarray(np.asarray(durs, dtype=np.float64).reshape(-1, 3))
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.uint8).reshape(-1, T * N))
    ms = np.empty(lab.shape[0])
    out = OracleSummary()
    rc = lib().oracle_eval_sequences(_p(d, C.c_double), T, N, int(dma), float(sigma), _p(lab, C.c_uint8),
                                     lab.shape[0], threads, _p(ms, C.c_double), C.byref(out))
    if rc:
        raise RuntimeError(f"oracle_eval_sequences rc={rc}")
    return out.as_dict(), ms


def micro(durs, order, dma, sigma, dt):
    """_micro_core: (makespan, start[n][3], end[n][3]) by task index."""
    d = _durs(durs)
    n = d.shape[0]
    o = np.ascontiguousarray(np.asarray(order, dtype=np.int32))
    st, en = np.empty((n, 3)), np.empty((n, 3))
    ms = C.c_double()
    rc = lib().oracle_micro(_p(d, C.c_double), n, int(dma), float(sigma), float(dt), _p(o, C.c_int),
                            _p(st, C.c_double), _p(en, C.c_double), C.byref(ms))
    if rc:
        raise RuntimeError(f"oracle_micro rc={rc}")
    return ms.value, st, en
