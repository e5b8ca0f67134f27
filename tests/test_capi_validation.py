"""C-ABI argument validation, without a device.

Every host entry point checks its arguments -- with the reference's error
semantics (empty group, bad profile, unresolvable or invalid durations,
duplicate ids, bad ranges) -- before it touches CUDA, so on a machine with no
GPU an invalid call reports OSIM_EINVAL (never OSIM_ENODEV) and a message
naming the problem.  Runs in the CPU suite.
"""

import math

import numpy as np
import pytest

from paper_1806_10113_b200 import _capi
from paper_1806_10113_b200._capi import UnresolvableDuration

GOOD = np.array([[1.0, 2.0, 0.5], [0.5, 1.0, 2.0], [2.0, 0.5, 1.0]])


def raises(fn, match, exc=ValueError):
    with pytest.raises(exc, match=match):
        fn()


@pytest.mark.parametrize("call", ["exhaustive", "timeline", "micro", "timeline_big"])
def test_group_and_profile_rules(call):
    def run(d, dma=2, sigma=0.5):
        n = np.asarray(d).reshape(-1, 3).shape[0]
        if call == "exhaustive":
            return _capi.exhaustive(d, dma, sigma, 0, math.factorial(min(n, 20)))
        if call == "timeline":
            return _capi.timeline(d, dma, sigma, list(range(n)))
        if call == "timeline_big":  # the any-size entry point directly
            return _capi.timeline_deps(np.concatenate([d, np.ones((65, 3))]) if n else d, dma, sigma,
                                       list(range(n + 65 if n else 0)))
        return _capi.micro(d, dma, sigma, 0.01, 0, 1)

    raises(lambda: run(np.zeros((0, 3))), "non-empty")
    # enumerated spaces stop at 16 tasks; single orderings take any size
    # (above 64 tasks: osim_timeline_u32, validated the same way)
    if call in ("exhaustive", "micro"):
        raises(lambda: run(np.ones((17, 3))), "exceeds the supported maximum")
    raises(lambda: run(GOOD, dma=3), "dma_engines must be 1 or 2")
    for s in (0.0, 1.5, float("nan")):
        raises(lambda s=s: run(GOOD, sigma=s), r"overlap_sigma must be in \(0, 1\]")
    bad = GOOD.copy()
    bad[1, 2] = -1.0
    raises(lambda: run(bad), "task 1: durations must be finite and non-negative")
    bad[1, 2] = float("inf")
    raises(lambda: run(bad), "task 1: durations must be finite and non-negative")
    bad = GOOD.copy()
    bad[2] = 0.0
    if call == "micro":
        # micro_simulate does not apply DeviceSim.submit's checks (oracle.py:72):
        # a task without commands passes validation (here: no device)
        raises(lambda: run(bad), "no CUDA device", _capi.OsimError)
    else:
        raises(lambda: run(bad), "task 2 has no commands", UnresolvableDuration)


def test_rank_ranges():
    raises(lambda: _capi.exhaustive(GOOD, 2, 0.5, 0, 7), "outside")
    raises(lambda: _capi.exhaustive(GOOD, 2, 0.5, 4, 3), "outside")
    raises(lambda: _capi.micro(GOOD, 2, 0.5, 0.01, 0, 7), "bad rank range")
    raises(lambda: _capi.interleavings(GOOD, 3, 1, 2, 0.5, 0, 7), "rank range outside")


def test_orders_must_be_permutations():
    raises(lambda: _capi.timeline(GOOD, 2, 0.5, [0, 0, 1]), "not a permutation")
    raises(lambda: _capi.eval_perms(GOOD, 2, 0.5, np.array([[0, 1, 2], [2, 2, 0]], np.uint8)),
           "row 1 is not a permutation")


def test_batch_limits_and_buffers():
    raises(lambda: _capi.exhaustive_batch(np.ones((4, 13, 3)), 2, 0.5), "supports n <= 12")
    L = _capi.load()
    d = np.ones((2, 3, 3))
    assert L.osim_heuristic_batch(_capi.ptr(d, _capi.C.c_double), None, 2, 3, 2, 0.5, 1, 1, None, None,
                                  None) == _capi.OSIM_EINVAL
    assert b"NULL buffer" in L.osim_last_error()


def test_wide_and_big_limits():
    # above 64 tasks the *_u32 entry points take over: same validation rules,
    # uint32 task ids / id ranks / labels
    big = np.ones((65, 3))
    raises(lambda: _capi.eval_perms(big, 2, 0.5, np.zeros((1, 65), np.uint32)), "perms row 0 is not a permutation")
    raises(lambda: _capi.heuristic_batch(big[None], np.zeros((1, 65), np.uint32), 2, 0.5, 1),
           "id_rank row 0 is not a permutation")
    raises(lambda: _capi.eval_sequences(big, 65, 1, 2, 0.5, np.zeros((1, 65), np.uint32)), "not an interleaving")
    raises(lambda: _capi.harness_batch(big[None], np.zeros((1, 65), np.uint32), 65, 1, 2, 0.5, 1),
           "id_rank row 0 is not a permutation")
    raises(lambda: _capi.timeline(big, 2, 0.5, [0] * 65), "order row 0 is not a permutation")
    raises(lambda: _capi.micro_timeline(np.ones((20, 3)), 2, 0.5, 0.0, list(range(20))), "dt must be positive")
    raises(lambda: _capi.timeline_deps(big, 2, 0.5, list(range(65)), [5] + [-1] * 63 + [64]), "bad dependency")
    huge = np.ones((1, 65536, 3))
    raises(lambda: _capi.heuristic_batch(huge, np.arange(65536, dtype=np.uint32)[None], 2, 0.5, 1),
           "limited to 65535")
    d = np.ones((20, 3))
    raises(lambda: _capi.heuristic_batch(d[None], np.zeros((1, 20), np.uint8), 2, 0.5, 1), "id ranks must be")
    raises(lambda: _capi.eval_perms(d, 2, 0.5, np.zeros((1, 20), np.uint8)), "row 0 is not a permutation")


def test_row_limits():
    raises(lambda: _capi.interleavings(np.ones((17, 3)), 17, 1, 2, 0.5, 0, 1), r"T\*N must be in")
    raises(lambda: _capi.micro(GOOD, 2, 0.5, 0.0, 0, 6), "dt must be positive")
    raises(lambda: _capi.micro_timeline(GOOD, 2, 0.5, -1.0, [0, 1, 2]), "dt must be positive")
