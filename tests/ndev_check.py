"""Run in a subprocess by tests/test_gpu_parity.py::test_virtual_multi_device_paths
with OSIM_VIRTUAL_DEVICES set: every C-ABI entry point that shards over
n_dev devices, at n_dev = 2..k, against its n_dev = 1 result (bit-exact for
makespans, ranks, orders, counts; 1e-12 relative for the Sigma / Sigma-log sums
whose summation order follows the partition) and against the oracle.

    OSIM_VIRTUAL_DEVICES=4 python tests/ndev_check.py
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b))


def same_summary(a, b):
    assert a["count"] == b["count"] and a["best"] == b["best"] and a["best_rank"] == b["best_rank"], (a, b)
    assert a["worst"] == b["worst"], (a, b)
    assert close(a["sum"], b["sum"]) and close(a["sum_log"], b["sum_log"]), (a, b)


def main():
    k = int(os.environ["OSIM_VIRTUAL_DEVICES"])
    assert _capi.init() == k, "library did not expose the virtual devices"
    thr = os.cpu_count() or 1
    c3 = synth.c3_group()
    c4 = synth.c4_group()
    d9 = synth.real_group("K20", 9, 5)[1]
    null9 = d9.copy()
    null9[3, 0] = 0.0
    big = c4 * 1e23  # the general path (durations outside the fast range)
    checked = []
    for nd in range(2, k + 1):
        # osim_exhaustive: fast, null-stage, general paths; with makespans
        for d, dma, sg, lo, hi in ((c3, 2, 0.5, 0, 3628800), (d9, 1, 1.0, 1000, 300000), (null9, 2, 0.375, 0, 362880),
                                   (big[:9], 2, 0.5, 5, 200005), (c4, 2, 0.5, 7_000_000, 7_000_011)):
            s1, m1 = _capi.exhaustive(d, dma, sg, lo, hi, n_dev=1, want_makespans=True)
            sn, mn = _capi.exhaustive(d, dma, sg, lo, hi, n_dev=nd, want_makespans=True)
            same_summary(sn, s1)
            assert np.array_equal(m1, mn)
        o, _ = O.exhaustive(d9, 1, 1.0, 1000, 300000, threads=thr)
        same_summary(_capi.exhaustive(d9, 1, 1.0, 1000, 300000, n_dev=nd)[0], o)
        # osim_exhaustive_stats (median from per-device histograms summed on the host)
        for d, dma, sg in ((c3, 2, 0.5), (null9, 1, 1.0)):
            tot = math.factorial(d.shape[0])
            s1, b1, m1 = _capi.exhaustive_stats(d, dma, sg, 0, tot, threshold=69.0, n_dev=1)
            sn, bn, mn = _capi.exhaustive_stats(d, dma, sg, 0, tot, threshold=69.0, n_dev=nd)
            same_summary(sn, s1)
            assert b1 == bn and m1 == mn, (b1, bn, m1, mn)
            _, ms = _capi.exhaustive(d, dma, sg, 0, tot, want_makespans=True)
            assert mn == float(np.median(ms)) and bn == int((ms < 69.0).sum())
        # osim_eval_perms
        rng = np.random.default_rng(nd)
        perms = np.array([rng.permutation(12) for _ in range(5000)], dtype=np.uint8)
        s1, m1 = _capi.eval_perms(c4, 2, 0.5, perms, n_dev=1)
        sn, mn = _capi.eval_perms(c4, 2, 0.5, perms, n_dev=nd)
        assert np.array_equal(m1, mn)
        same_summary(sn, s1)
        # osim_exhaustive_batch (group-range shards)
        b2 = synth.c2_batch(301)
        o1 = _capi.exhaustive_batch(b2, 2, 0.5, n_dev=1)
        on = _capi.exhaustive_batch(b2, 2, 0.5, n_dev=nd)
        assert o1.tobytes() == on.tobytes()
        # osim_heuristic_batch: fast path, null stages (re-run per shard), 1-DMA, > 16 tasks
        for prof in ("nvidia", "phi"):
            d5, r5 = synth.c5_batch_fast(prof, 3001)
            _, dma, sg = synth.PROFILES[prof]
            a1 = _capi.heuristic_batch(d5, r5, dma, sg, 1, n_dev=1)
            an = _capi.heuristic_batch(d5, r5, dma, sg, 1, n_dev=nd)
            for x, y in zip(a1, an):
                assert np.array_equal(x, y)
            dn = d5.copy()
            dn[1500:, 2, 2] = 0.0  # the later shards are not fast-eligible
            a1 = _capi.heuristic_batch(dn, r5, dma, sg, 1, n_dev=1)
            an = _capi.heuristic_batch(dn, r5, dma, sg, 1, n_dev=nd)
            for x, y in zip(a1, an):
                assert np.array_equal(x, y)
            want = O.reorder_batch(dn[1490:1510], r5[1490:1510], dma, sg, 1, threads=thr)
            assert np.array_equal(an[0][1490:1510], want[0]) and np.array_equal(an[1][1490:1510], want[1])
        dw = np.stack([synth.real_group("AMD", 20, 900 + b)[1] for b in range(37)])
        rw = np.stack([np.random.default_rng(b).permutation(20) for b in range(37)]).astype(np.uint8)
        a1 = _capi.heuristic_batch(dw, rw, 2, 0.375, 1, n_dev=1)
        an = _capi.heuristic_batch(dw, rw, 2, 0.375, 1, n_dev=nd)
        for x, y in zip(a1, an):
            assert np.array_equal(x, y)
        # an invalid group in the last shard: the reference's error, every device drained
        bad = d5.copy()
        bad[2999, 4, 1] = -1.0
        try:
            _capi.heuristic_batch(bad, r5, 1, 1.0, 1, n_dev=nd)
            raise AssertionError("negative duration accepted")
        except ValueError:
            pass
        a2 = _capi.heuristic_batch(d5, r5, 1, 1.0, 1, n_dev=nd)  # the devices are usable afterwards
        assert np.array_equal(a2[0], _capi.heuristic_batch(d5, r5, 1, 1.0, 1)[0])
        # osim_interleavings / osim_eval_sequences (f1)
        d16 = synth.real_group("K20", 16, 41)[1]
        s1, _, _ = _capi.interleavings(d16, 4, 4, 2, 0.5, 10_000, 2_000_000, threshold=70.0, n_dev=1)
        sn, _, _ = _capi.interleavings(d16, 4, 4, 2, 0.5, 10_000, 2_000_000, threshold=70.0, n_dev=nd)
        same_summary(sn, s1)
        labels = np.array([rng.permutation(np.repeat(np.arange(4), 4)) for _ in range(999)], dtype=np.uint8)
        e1 = _capi.eval_sequences(d16, 4, 4, 1, 1.0, labels, n_dev=1)
        en = _capi.eval_sequences(d16, 4, 4, 1, 1.0, labels, n_dev=nd)
        assert np.array_equal(e1[1], en[1])
        same_summary(en[0], e1[0])
        # osim_micro (f4) and osim_harness_batch (f3)
        d8 = synth.c2_batch(1)[0]
        u1 = _capi.micro(d8, 2, 0.5, 0.01, 0, 4000, n_dev=1)
        un = _capi.micro(d8, 2, 0.5, 0.01, 0, 4000, n_dev=nd)
        assert np.array_equal(np.asarray(u1), np.asarray(un))
        dh = np.stack([synth.real_group("K20", 12, 20_000 + s)[1] for s in range(203)])
        rh = np.tile(np.argsort(np.argsort([f"w{w}.{j}" for w in range(4) for j in range(3)])).astype(np.uint8),
                     (203, 1))
        h1 = _capi.harness_batch(dh, rh, 4, 3, 2, 0.5, 1, n_dev=1)
        hn = _capi.harness_batch(dh, rh, 4, 3, 2, 0.5, 1, n_dev=nd)
        for x, y in zip(h1[:3], hn[:3]):
            assert np.array_equal(x, y)
        checked.append(nd)
    print("ndev ok", checked)


if __name__ == "__main__":
    main()
