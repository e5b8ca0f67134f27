"""Small invocations of every kernel family for compute-sanitizer
(racecheck / synccheck / memcheck, one tool per run):

    compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_run.py

Covers the prefix-sharing exhaustive kernel with its barrier-free
shared-memory reuse across calls and the fused last-CTA reduce (C4 / C3
windows, interleaved shards, the split small-shard mode), the batched
prefix kernel (C2), the null-stage kernels, the general path, the heuristic
kernels (fast / null-stage / general / wide / any-size), f1 interleavings,
f2 radix selection, f3 harness, f4 micro, and the any-size (u32) paths.
Each result is checked against the oracle so a sanitizer run is also a
parity run."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def same(s, o):
    assert s["count"] == o["count"] and s["best"] == o["best"] and s["best_rank"] == o["best_rank"], (s, o)
    assert s["worst"] == o["worst"]


def main():
    _capi.set_device(0)
    th = os.cpu_count() or 1
    c4, c3 = synth.c4_group(), synth.c3_group()
    # exhaustive prefix kernel: two CTA calls' worth of a C4 window (fused final reduce), sigma 0.375 path
    for d, dma, sg, lo, hi in ((c4, 2, 0.5, 1_000_000, 1_049_152), (c4, 2, 0.375, 5, 30_000), (c3, 1, 1.0, 0, 40_000)):
        s, ms = _capi.exhaustive(d, dma, sg, lo, hi, want_makespans=True)
        o, oms = O.exhaustive(d, dma, sg, lo, hi, threads=th, makespans=True)
        same(s, o)
        assert np.array_equal(ms, oms)
    # interleaved shards (C3 at 8 ranks: the split small-shard mode) -- first two shards
    for r in range(2):
        _capi.exhaustive_shard(c3, 2, 0.5, r, 8)
    # f2: exact median through radix selection
    d9 = synth.real_group("K20", 9, 5)[1]
    s, below, med = _capi.exhaustive_stats(d9, 2, 0.5, 0, math.factorial(9), threshold=60.0)
    _, oms = O.exhaustive(d9, 2, 0.5, threads=th, makespans=True)
    assert med == float(np.median(oms)) and below == int((oms < 60.0).sum())
    # C2 batch prefix kernel and the null-stage batch kernel
    b2 = synth.c2_batch(6)
    out = _capi.exhaustive_batch(b2, 2, 0.5)
    o, _ = O.exhaustive(b2[3], 2, 0.5, threads=th)
    assert out[3]["best"] == o["best"] and out[3]["best_rank"] == o["best_rank"]
    bn = b2.copy()
    bn[:, 2, 0] = 0.0
    out = _capi.exhaustive_batch(bn[:, :7], 1, 1.0)
    o, _ = O.exhaustive(bn[2, :7], 1, 1.0, threads=th)
    assert out[2]["best"] == o["best"]
    # null-stage exhaustive (NullSim) and the general path (durations beyond 2^22)
    n9 = d9.copy()
    n9[4, 2] = 0.0
    same(_capi.exhaustive(n9, 2, 0.5, 0, 20_000)[0], O.exhaustive(n9, 2, 0.5, 0, 20_000, threads=th)[0])
    same(_capi.exhaustive(d9 * 1e23, 2, 0.5, 0, 5_000)[0], O.exhaustive(d9 * 1e23, 2, 0.5, 0, 5_000, threads=th)[0])
    # heuristic kernels: fast (both DMA modes), null-stage, general, wide (20 tasks), any-size (70 tasks)
    for prof in ("nvidia", "phi"):
        _, dma, sg = synth.PROFILES[prof]
        d5, r5 = synth.c5_batch_fast(prof, 300)
        got = _capi.heuristic_batch(d5, r5, dma, sg, 1)
        want = O.reorder_batch(d5, r5, dma, sg, 1, threads=th)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
        dn = d5.copy()
        dn[:, 3, 2] = 0.0
        got = _capi.heuristic_batch(dn, r5, dma, sg, 1)
        assert np.array_equal(got[0], O.reorder_batch(dn, r5, dma, sg, 1, threads=th)[0])
        got = _capi.heuristic_batch(d5[:40] * 1e23, r5[:40], dma, sg, 1)
        assert np.array_equal(got[0], O.reorder_batch(d5[:40] * 1e23, r5[:40], dma, sg, 1, threads=th)[0])
    dw = np.stack([synth.real_group("AMD", 20, 900 + b)[1] for b in range(8)])
    rw = np.stack([np.random.default_rng(b).permutation(20) for b in range(8)]).astype(np.uint8)
    got = _capi.heuristic_batch(dw, rw, 2, 0.375, 1)
    assert np.array_equal(got[0], O.reorder_batch(dw, rw, 2, 0.375, 1, threads=th)[0])
    db = np.stack([synth.real_group("K20", 70, 70 + b)[1] for b in range(3)])
    rb = np.stack([np.random.default_rng(b).permutation(70) for b in range(3)])
    got = _capi.heuristic_batch(db, rb.astype(np.uint32), 2, 0.5, 1)
    assert np.array_equal(got[0], O.reorder_batch(db, rb.astype(np.uint8), 2, 0.5, 1, threads=th)[0])
    # timelines: 16-task general, wide (40), any-size (90, deps + 1-DMA waves)
    rng = np.random.default_rng(5)
    for n in (16, 40, 90):
        d = rng.uniform(0.1, 3.0, (n, 3))
        order = rng.permutation(n)
        st, en, ms, idle = _capi.timeline(d, 1, 1.0, order)
        assert ms == O.simulate(d, order, 1, 1.0).makespan
    T, N = 9, 10
    d = rng.uniform(0.1, 3.0, (T * N, 3))
    labels = rng.permutation(np.repeat(np.arange(T), N))
    cnt, order = [0] * T, []
    for w in labels:
        order.append(w * N + cnt[w])
        cnt[w] += 1
    dep = [(w * N + j - 1 if j else -1) for w in range(T) for j in range(N)]
    _, _, ms, _ = _capi.timeline_deps(d, 1, 1.0, order, dep, waves=True)
    assert ms == O.simulate_seq(d, order, 1, 1.0, dep).makespan
    # eval_perms: 12-task, wide 40, any-size 80
    for n in (12, 40, 80):
        d = rng.uniform(0.1, 3.0, (n, 3))
        perms = np.stack([rng.permutation(n) for _ in range(300)])
        s, ms = _capi.eval_perms(d, 2, 0.5, perms.astype(np.uint8 if n <= 64 else np.uint32))
        if n <= 64:
            assert np.array_equal(ms, O.eval_perms(d, 2, 0.5, perms.astype(np.uint8), threads=th)[1])
    # f1 interleavings (prefix kernels, both DMA modes) and label sequences (wide, any-size)
    d16 = synth.real_group("K20", 16, 41)[1]
    for dma, sg in ((2, 0.5), (1, 1.0)):
        s, _, _ = _capi.interleavings(d16, 4, 4, dma, sg, 1000, 9000)
        same(s, O.interleavings(d16, 4, 4, dma, sg, 1000, 9000, threads=th)[0])
    for T, N in ((4, 5), (7, 10)):
        lab = np.stack([rng.permutation(np.repeat(np.arange(T), N)) for _ in range(64)])
        dd = rng.uniform(0.1, 3.0, (T * N, 3))
        s, ms = _capi.eval_sequences(dd, T, N, 1, 1.0, lab.astype(np.uint8 if T * N <= 64 else np.uint32))
    # f3 harness (16-task, wide, any-size) and f4 micro (sweep, timeline, any-size timeline)
    for T, N in ((4, 3), (8, 4), (9, 8)):
        n = T * N
        dh = np.stack([synth.real_group("K20", n, 300 + s)[1] for s in range(8)])
        rh = np.tile(np.argsort(np.argsort([f"w{w}.{j}" for w in range(T) for j in range(N)])), (8, 1))
        _capi.harness_batch(dh, rh.astype(np.uint8 if n <= 64 else np.uint32), T, N, 2, 0.5, 1, timeline=True)
    d8 = synth.c2_batch(1)[0]
    _capi.micro(d8, 2, 0.5, 0.01, 0, 500)
    _capi.micro_timeline(d8, 1, 1.0, 0.01, list(range(8)))
    _capi.micro_timeline(np.tile(d8, (5, 1)), 2, 0.5, 0.01, list(range(40)))
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
