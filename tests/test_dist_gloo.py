"""N>1 path on CPU: world_size-2 gloo process group, rank-range sharding and
the all_gather combine of dist.exhaustive_summary_distributed.  The local
shard reduction is the CPU oracle here (no GPU in this container); the
combine must reproduce the single-process whole-space summary."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import oracle as O
from tests._golden import F, close, durs, load


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_local(d, dma, sigma, lo, hi):
    s, _ = O.exhaustive(d, dma, sigma, lo, hi, threads=2)
    return s


def _worker(rank, world, port, d, dma, sigma, q, interleaved=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1806_10113_b200.dist import exhaustive_summary_distributed

        s = exhaustive_summary_distributed(d, dma, sigma, local_fn=_oracle_local, interleaved=interleaved)
        q.put((rank, s.best, s.best_rank, s.worst, s.count, s.sum, s.sum_log))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,interleaved", [(2, False), (3, False), (2, True), (3, True)])
def test_gloo_sharded_exhaustive_matches_whole_space(world, interleaved):
    # interleaved: the library's partition (512-prefix calls of 3072 ranks at
    # n = 7: two calls, so at world 3 one rank has an empty shard)
    c = load("c1_bk.json")["cases"][3]  # BK25 2-DMA: a unique best at rank 19
    d = np.concatenate([durs(c["durs"]), durs(c["durs"])[:3] * 1.25])  # 7 tasks, 5040 orderings
    dma, sigma = c["dma"], F(c["sigma"])
    whole, _ = O.exhaustive(d, dma, sigma, threads=4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, dma, sigma, q, interleaved)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, best, rank, worst, count, sm, sl in results:
        assert best == whole["best"] and rank == whole["best_rank"] and worst == whole["worst"]
        assert count == whole["count"] == 5040
        assert close(sm, whole["sum"]) and close(sl, whole["sum_log"])
    # every rank holds the identical combined summary
    assert len({r[1:] for r in results}) == 1


def _median_worker(rank, world, port, vals, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1806_10113_b200.dist import median_distributed, numpy_hist, select_kth_distributed, shard

        lo, hi = shard(len(vals), rank, world)
        mine = vals[lo:hi]
        h = numpy_hist(mine)
        med = median_distributed(h, len(vals))
        # starting below the common prefix of the set's min and max
        med2 = median_distributed(h, len(vals), vmin=float(vals.min()), vmax=float(vals.max()))
        k7 = select_kth_distributed(h, 7, vmin=float(vals.min()), vmax=float(vals.max()))
        q.put((rank, med, k7, med2))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("count", [5040, 5039])
def test_gloo_sharded_median_selection(count):
    # the makespans of a 7-task group (with ties) from the pinned oracle
    c = load("c1_bk.json")["cases"][3]
    d = np.concatenate([durs(c["durs"]), durs(c["durs"])[:3] * 1.25])
    _, ms = O.exhaustive(d, c["dma"], F(c["sigma"]), threads=4, makespans=True)
    vals = ms[:count].copy()
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_median_worker, args=(r, world, port, vals, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, med, k7, med2 in res:
        assert med == med2 == float(np.median(vals))
        assert k7 == float(np.sort(vals)[7])


def _oracle_reorder(dd, rr):
    return O.reorder_batch(dd, rr, 2, 0.5, 1, threads=2)


def _oracle_batch(dd):
    from paper_1806_10113_b200 import _capi

    out = np.zeros(dd.shape[0], dtype=_capi.SUMMARY_DTYPE)
    for i in range(dd.shape[0]):
        s, _ = O.exhaustive(dd[i], 2, 0.5, threads=1)
        for k in out.dtype.names:
            out[i][k] = s[k]
    return out


def _batch_worker(rank, world, port, d, r, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1806_10113_b200.dist import exhaustive_summary_batch_distributed, reorder_durs_distributed

        order, ms, sims = reorder_durs_distributed(d, r, 2, 0.5, 1, local_fn=_oracle_reorder)
        summ = exhaustive_summary_batch_distributed(d[:, :6], 2, 0.5, local_fn=_oracle_batch)
        q.put((rank, order, ms, sims, summ))
    finally:
        tdist.destroy_process_group()


def test_gloo_batch_shards_gather_whole_batch():
    # configs 2/5 over 3 ranks: ragged group-range shards (101 groups), the
    # gathered arrays equal the single-process batch on every rank
    from paper_1806_10113_b200 import synth

    B, n = 101, 9
    d = np.stack([synth.real_group("K20", n, 40 + b)[1] for b in range(B)])
    r = np.stack([np.random.default_rng(b).permutation(n) for b in range(B)]).astype(np.uint8)
    want = O.reorder_batch(d, r, 2, 0.5, 1, threads=4)
    want_s = _oracle_batch(d[:, :6])
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(k, world, port, d, r, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, order, ms, sims, summ in res:
        assert np.array_equal(order, want[0]) and np.array_equal(ms, want[1]) and np.array_equal(sims, want[2])
        assert summ.tobytes() == want_s.tobytes()


def test_gloo_batch_smaller_than_world():
    # B = 2 groups over 3 ranks: one rank's group-range shard is empty; it
    # must still join the all_gathers (no reshape error, no hang)
    from paper_1806_10113_b200 import synth

    B, n = 2, 7
    d = np.stack([synth.real_group("K20", n, 70 + b)[1] for b in range(B)])
    r = np.stack([np.random.default_rng(b).permutation(n) for b in range(B)]).astype(np.uint8)
    want = O.reorder_batch(d, r, 2, 0.5, 1, threads=2)
    want_s = _oracle_batch(d[:, :6])
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(k, world, port, d, r, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, order, ms, sims, summ in res:
        assert np.array_equal(order, want[0]) and np.array_equal(ms, want[1]) and np.array_equal(sims, want[2])
        assert summ.tobytes() == want_s.tobytes()


def _pfx_env_worker(rank, world, port, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # rank 1 overrides the suffix length of the library's partition
    if rank == 1:
        os.environ["OSIM_PFX_L"] = "5"
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1806_10113_b200.dist import exhaustive_summary_distributed

        try:
            exhaustive_summary_distributed(d, 2, 0.5, local_fn=_oracle_local, interleaved=True)
            q.put((rank, "ok"))
        except ValueError as e:
            q.put((rank, str(e)))
    finally:
        tdist.destroy_process_group()


def test_gloo_mismatched_partitions_are_rejected():
    # OSIM_PFX_L differing between ranks would double-count or drop
    # orderings: every rank sees every rank's partition and raises
    d = np.stack([[1.0 + i, 2.0 + (i * 7) % 5, 1.5] for i in range(8)])
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pfx_env_worker, args=(k, world, port, d, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all("partitioned the rank space differently" in m for _, m in res)


@pytest.mark.parametrize("fast", [True, False])
def test_shard_ranges_partition_every_space(fast):
    # every ordering of n! in exactly one rank's ranges, for any world size
    import math

    from paper_1806_10113_b200.dist import shard_ranges

    for n in range(1, 13 if fast else 17):
        total = math.factorial(n)
        for world in (1, 2, 3, 5, 8, 13):
            rs = sorted(r for w in range(world) for r in shard_ranges(n, w, world, fast=fast))
            rs = [r for r in rs if r[1] > r[0]]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
