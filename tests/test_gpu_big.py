"""Groups of more than 64 tasks (csrc/osim_big.cuh, the *_u32 entry points)
and the other drop-in divergences of round 1, against reference-generated
goldens (tests/golden/big.json: make_golden.py gen_big) and the oracle:
engine.simulate (engine.py:252-263), simulate_sequence (workload.py:277-304),
reorder_batch (heuristic.py:105-125), sampled exhaustive_search
(oracle.py:98-136), noreorder_distribution beyond 16 tasks
(workload.py:259-327), micro_simulate beyond 16 tasks (oracle.py:60-95) and
the proxy-thread harness beyond 64 tasks (workload.py:197-256).  Bit-exact."""

import hashlib
import os

import numpy as np
import pytest

import paper_1806_10113_b200 as osim
from oracle import oracle as O
from paper_1806_10113_b200 import _capi
from tests._golden import F, durs, fl, load, sha

pytestmark = pytest.mark.gpu


def _check_timeline(st, en, c, n):
    for t in range(n):
        for k in range(3):
            if c["start"][t][k] is None:
                assert st[t, k] == -1.0
            else:
                assert st[t, k] == F(c["start"][t][k]) and en[t, k] == F(c["end"][t][k]), (n, t, k)


def _prof(c):
    return osim.DeviceProfile("g", c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))


def test_big_timelines_bit_exact():
    g = load("big.json")
    for c in g["timelines"]:
        st, en, ms, idle = _capi.timeline(durs(c["durs"]), c["dma"], F(c["sigma"]), c["order"])
        assert ms == F(c["makespan"]) and idle.tolist() == fl(c["idle"]), c["n"]
        _check_timeline(st, en, c, c["n"])
    for c in g["sequences"]:
        T, N = c["T"], c["N"]
        cnt = [0] * T
        order = []
        for w in c["labels"]:
            order.append(w * N + cnt[w])
            cnt[w] += 1
        dep = [(w * N + j - 1 if j else -1) for w in range(T) for j in range(N)]
        st, en, ms, idle = _capi.timeline_deps(durs(c["durs"]), c["dma"], F(c["sigma"]), order, dep,
                                               waves=(c["dma"] == 1))
        assert ms == F(c["makespan"]) and idle.tolist() == fl(c["idle"]), (T, N)
        _check_timeline(st, en, c, T * N)


def test_big_simulate_and_sequence_dropins():
    g = load("big.json")
    for c in g["timelines"][:4]:
        d = durs(c["durs"])
        tasks = [osim.TaskSpec(f"t{i}", fixed_durations=tuple(d[i])) for i in c["order"]]
        tl = osim.simulate(tasks, _prof(c))
        assert tl.makespan == F(c["makespan"]) and [tl.idle[k] for k in osim.KINDS] == fl(c["idle"])
        assert [osim.KINDS.index(x.kind) for x in tl.commands] == c["sorted_kinds"]
        assert [int(x.task_id[1:]) for x in tl.commands] == c["sorted_tasks"]
    from paper_1806_10113_b200 import noreorder as nr

    for c in g["sequences"]:
        T, N = c["T"], c["N"]
        d = durs(c["durs"])
        grid = [[osim.TaskSpec(f"w{w}.{j}", fixed_durations=tuple(d[w * N + j])) for j in range(N)]
                for w in range(T)]
        cnt = [0] * T
        seq = []
        for w in c["labels"]:
            seq.append(grid[w][cnt[w]])
            cnt[w] += 1
        deps = {grid[w][j].id: grid[w][j - 1].id for w in range(T) for j in range(1, N)}
        tl = nr.simulate_sequence(seq, _prof(c), deps)
        assert tl.makespan == F(c["makespan"]) and [tl.idle[k] for k in osim.KINDS] == fl(c["idle"])


def test_big_timelines_vs_oracle_fuzz():
    # random groups of 65..320 tasks (null stages, integer ties, both DMA modes)
    rng = np.random.default_rng(650)
    for c in range(24):
        n = int(rng.integers(65, 321))
        d = rng.uniform(0.1, 5.0, (n, 3)) if c % 2 else rng.integers(0, 6, (n, 3)).astype(np.float64)
        d[rng.random((n, 3)) < 0.1] = 0.0
        d[:, 1] = np.where(d.sum(1) == 0.0, 1.0, d[:, 1])
        order = rng.permutation(n)
        dma, sigma = 1 + c % 2, [0.5, 0.375, 1.0, 0.8][c % 4]
        st, en, ms, idle = _capi.timeline(d, dma, sigma, order)
        o = O.simulate(d, order, dma, sigma)
        assert ms == o.makespan and idle.tolist() == list(o.idle), (n, dma, sigma)
        assert np.array_equal(st, o.start) and np.array_equal(en, o.end)


def test_big_heuristic_goldens_and_dropin():
    g = load("big.json")
    mode = g["meta"]["sum_mode"]
    assert mode == osim.SUM_MODE
    for c in g["heuristic"]:
        order, ms, sims = _capi.heuristic_batch(durs(c["durs"])[None], np.array(c["id_rank"], np.uint32)[None],
                                                c["dma"], F(c["sigma"]), mode)
        assert order[0].tolist() == c["order"] and ms[0] == F(c["makespan"]) and sims[0] == c["n_sims"], c["n"]
    # through the drop-in with the golden's string ids (tie order = Python string order)
    c = [x for x in g["heuristic"] if x["profile"] == "rand" and x["n"] == 70][0]
    d = durs(c["durs"])
    tasks = [osim.TaskSpec(c["ids"][i], fixed_durations=tuple(d[i])) for i in range(c["n"])]
    out = osim.reorder_batch(tasks, _prof(c))
    assert [c["ids"].index(t.id) for t in out] == c["order"]


def test_big_heuristic_batch_vs_oracle():
    # a batch of 80-task groups (several groups per CTA round) against the oracle
    from paper_1806_10113_b200 import synth

    mode = osim.SUM_MODE
    B, n = 24, 80
    for prof in ("nvidia", "phi"):
        _, dma, sigma = synth.PROFILES[prof]
        dev = {"nvidia": "K20", "phi": "PHI"}[prof]
        d = np.stack([synth.real_group(dev, n, 800 + b)[1] for b in range(B)])
        r = np.stack([np.random.default_rng(b).permutation(n) for b in range(B)])
        order, ms, sims = _capi.heuristic_batch(d, r.astype(np.uint32), dma, sigma, mode)
        oo, om, osims = O.reorder_batch(d, r.astype(np.uint8), dma, sigma, mode, threads=os.cpu_count() or 4)
        assert np.array_equal(order, oo) and np.array_equal(ms, om) and np.array_equal(sims, osims)


def test_big_sampled_search():
    from paper_1806_10113_b200.search import sample_permutations

    for c in load("big.json")["sampled"]:
        d = durs(c["durs"])
        tasks = [osim.TaskSpec(f"t{i}", fixed_durations=tuple(d[i])) for i in range(c["n"])]
        rep = osim.exhaustive_search(tasks, _prof(c), cap=c["cap"], seed=c["seed"])
        assert rep.exhaustive is False
        assert sha(np.array(rep.makespans)) == c["makespans_sha256"]
        assert [int(x[1:]) for x in rep.best_ordering] == c["best_ordering"]
        assert rep.best == F(c["best"]) and rep.median == F(c["median"]) and rep.worst == F(c["worst"])
        assert rep.geomean == F(c["geomean"]) or abs(rep.geomean - F(c["geomean"])) <= 1e-12 * F(c["geomean"])
        perms = sample_permutations(c["n"], c["cap"], c["seed"])
        assert hashlib.sha256(perms.astype(np.uint32).tobytes()).hexdigest() == c["orderings_sha256"]
        s, ms = _capi.eval_perms(d, c["dma"], F(c["sigma"]), perms)
        assert s["best_rank"] == c["argmin"] and sha(ms) == c["makespans_sha256"]


def test_big_noreorder_distributions():
    # exhaustive beyond 16 tasks (2 workers x 9 and x 10: 48,620 / 184,756
    # sequences in sorted(set(permutations)) order) and sampled beyond 64
    from paper_1806_10113_b200 import noreorder as nr

    for c in load("big.json")["noreorder"]:
        d = np.array([[[F(x) for x in r] for r in row] for row in c["durs"]])
        labels, ms, summ, exhaustive = nr.distribution_durs(d, c["dma"], F(c["sigma"]), c["cap"], c["seed"])
        assert exhaustive is c["exhaustive"] and len(ms) == c["count"]
        assert hashlib.sha256(np.asarray(labels, dtype=np.uint8).tobytes()).hexdigest() == c["labels_sha256"]
        assert hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest() == c["makespans_sha256"]
        assert summ["best_rank"] == c["argmin"] and summ["best"] == F(c["best"]) and summ["worst"] == F(c["worst"])
        assert float(np.median(ms)) == F(c["median"])


def test_big_micro_simulate():
    for c in load("big.json")["micro"]:
        n = c["n"]
        d = durs(c["durs"])
        st, en, ms = _capi.micro_timeline(d, c["dma"], F(c["sigma"]), F(c["dt"]), c["order"])
        assert ms == F(c["makespan"]), n
        _check_timeline(st, en, c, n)
        tasks = [osim.TaskSpec(f"t{i}", fixed_durations=tuple(d[i])) for i in c["order"]]
        tl = osim.micro_simulate(tasks, _prof(c), dt=F(c["dt"]))
        assert tl.makespan == F(c["makespan"]) and [tl.idle[k] for k in osim.KINDS] == fl(c["idle"])


def test_big_harness():
    g = load("big.json")
    mode = g["meta"]["sum_mode"]
    for c in g["harness"]:
        d = durs(c["durs"])[None]
        r = np.array(c["id_rank"], dtype=np.uint32)[None]
        ms, ng, sz, st, en = _capi.harness_batch(d, r, c["T"], c["N"], c["dma"], F(c["sigma"]), mode, timeline=True)
        assert ms[0] == F(c["makespan"]) and sz[0, : ng[0]].tolist() == c["tg_sizes"], (c["T"], c["N"])
        assert not sz[0, ng[0]:].any()
    from paper_1806_10113_b200 import workload as wl

    c = g["harness"][0]  # 5 workers x 14 tasks of a BK pool, through run_scenario
    p = osim.DeviceProfile("p", c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))
    sc = wl.Scenario(c["T"], c["N"], wl.load_bk_benchmark(c["bk"]), c["seed"], p)
    res = wl.run_scenario(sc, evaluate_noreorder=True, cap=200)  # NoReorder sampled over 70-task sequences
    assert res.heuristic_makespan == F(c["makespan"]) and res.tg_sizes == c["tg_sizes"]
    assert [res.timeline.idle[k] for k in osim.KINDS] == fl(c["idle"])
    assert len(res.noreorder.makespans) == 200
