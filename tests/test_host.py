"""Host-side logic and the C-ABI boundary, without a GPU."""

import ctypes
import math
import os
import re
from itertools import permutations

import numpy as np
import pytest

import paper_1806_10113_b200 as osim
from paper_1806_10113_b200 import _capi, dist, model, search, synth
from tests._golden import F, durs, load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "offsim_b200.h")) as fh:
        src = fh.read()
    return sorted(set(re.findall(r"\b(osim_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_capi.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(_capi.LIB_PATH):
        from paper_1806_10113_b200 import _build

        _build.build()
    lib = ctypes.CDLL(_capi.LIB_PATH)
    for name in header_symbols():
        assert hasattr(lib, name), name
    L = _capi.load()
    assert b"sm_100a" in L.osim_version()


def test_library_without_device_reports_enodev():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    L = _capi.load()
    got = ctypes.c_int(-1)
    assert L.osim_init(0, ctypes.byref(got)) == _capi.OSIM_ENODEV
    assert b"no CUDA device" in L.osim_last_error()


def test_validation_happens_before_the_device():
    p = model.DeviceProfile("p", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=0.5)
    with pytest.raises(ValueError):
        osim.simulate([], p)
    with pytest.raises(ValueError):
        osim.exhaustive_search([], p)
    t = model.TaskSpec("a", fixed_durations=(1.0, 1.0, 1.0))
    with pytest.raises(ValueError):
        osim.exhaustive_search([t], p, cap=0)
    with pytest.raises(ValueError):
        osim.reorder_batch([], p)
    with pytest.raises(ValueError):  # duplicate ids (engine.py:126-127)
        osim.simulate([t, t], p)
    with pytest.raises(osim.UnresolvableDuration):
        osim.simulate([model.TaskSpec("z", htd_bytes=0.0)], p)
    with pytest.raises(RuntimeError):  # prerequisite outside the group: the reference stalls
        osim.simulate([t], p, deps={"a": "b"})
    with pytest.raises(ValueError):
        model.DeviceProfile("bad", 3, 0.0, 1.0, 0.0, 1.0)
    with pytest.raises(ValueError):
        model.DeviceProfile("bad", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=0.0)
    with pytest.raises(ValueError):
        model.TaskSpec("n", fixed_durations=(0.0, 0.0, 0.0))


def test_stage_times_estimators():
    p = model.DeviceProfile("p", 2, 0.01, 6e6, 0.02, 3e6)
    t = model.TaskSpec("t", htd_bytes=6e6, kernel_work=10.0, eta=0.5, gamma=0.1, dth_bytes=3e6)
    assert model.stage_times(t, p) == (0.01 + 1.0, 0.5 * 10.0 + 0.1, 0.02 + 1.0)
    k = model.TaskSpec("k", kernel_work=2.0, eta=1.0)
    assert model.stage_times(k) == (0.0, 2.0, 0.0)
    with pytest.raises(osim.UnresolvableDuration):
        model.stage_times(model.TaskSpec("x", htd_bytes=1.0))
    assert model.classify_task(model.TaskSpec("a", fixed_durations=(1, 2, 1))) is model.TaskDominance.DOMINANT_KERNEL
    eta, gamma = model.fit_kernel_model([(1.0, 3.0), (2.0, 5.0), (3.0, 7.0)])
    assert eta == pytest.approx(2.0) and gamma == pytest.approx(1.0)


def test_recompute_overlap_fig4():
    # Fig. 4 example (tests/test_engine.py:70-76 of the reference)
    p = model.DeviceProfile("fig", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=0.375)
    h = osim.Command("t1", "HtD", 10.0, start=200.0, remaining_work=0.3)
    d = osim.Command("t0", "DtH", 13.0, start=207.0, remaining_work=1.0)
    assert osim.recompute_overlap(h, d, 207.0, p)[0] == pytest.approx(215.0)


def test_id_ranks_follow_python_string_order():
    ts = [model.TaskSpec(i, fixed_durations=(1, 1, 1)) for i in ("CONV-10", "CONV-4", "BS-2", "t")]
    r = model.id_ranks(ts)
    assert [ts[i].id for i in np.argsort(r)] == sorted(t.id for t in ts)


def test_unrank_matches_itertools():
    for n in range(1, 7):
        for r, p in enumerate(permutations(range(n))):
            assert search.unrank(r, n) == p


def test_sample_permutations_match_reference():
    g = load("sampled.json")
    for c in g["cases"]:
        n = len(c["durs"])
        perms = search.sample_permutations(n, c["cap"], c["seed"])
        assert perms[: len(c["orderings"])].tolist() == c["orderings"]


def test_synthetic_inputs_match_reference_generators():
    assert np.array_equal(synth.c3_group(), durs(load("c3_full.json")["durs"]))
    assert np.array_equal(synth.c4_group(), durs(load("c4_sample.json")["durs"]))
    c2 = load("c2_tg.json")
    batch = synth.c2_batch(4)
    for tg in c2["tgs"]:
        assert np.array_equal(batch[tg["tg"]], durs(tg["durs"]))
    for p in load("c5_sample.json")["profiles"]:
        d, r = synth.c5_batch(p["profile"], 20)
        for j in range(20):
            row = p["rows"][j]
            assert np.array_equal(d[j], durs(row["durs"]))
            assert r[j].tolist() == row["id_rank"]
    for c in load("c1_bk.json")["cases"]:
        ids, d = synth.bk_group(c["bk"])
        assert ids == c["ids"] and np.array_equal(d, durs(c["durs"]))


def test_summary_pack_roundtrip_and_combine():
    s = {"best": 1.5, "best_rank": 2**40 + 3, "worst": 9.0, "sum": 10.0, "sum_log": 2.0, "count": 2**33}
    assert dist.unpack(dist.pack(s)) == s
    a = {"best": 2.0, "best_rank": 5, "worst": 3.0, "sum": 5.0, "sum_log": 1.0, "count": 2}
    b = {"best": 2.0, "best_rank": 1, "worst": 4.0, "sum": 6.0, "sum_log": 1.5, "count": 3}
    c = dist.combine([a, b])
    assert c["best_rank"] == 1 and c["worst"] == 4.0 and c["count"] == 5 and c["sum"] == 11.0
    assert dist.shard(10, 0, 3) == (0, 3) and dist.shard(10, 2, 3) == (6, 10)


def test_summary_from_dict():
    s = search.summary_from_dict({"best": 2.0, "best_rank": 3, "worst": 4.0, "sum": 6.0,
                                  "sum_log": math.log(8.0), "count": 2}, 3)
    assert s.best_ordering == (1, 2, 0) and s.mean == 3.0 and s.geomean == pytest.approx(math.sqrt(8.0))


def test_noreorder_host_enumeration_matches_reference():
    from paper_1806_10113_b200 import noreorder as nr
    import hashlib

    g = load("noreorder.json")
    for c in g["cases"]:
        T, N = c["T"], c["N"]
        if c["exhaustive"]:
            assert nr.interleaving_count(T, N) == c["count"]
            assert [list(nr.unrank_labels(r, T, N)) for r in range(len(c["labels_head"]))] == c["labels_head"]
        else:
            lab = nr.sample_interleavings(T, N, c["cap"], c["seed"])
            assert hashlib.sha256(lab.tobytes()).hexdigest() == c["labels_sha256"]


def test_worker_task_draws_match_reference():
    from paper_1806_10113_b200 import workload as wl

    g = load("harness.json")
    for c in g["cases"]:
        if c["bk"] == "real":
            continue
        p = model.DeviceProfile("p", c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))
        sc = wl.Scenario(c["T"], c["N"], wl.load_bk_benchmark(c["bk"]), c["seed"], p)
        flat = [t for row in wl.draw_worker_tasks(sc) for t in row]
        assert [t.id for t in flat] == c["ids"]
        assert [list(t.fixed_durations) for t in flat] == durs(c["durs"]).tolist()


def test_common_prefix_of_value_range():
    import numpy as np

    from paper_1806_10113_b200.dist import common_prefix

    rng = np.random.default_rng(5)
    for _ in range(200):
        v = np.sort(rng.uniform(0.1, 100.0, 50) * 2.0 ** rng.integers(-3, 4))
        p, bits = common_prefix(float(v[0]), float(v[-1]))
        u = v.view(np.uint64)
        assert bits == 0 or all(int(x) >> (64 - bits) == p for x in u)
    assert common_prefix(2.0, 2.0)[1] == 63
    assert common_prefix(0.0, 1.0) == (0, 0)


def test_reorder_batch_single_task_is_not_resolved():
    # heuristic.py:113-114: a one-task group comes back as is, without
    # stage_times (an unresolvable task does not raise) -- big.json "single"
    import paper_1806_10113_b200 as osim
    from tests._golden import load

    g = load("big.json")["single"]
    lone = osim.TaskSpec(g["id"], kernel_work=0.0)
    with pytest.raises(osim.UnresolvableDuration):
        osim.stage_times(lone, None)
    p = osim.DeviceProfile("2dma", 2, 0.01, 6e6, 0.01, 6e6, overlap_sigma=0.5)
    assert [t.id for t in osim.reorder_batch([lone], p)] == g["returned"]
    assert osim.reorder_batch_many([[lone], [lone]], p) == [[lone], [lone]]


def test_all_interleavings_is_sorted_set_of_permutations():
    # the host enumeration used beyond 16 tasks (noreorder.all_interleavings)
    # against workload.py:262-265's sorted(set(permutations(labels)))
    import hashlib
    from itertools import permutations

    from paper_1806_10113_b200.noreorder import all_interleavings, interleaving_count, unrank_labels
    from tests._golden import load

    for T, N in ((1, 3), (2, 2), (2, 3), (3, 2), (3, 3), (4, 2)):
        labels = [w for w in range(T) for _ in range(N)]
        want = sorted(set(permutations(labels)))
        got = all_interleavings(T, N)
        assert [tuple(r) for r in got.tolist()] == want
        assert [unrank_labels(r, T, N) for r in range(interleaving_count(T, N))] == want
    for c in load("big.json")["noreorder"]:
        if c["exhaustive"]:
            lab = all_interleavings(c["T"], c["N"])
            assert len(lab) == c["count"]
            assert hashlib.sha256(lab.astype(np.uint8).tobytes()).hexdigest() == c["labels_sha256"]


def test_micro_simulate_empty_group():
    # micro_core over empty arrays: no commands, makespan 0 (_micro.py:68-71)
    import paper_1806_10113_b200 as osim

    p = osim.DeviceProfile("2dma", 2, 0.01, 6e6, 0.01, 6e6, overlap_sigma=0.5)
    tl = osim.micro_simulate([], p)
    assert tl.commands == [] and tl.makespan == 0.0 and set(tl.idle.values()) == {0.0}
