"""The reference suite's own checks, restated against the B200 drop-in.

SURVEY.md §4 lists what pkg/tests pins for this path: exact timelines of
small cases (tests/test_engine.py:22-67), structural invariants over every
ordering of the BK sets (test_engine.py:96-153), the heuristic's selection
rules and permutation property (tests/test_heuristic.py:22-128), the
exhaustive search report (tests/test_oracle.py:51-93), and the acceptance
criteria 1-6 (tests/test_acceptance.py:70-131).  Each is restated here
through `paper_1806_10113_b200`'s public API (the CUDA library underneath);
where the reference compares with `approx` and the value is exact, the
check here is exact.
"""

from itertools import permutations

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1806_10113_b200 as osim
from paper_1806_10113_b200.engine import KIND_DTH, KIND_HTD, KIND_K

pytestmark = pytest.mark.gpu

DT = 0.001  # ms (the reference's micro-step)
BK = ["BK0", "BK25", "BK50", "BK75", "BK100"]


# the bundled profiles (data/profiles/one_dma.json, two_dma.json)
@pytest.fixture(scope="module")
def one_dma():
    return osim.DeviceProfile("generic-1dma", 1, 0.02, 6.0, 0.02, 6.0, overlap_sigma=1.0)


@pytest.fixture(scope="module")
def two_dma():
    return osim.DeviceProfile("generic-2dma", 2, 0.01, 6.0, 0.01, 6.0, overlap_sigma=0.5)


@pytest.fixture(scope="module")
def synthetic():
    return {t.id: t for t in osim.load_table2_tasks()}


def spans(tl):
    return {(c.task_id, c.kind): (c.start, c.end) for c in tl.commands}


def task(tid, h, k, d):
    return osim.TaskSpec(id=tid, fixed_durations=(float(h), float(k), float(d)))


def bk(name):
    return list(osim.load_bk_benchmark(name).tasks)


# ---- exact small cases (test_engine.py:22-67) ---------------------------------

def test_single_task_is_a_chain(two_dma, synthetic):
    tl = osim.simulate([synthetic["T0"]], two_dma)
    assert tl.makespan == 10.0
    assert spans(tl) == {("T0", KIND_HTD): (0.0, 1.0), ("T0", KIND_K): (1.0, 9.0), ("T0", KIND_DTH): (9.0, 10.0)}


def test_identical_tasks_serialize_on_the_kernel_engine(synthetic):
    p = osim.DeviceProfile("sigma1", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=1.0)
    tl = osim.simulate([synthetic["T0"], task("T0b", 1, 8, 1)], p)
    assert tl.makespan == 18.0
    assert spans(tl) == {
        ("T0", KIND_HTD): (0.0, 1.0), ("T0b", KIND_HTD): (1.0, 2.0),
        ("T0", KIND_K): (1.0, 9.0), ("T0b", KIND_K): (9.0, 17.0),
        ("T0", KIND_DTH): (9.0, 10.0), ("T0b", KIND_DTH): (17.0, 18.0),
    }


def test_null_stages_make_no_commands(two_dma):
    tl = osim.simulate([task("k-only", 0, 5, 0)], two_dma)
    assert [c.kind for c in tl.commands] == [KIND_K] and tl.makespan == 5.0


def test_empty_group_is_rejected(two_dma):
    with pytest.raises(ValueError):
        osim.simulate([], two_dma)


def test_full_overlap_doubles_both_transfers():
    # criterion 5 as well (test_acceptance.py:112-131)
    p = osim.DeviceProfile("s5", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=0.5)
    full = osim.simulate([task("out", 0, 0, 10), task("in", 10, 0, 0)], p)
    assert all(c.end == 20.0 for c in full.commands)
    zero = spans(osim.simulate([task("A", 0, 12, 5), task("B", 10, 0, 0)], p))
    assert zero[("B", KIND_HTD)] == (0.0, 10.0) and zero[("A", KIND_DTH)] == (12.0, 17.0)


def test_recompute_overlap_fig4():
    p = osim.DeviceProfile("fig", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=0.375)
    htd = osim.Command("t1", KIND_HTD, 10.0, start=200.0, remaining_work=0.3)
    dth = osim.Command("t0", KIND_DTH, 13.0, start=207.0, remaining_work=1.0)
    assert osim.recompute_overlap(htd, dth, 207.0, p)[0] == pytest.approx(215.0)


# ---- structural invariants over every BK ordering (test_engine.py:96-153) ----

@pytest.fixture(scope="module")
def sweeps(one_dma, two_dma):
    out = {}
    for name in BK:
        for pname, p in (("1dma", one_dma), ("2dma", two_dma)):
            out[(name, pname)] = [(perm, osim.simulate(list(perm), p)) for perm in permutations(bk(name))]
    return out


@pytest.mark.parametrize("name", BK)
def test_invariants_two_dma(name, sweeps):
    tasks = bk(name)
    serial = sum(sum(t.fixed_durations) for t in tasks)
    critical = max(sum(t.fixed_durations) for t in tasks)
    for _, tl in sweeps[(name, "2dma")]:
        s = spans(tl)
        for tid in {c.task_id for c in tl.commands}:  # dependency soundness
            assert s[(tid, KIND_K)][0] >= s[(tid, KIND_HTD)][1]
            assert s[(tid, KIND_DTH)][0] >= s[(tid, KIND_K)][1]
        for kind in (KIND_HTD, KIND_K, KIND_DTH):  # FIFO per queue
            cs = tl.commands_of_kind(kind)
            assert [c.end for c in cs] == sorted(c.end for c in cs)
            assert [c.start for c in cs] == sorted(c.start for c in cs)
        ks = tl.commands_of_kind(KIND_K)  # one kernel engine
        assert all(b.start >= a.end - 1e-9 for a, b in zip(ks, ks[1:]))
        assert critical - 1e-9 <= tl.makespan <= serial + 1e-9


@pytest.mark.parametrize("name", BK)
def test_invariants_one_dma(name, sweeps):
    # criterion 6 (test_acceptance.py:134-152)
    for _, tl in sweeps[(name, "1dma")]:
        xs = sorted((c for c in tl.commands if c.kind != KIND_K), key=lambda c: c.start)
        assert all(b.start >= a.end - 1e-9 for a, b in zip(xs, xs[1:]))
        first_dth = min(c.start for c in tl.commands_of_kind(KIND_DTH))
        last_htd = max(c.end for c in tl.commands_of_kind(KIND_HTD))
        assert first_dth >= last_htd - 1e-9


@pytest.mark.parametrize("name", BK)
def test_work_conservation_at_sigma_one(name):
    p = osim.DeviceProfile("s1", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=1.0)
    for perm in permutations(bk(name)):
        for c in osim.simulate(list(perm), p).commands:
            assert c.end - c.start == pytest.approx(c.nominal_duration)


# ---- heuristic (test_heuristic.py:22-128) ---------------------------------------

def test_first_task_rules(two_dma, synthetic):
    assert osim.select_first_task([synthetic[i] for i in ("T0", "T1", "T2", "T3")], two_dma).id == "T0"
    assert osim.select_first_task([task("a", 1, 4, 1), task("b", 2, 5, 2)], two_dma).id == "b"
    assert osim.select_first_task([synthetic["T5"]], two_dma) is synthetic["T5"]


def test_next_task_rules(two_dma, synthetic):
    assert osim.select_next_task([synthetic["T4"], synthetic["T7"]], [synthetic["T0"]], two_dma).id == "T4"
    assert osim.select_next_task([synthetic["T6"]], [synthetic["T0"]], two_dma).id == "T6"
    twins = [task("b", 2, 2, 2), task("a", 2, 2, 2)]
    assert osim.select_next_task(twins, [task("z", 1, 8, 1)], two_dma).id == "a"


def test_last_tasks_rules(two_dma, synthetic):
    ot = [synthetic["T0"], synthetic["T1"]]
    a, b = osim.select_last_tasks([synthetic["T4"], synthetic["T5"]], ot, two_dma)
    assert osim.simulate(ot + [a, b], two_dma).makespan <= osim.simulate(ot + [b, a], two_dma).makespan
    _, last = osim.select_last_tasks([task("no-dth", 2, 2, 0), task("with-dth", 2, 2, 1)],
                                     [task("head", 1, 30, 1)], two_dma)
    assert last.id == "no-dth"
    x, y = osim.select_last_tasks([task("x", 2, 2, 2), task("y", 2, 2, 2)], [task("head", 1, 8, 1)], two_dma)
    assert {x.id, y.id} == {"x", "y"}


def test_reorder_batch_rules(two_dma, synthetic):
    assert osim.reorder_batch([synthetic["T2"]], two_dma) == [synthetic["T2"]]
    tg = [task(f"c{i}", 6, 2, 2) for i in range(4)]
    assert sorted(t.id for t in osim.reorder_batch(tg, two_dma)) == sorted(t.id for t in tg)
    rep = osim.exhaustive_search(tg, two_dma)
    assert rep.best == rep.worst
    bk25 = bk("BK25")
    assert [t.id for t in osim.reorder_batch(bk25, two_dma)] == [t.id for t in osim.reorder_batch(bk25, two_dma)]


@settings(max_examples=40, deadline=None)
@given(st.lists(st.tuples(*(st.floats(min_value=0.1, max_value=8.0),) * 3), min_size=1, max_size=8))
def test_reorder_batch_is_a_permutation(stage_triples):
    p = osim.DeviceProfile("generic-2dma", 2, 0.01, 6.0, 0.01, 6.0, overlap_sigma=0.5)
    tg = [task(f"t{i}", *s) for i, s in enumerate(stage_triples)]
    assert sorted(t.id for t in osim.reorder_batch(tg, p)) == sorted(t.id for t in tg)


# ---- exhaustive search report (test_oracle.py:51-93) ----------------------------

def test_exhaustive_report(two_dma, synthetic):
    tasks = bk("BK50")
    rep = osim.exhaustive_search(tasks, two_dma)
    assert len(rep.makespans) == 24 and rep.exhaustive
    by_id = {t.id: t for t in tasks}
    assert osim.simulate([by_id[i] for i in rep.best_ordering], two_dma).makespan == rep.best
    assert all(rep.best <= m for m in rep.makespans)
    r25 = osim.exhaustive_search(bk("BK25"), two_dma)
    assert r25.best <= r25.median <= r25.worst and r25.best <= r25.geomean <= r25.worst
    single = osim.exhaustive_search([synthetic["T3"]], two_dma)
    assert len(single.makespans) == 1 and single.best == single.worst
    clones = [osim.TaskSpec(id=f"c{i}", fixed_durations=synthetic["T4"].fixed_durations) for i in range(4)]
    cr = osim.exhaustive_search(clones, two_dma)
    assert cr.best == cr.worst
    six = [osim.TaskSpec(id=f"t{i}", fixed_durations=(0.5 + 0.1 * i, 2.0, 0.5)) for i in range(6)]
    a = osim.exhaustive_search(six, two_dma, cap=50, seed=9)
    b = osim.exhaustive_search(six, two_dma, cap=50, seed=9)
    assert not a.exhaustive and a.orderings == b.orderings and a.makespans == b.makespans


# ---- acceptance criteria 1-4 (test_acceptance.py:70-109) ------------------------

def test_criterion_1_engine_matches_micro_steps(sweeps, one_dma, two_dma):
    worst = 0.0
    for (name, pname), entries in sweeps.items():
        p = one_dma if pname == "1dma" else two_dma
        for perm, tl in entries:
            micro = osim.micro_simulate(list(perm), p, dt=DT).makespan
            worst = max(worst, abs(tl.makespan - micro) / tl.makespan)
            assert abs(tl.makespan - micro) <= 2 * DT  # test_oracle.py:33-41
    assert worst <= 1e-3


def test_criteria_2_to_4_heuristic_quality(one_dma, two_dma):
    spread = {}
    for name in BK:
        tasks = bk(name)
        for pname, p in (("1dma", one_dma), ("2dma", two_dma)):
            rep = osim.exhaustive_search(tasks, p)
            h = osim.simulate(osim.reorder_batch(tasks, p), p).makespan
            assert h <= rep.median + 1e-9  # criterion 2
            if pname == "2dma":
                assert h <= 1.05 * rep.best + 1e-9  # criterion 3
                spread[name] = (rep.worst - rep.best) / rep.worst
    # criterion 4: mixed sets are more order-sensitive than pure ones
    assert min(spread[n] for n in ("BK25", "BK50", "BK75")) > max(spread["BK0"], spread["BK100"])
