"""Pin the CPU oracle (oracle/osim_oracle.c) to the reference's own outputs.

Every fixture in tests/golden/ was produced by running the unmodified
reference (tests/golden/make_golden.py); the oracle must reproduce it bit
for bit before it is trusted as the checker of the CUDA path.
"""

import math
import random
import sys

import numpy as np
import pytest

from oracle import oracle as O
from tests._golden import F, close, durs, fl, load, sha


def sum_mode_of(doc):
    return doc["meta"]["sum_mode"]


def test_golden_python_matches_interpreter_sum_mode():
    # the heuristic goldens depend on builtin sum(); the box runs the same image
    assert load("c1_bk.json")["meta"]["sum_mode"] == (1 if sys.version_info >= (3, 12) else 0)


def test_random_timelines_bit_exact():
    g = load("sim_random.json")
    for c in g["cases"]:
        r = O.simulate(durs(c["durs"]), c["order"], c["dma"], F(c["sigma"]))
        assert r.makespan == F(c["makespan"])
        assert r.k_end == F(c["k_end"])
        assert r.idle.tolist() == fl(c["idle"])
        assert r.steps == c["steps"]
        for t in range(c["n"]):
            for k in range(3):
                if c["start"][t][k] is None:
                    assert r.start[t, k] == -1.0
                else:
                    assert r.start[t, k] == F(c["start"][t][k])
                    assert r.end[t, k] == F(c["end"][t][k])


@pytest.mark.parametrize("idx", range(10))
def test_c1_exhaustive_and_heuristic(idx):
    c = load("c1_bk.json")["cases"][idx]
    d = durs(c["durs"])
    s, ms = O.exhaustive(d, c["dma"], F(c["sigma"]), makespans=True)
    rep = c["report"]
    assert ms.tolist() == fl(rep["makespans"])
    assert s["best"] == F(rep["best"]) and s["best_rank"] == rep["argmin"]
    assert rep["orderings"][rep["argmin"]] == rep["best_ordering"]
    assert s["worst"] == F(rep["worst"])
    assert float(np.median(ms)) == F(rep["median"])
    assert float(np.exp(np.log(ms).mean())) == F(rep["geomean"])
    assert close(s["sum"] / s["count"], F(rep["mean"]))
    assert close(math.exp(s["sum_log"] / s["count"]), F(rep["geomean"]))
    h = c["heuristic"]
    order, m, sims = O.reorder(d, c["id_rank"], c["dma"], F(c["sigma"]), sum_mode_of(load("c1_bk.json")))
    assert order == h["order"] and m == F(h["makespan"]) and sims == h["n_sims"]


def test_heuristic_random_bit_exact():
    g = load("heuristic_random.json")
    mode = sum_mode_of(g)
    for c in g["cases"]:
        order, m, sims = O.reorder(durs(c["durs"]), c["id_rank"], c["dma"], F(c["sigma"]), mode)
        assert order == c["order"], (c["profile"], c["n"], c["seed"])
        assert m == F(c["makespan"])
        assert sims == c["n_sims"]


def test_heuristic_sum_mode_matters():
    # the naive sum changes decisions on many 16-task groups
    g = load("heuristic_random.json")
    flips = 0
    for c in g["cases"]:
        if c["n"] != 16:
            continue
        order, _, _ = O.reorder(durs(c["durs"]), c["id_rank"], c["dma"], F(c["sigma"]), 0)
        flips += order != c["order"]
    assert flips > 0


def test_c2_tgs():
    g = load("c2_tg.json")
    for tg in g["tgs"]:
        s, ms = O.exhaustive(durs(tg["durs"]), g["dma"], F(g["sigma"]), threads=8, makespans=True)
        assert sha(ms) == tg["makespans_sha256"]
        assert s["best"] == F(tg["best"]) and s["best_rank"] == tg["argmin"] and s["worst"] == F(tg["worst"])
        assert float(np.median(ms)) == F(tg["median"])
        assert close(s["sum"] / s["count"], F(tg["mean"]))
        assert close(math.exp(s["sum_log"] / s["count"]), F(tg["geomean"]))


@pytest.mark.slow
def test_c3_full_space():
    g = load("c3_full.json")
    s, ms = O.exhaustive(durs(g["durs"]), g["dma"], F(g["sigma"]), threads=8, makespans=True)
    assert s["count"] == g["count"] == 3628800
    assert sha(ms) == g["makespans_sha256"]
    assert s["best"] == F(g["best"]) and s["best_rank"] == g["argmin"] and s["worst"] == F(g["worst"])
    assert float(np.median(ms)) == F(g["median"])
    assert close(s["sum"] / s["count"], F(g["mean"]))
    assert close(math.exp(s["sum_log"] / s["count"]), F(g["geomean"]))
    h = g["heuristic_relabeled_t00"]
    ranks = list(range(10))  # ids t00..t09 sort like indices
    order, m, sims = O.reorder(durs(g["durs"]), ranks, g["dma"], F(g["sigma"]), sum_mode_of(g))
    assert order == h["order"] and m == F(h["makespan"]) and sims == h["n_sims"]
    assert int((ms < m).sum()) == g["below_heuristic"]


def test_c4_sampled_ranks():
    g = load("c4_sample.json")
    d = durs(g["durs"])
    perms = np.array([O.unrank(r, 12) for r in g["ranks"]], dtype=np.uint8)
    for sig, want in g["makespans"].items():
        _, ms = O.eval_perms(d, g["dma"], float(sig), perms, threads=8)
        assert ms.tolist() == fl(want)


def test_c5_heuristic_rows():
    g = load("c5_sample.json")
    mode = sum_mode_of(g)
    for p in g["profiles"]:
        rows = p["rows"]
        d = np.stack([durs(r["durs"]) for r in rows])
        ranks = np.array([r["id_rank"] for r in rows], dtype=np.uint8)
        order, ms, sims = O.reorder_batch(d, ranks, p["dma"], F(p["sigma"]), mode, threads=8)
        for i, r in enumerate(rows):
            assert order[i].tolist() == r["order"], (p["profile"], r["b"])
            assert ms[i] == F(r["makespan"])
            assert sims[i] == r["n_sims"]


def test_unrank_matches_itertools():
    from itertools import permutations

    for n in range(1, 7):
        for r, p in enumerate(permutations(range(n))):
            assert tuple(O.unrank(r, n)) == p


def test_pysum_restatement_matches_builtin():
    rng = random.Random(5)
    mode = 1 if sys.version_info >= (3, 12) else 0
    for _ in range(20000):
        xs = [rng.uniform(0.05, 15.0) * (10 ** rng.randint(-3, 2)) for _ in range(rng.randint(1, 15))]
        assert O.pysum(xs, mode) == sum(xs)


def test_sampled_mode_makespans():
    g = load("sampled.json")
    from paper_1806_10113_b200.search import sample_permutations

    for c in g["cases"]:
        n = len(c["durs"])
        perms = sample_permutations(n, c["cap"], c["seed"])
        assert sha_u8(perms) == c["orderings_sha256"]
        _, ms = O.eval_perms(durs(c["durs"]), g["dma"], F(g["sigma"]), perms)
        assert sha(ms) == c["makespans_sha256"]
        assert ms[: len(c["makespans"])].tolist() == fl(c["makespans"])


def sha_u8(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint8).tobytes()).hexdigest()


def test_noreorder_oracle_pinned():
    import hashlib

    g = load("noreorder.json")
    for c in g["sequences"]:
        T, N = c["T"], c["N"]
        cnt = [0] * T
        order = []
        for w in c["labels"]:
            order.append(w * N + cnt[w])
            cnt[w] += 1
        dep = [(w * N + j - 1 if j else -1) for w in range(T) for j in range(N)]
        r = O.simulate_seq(durs(c["durs"]), order, c["dma"], F(c["sigma"]), dep)
        assert r.makespan == F(c["makespan"]) and r.idle.tolist() == fl(c["idle"])
        for t in range(T * N):
            for k in range(3):
                s = c["start"][t][k]
                if s is None:
                    assert r.start[t, k] == -1.0
                else:
                    assert r.start[t, k] == F(s) and r.end[t, k] == F(c["end"][t][k])
    for c in g["cases"]:
        T, N = c["T"], c["N"]
        d = np.array(c["durs"], dtype=object)
        d = np.array([[[F(x) for x in r] for r in row] for row in c["durs"]]).reshape(-1, 3)
        if c["exhaustive"]:
            s, ms = O.interleavings(d, T, N, c["dma"], F(c["sigma"]), threads=8, makespans=True)
        else:
            from paper_1806_10113_b200.noreorder import sample_interleavings

            s, ms = O.eval_sequences(d, T, N, c["dma"], F(c["sigma"]), sample_interleavings(T, N, c["cap"], c["seed"]))
        assert hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest() == c["makespans_sha256"]
        assert s["best_rank"] == c["argmin"] and s["best"] == F(c["best"]) and s["worst"] == F(c["worst"])
        assert float(np.median(ms)) == F(c["median"])


def test_micro_oracle_pinned():
    from itertools import permutations

    g = load("micro.json")
    for c in g["cases"]:
        d = durs(c["durs"])
        ms = [O.micro(d, list(p), c["dma"], F(c["sigma"]), F(c["dt"]))[0] for p in permutations(range(4))]
        assert ms == fl(c["makespans"])
    for c in g["random"]:
        ms, st, en = O.micro(durs(c["durs"]), c["order"], c["dma"], F(c["sigma"]), F(c["dt"]))
        assert ms == F(c["makespan"])
        for t in range(c["n"]):
            for k in range(3):
                s = c["start"][t][k]
                if s is None:
                    assert st[t, k] == -1.0
                else:
                    assert st[t, k] == F(s) and en[t, k] == F(c["end"][t][k])


def test_harness_oracle_pinned():
    import ctypes as C

    L = O.lib()
    L.oracle_harness.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int,
                                 C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    g = load("harness.json")
    for c in g["cases"]:
        d = np.ascontiguousarray(durs(c["durs"]))
        r = np.array(c["id_rank"], dtype=np.uint8)
        ms, ng, sizes = C.c_double(), C.c_int(), np.zeros(64, dtype=np.int32)
        rc = L.oracle_harness(d.ctypes.data_as(C.POINTER(C.c_double)), r.ctypes.data_as(C.POINTER(C.c_uint8)),
                              c["T"], c["N"], c["dma"], F(c["sigma"]), sum_mode_of(g), C.byref(ms), C.byref(ng),
                              sizes.ctypes.data_as(C.POINTER(C.c_int)))
        assert rc == 0 and ms.value == F(c["makespan"]) and sizes[: ng.value].tolist() == c["tg_sizes"]


# ---- groups of 17..64 tasks (tests/golden/wide.json) -----------------------

def _check_timeline(r, c, n):
    for t in range(n):
        for k in range(3):
            s = c["start"][t][k]
            if s is None:
                assert r.start[t, k] == -1.0
            else:
                assert r.start[t, k] == F(s) and r.end[t, k] == F(c["end"][t][k])


def test_wide_timelines_oracle_pinned():
    g = load("wide.json")
    for c in g["timelines"]:
        r = O.simulate(durs(c["durs"]), c["order"], c["dma"], F(c["sigma"]))
        assert r.makespan == F(c["makespan"]) and r.k_end == F(c["k_end"])
        assert r.idle.tolist() == fl(c["idle"]) and r.steps == c["steps"]
        _check_timeline(r, c, c["n"])
    for c in g["sequences"]:
        T, N = c["T"], c["N"]
        cnt = [0] * T
        order = []
        for w in c["labels"]:
            order.append(w * N + cnt[w])
            cnt[w] += 1
        dep = [(w * N + j - 1 if j else -1) for w in range(T) for j in range(N)]
        r = O.simulate_seq(durs(c["durs"]), order, c["dma"], F(c["sigma"]), dep)
        assert r.makespan == F(c["makespan"]) and r.idle.tolist() == fl(c["idle"])
        _check_timeline(r, c, T * N)


def test_wide_heuristic_sampled_noreorder_oracle_pinned():
    import hashlib

    from paper_1806_10113_b200.noreorder import sample_interleavings
    from paper_1806_10113_b200.search import sample_permutations

    g = load("wide.json")
    mode = sum_mode_of(g)
    for c in g["heuristic"]:
        order, m, sims = O.reorder(durs(c["durs"]), c["id_rank"], c["dma"], F(c["sigma"]), mode)
        assert order == c["order"] and m == F(c["makespan"]) and sims == c["n_sims"], (c["profile"], c["n"])
    for c in g["sampled"]:
        perms = sample_permutations(c["n"], c["cap"], c["seed"])
        assert sha_u8(perms) == c["orderings_sha256"]
        s, ms = O.eval_perms(durs(c["durs"]), c["dma"], F(c["sigma"]), perms)
        assert sha(ms) == c["makespans_sha256"] and s["best_rank"] == c["argmin"]
        assert float(np.median(ms)) == F(c["median"])
    for c in g["noreorder"]:
        T, N = c["T"], c["N"]
        d = np.array([[[F(x) for x in r] for r in row] for row in c["durs"]]).reshape(-1, 3)
        lab = sample_interleavings(T, N, c["cap"], c["seed"])
        assert sha_u8(lab) == c["labels_sha256"]
        s, ms = O.eval_sequences(d, T, N, c["dma"], F(c["sigma"]), lab)
        assert hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest() == c["makespans_sha256"]
        assert s["best_rank"] == c["argmin"] and float(np.median(ms)) == F(c["median"])


def test_wide_harness_oracle_pinned():
    import ctypes as C

    L = O.lib()
    L.oracle_harness.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int,
                                 C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    g = load("wide.json")
    for c in g["harness"]:
        d = np.ascontiguousarray(durs(c["durs"]))
        r = np.array(c["id_rank"], dtype=np.uint8)
        ms, ng, sizes = C.c_double(), C.c_int(), np.zeros(64, dtype=np.int32)
        rc = L.oracle_harness(d.ctypes.data_as(C.POINTER(C.c_double)), r.ctypes.data_as(C.POINTER(C.c_uint8)),
                              c["T"], c["N"], c["dma"], F(c["sigma"]), sum_mode_of(g), C.byref(ms), C.byref(ng),
                              sizes.ctypes.data_as(C.POINTER(C.c_int)))
        assert rc == 0 and ms.value == F(c["makespan"]) and sizes[: ng.value].tolist() == c["tg_sizes"], (c["T"], c["N"])


# ---- groups above 64 tasks and the round-1 drop-in divergences (tests/golden/big.json)

def test_big_oracle_pinned():
    import hashlib

    from paper_1806_10113_b200.noreorder import sample_interleavings
    from paper_1806_10113_b200.search import sample_permutations

    g = load("big.json")
    mode = sum_mode_of(g)
    for c in g["timelines"]:
        r = O.simulate(durs(c["durs"]), c["order"], c["dma"], F(c["sigma"]))
        assert r.makespan == F(c["makespan"]) and r.k_end == F(c["k_end"])
        assert r.idle.tolist() == fl(c["idle"]) and r.steps == c["steps"]
        _check_timeline(r, c, c["n"])
    for c in g["sequences"]:
        T, N = c["T"], c["N"]
        cnt = [0] * T
        order = []
        for w in c["labels"]:
            order.append(w * N + cnt[w])
            cnt[w] += 1
        dep = [(w * N + j - 1 if j else -1) for w in range(T) for j in range(N)]
        r = O.simulate_seq(durs(c["durs"]), order, c["dma"], F(c["sigma"]), dep)
        assert r.makespan == F(c["makespan"]) and r.idle.tolist() == fl(c["idle"])
        _check_timeline(r, c, T * N)
    for c in g["heuristic"]:
        order, m, sims = O.reorder(durs(c["durs"]), c["id_rank"], c["dma"], F(c["sigma"]), mode)
        assert order == c["order"] and m == F(c["makespan"]) and sims == c["n_sims"], (c["profile"], c["n"])
    for c in g["sampled"]:
        perms = sample_permutations(c["n"], c["cap"], c["seed"])
        assert hashlib.sha256(perms.astype(np.uint32).tobytes()).hexdigest() == c["orderings_sha256"]
        s, ms = O.eval_perms(durs(c["durs"]), c["dma"], F(c["sigma"]), perms.astype(np.uint8))
        assert sha(ms) == c["makespans_sha256"] and s["best_rank"] == c["argmin"]
    for c in g["noreorder"]:
        if c["exhaustive"]:
            continue  # the enumeration is checked in test_host (all_interleavings)
        T, N = c["T"], c["N"]
        d = np.array([[[F(x) for x in r] for r in row] for row in c["durs"]]).reshape(-1, 3)
        lab = sample_interleavings(T, N, c["cap"], c["seed"])
        assert hashlib.sha256(lab.astype(np.uint8).tobytes()).hexdigest() == c["labels_sha256"]
        s, ms = O.eval_sequences(d, T, N, c["dma"], F(c["sigma"]), lab)
        assert hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest() == c["makespans_sha256"]
        assert s["best_rank"] == c["argmin"] and float(np.median(ms)) == F(c["median"])
    for c in g["micro"]:
        ms, st, en = O.micro(durs(c["durs"]), c["order"], c["dma"], F(c["sigma"]), F(c["dt"]))
        assert ms == F(c["makespan"])
    single = g["single"]
    assert single["resolvable"] is False and single["returned"] == [single["id"]]
