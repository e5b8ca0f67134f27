"""Parity of the CUDA path (through the C-ABI) with the reference goldens and
the pinned CPU oracle.  Bit-exact for makespans, argmin ranks, heuristic
orderings and simulation counts; 1e-12 relative for mean and geomean
(north_star tolerance)."""

import math
import os

import numpy as np
import pytest

import paper_1806_10113_b200 as osim
from oracle import oracle as O
from paper_1806_10113_b200 import _capi, synth
from tests._golden import F, close, durs, fl, load, sha

pytestmark = pytest.mark.gpu

REL = 1e-12


def assert_summary_vs_oracle(s, o):
    assert s["count"] == o["count"]
    # an empty range (a shard with no calls, e.g. under an OSIM_PFX_L override)
    # has no argmin: only the identities are compared
    assert s["best"] == o["best"] and (s["count"] == 0 or s["best_rank"] == o["best_rank"])
    assert s["worst"] == o["worst"]
    assert close(s["sum"], o["sum"], REL)
    assert close(s["sum_log"], o["sum_log"], REL)


def test_device_present_and_library_loaded():
    assert _capi.init() >= 1
    assert b"sm_100a" in _capi.load().osim_version()


def test_fast_division_matches_ieee():
    assert _capi.selftest_div(200_000_000, seed=7) == 0
    assert _capi.selftest_div(50_000_000, seed=12345) == 0
    # adversarial operands: rounding-boundary mantissas, binade edges
    assert _capi.selftest_div(500_000_000, seed=99, mode=1) == 0


def test_timelines_bit_exact():
    g = load("sim_random.json")
    for c in g["cases"]:
        d = durs(c["durs"])
        st, en, ms, idle = _capi.timeline(d, c["dma"], F(c["sigma"]), c["order"])
        assert ms == F(c["makespan"])
        assert idle.tolist() == fl(c["idle"])
        for t in range(c["n"]):
            for k in range(3):
                if c["start"][t][k] is None:
                    assert st[t, k] == -1.0
                else:
                    assert st[t, k] == F(c["start"][t][k]) and en[t, k] == F(c["end"][t][k])


def test_simulate_dropin_timeline_order():
    c = load("c1_bk.json")["cases"][5]
    p = osim.DeviceProfile("2dma", 2, 0.01, 6e6, 0.01, 6e6, overlap_sigma=0.5)
    ids, d = synth.bk_group(c["bk"])
    tasks = [osim.TaskSpec(i, fixed_durations=tuple(r)) for i, r in zip(ids, d.tolist())]
    tl = osim.simulate(tasks, p)
    want = c["timeline_identity"]
    assert tl.makespan == F(want["makespan"])
    kinds = {"HtD": 0, "K": 1, "DtH": 2}
    assert [kinds[x.kind] for x in tl.commands] == want["sorted_kinds"]
    assert [ids.index(x.task_id) for x in tl.commands] == want["sorted_tasks"]
    assert [tl.idle[k] for k in osim.KINDS] == fl(want["idle"])


@pytest.mark.parametrize("idx", range(10))
def test_c1_dropin_report_and_heuristic(idx):
    c = load("c1_bk.json")["cases"][idx]
    p = osim.DeviceProfile(c["profile"], c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))
    ids = c["ids"]
    tasks = [osim.TaskSpec(i, fixed_durations=tuple(r)) for i, r in zip(ids, durs(c["durs"]).tolist())]
    rep = osim.exhaustive_search(tasks, p)
    want = c["report"]
    assert rep.exhaustive is True
    assert rep.makespans == fl(want["makespans"])
    assert [[ids.index(x) for x in o] for o in rep.orderings] == want["orderings"]
    assert rep.best == F(want["best"]) and rep.worst == F(want["worst"])
    assert [ids.index(x) for x in rep.best_ordering] == want["best_ordering"]
    assert rep.median == F(want["median"]) and rep.geomean == F(want["geomean"])
    out = osim.reorder_batch(tasks, p)
    assert [ids.index(t.id) for t in out] == c["heuristic"]["order"]
    assert osim.simulate(out, p).makespan == F(c["heuristic"]["makespan"])


def test_c2_tgs_full_space():
    g = load("c2_tg.json")
    for tg in g["tgs"]:
        s, ms = _capi.exhaustive(durs(tg["durs"]), g["dma"], F(g["sigma"]), 0, 40320, want_makespans=True)
        assert sha(ms) == tg["makespans_sha256"]
        assert s["best"] == F(tg["best"]) and s["best_rank"] == tg["argmin"] and s["worst"] == F(tg["worst"])
        assert float(np.median(ms)) == F(tg["median"])
        assert close(s["sum"] / s["count"], F(tg["mean"]), REL)
        assert close(math.exp(s["sum_log"] / s["count"]), F(tg["geomean"]), REL)


def test_c2_batch_vs_oracle():
    # the full config-2 batch (10^5 x 8-task groups); SURVEY 8(d) parity bar:
    # groups 0-255 plus 256 seeded-random indices against the oracle
    d = synth.c2_batch(100_000)
    out = _capi.exhaustive_batch(d, 2, 0.5)
    g = load("c2_tg.json")
    for tg in g["tgs"]:
        o = out[tg["tg"]]
        assert o["best"] == F(tg["best"]) and o["best_rank"] == tg["argmin"] and o["worst"] == F(tg["worst"])
        assert close(o["sum"] / o["count"], F(tg["mean"]), REL)
    rng = np.random.default_rng(3)
    idx = np.concatenate([np.arange(256), rng.choice(np.arange(256, 100_000), 256, replace=False)])
    cpus = os.cpu_count() or 4
    for b in idx:
        o, _ = O.exhaustive(d[b], 2, 0.5, threads=cpus)
        assert_summary_vs_oracle({k: out[b][k].item() for k in out.dtype.names}, o)
    # 1-DMA on the same groups
    out1 = _capi.exhaustive_batch(d[:4096], 1, 1.0)
    for b in list(range(0, 64)) + list(rng.choice(4096, 64, replace=False)):
        o, _ = O.exhaustive(d[b], 1, 1.0, threads=cpus)
        assert_summary_vs_oracle({k: out1[b][k].item() for k in out1.dtype.names}, o)


def test_c3_full_space_bit_exact():
    g = load("c3_full.json")
    s, ms = _capi.exhaustive(durs(g["durs"]), g["dma"], F(g["sigma"]), 0, 3628800, want_makespans=True)
    assert s["count"] == 3628800
    assert sha(ms) == g["makespans_sha256"]
    assert s["best"] == F(g["best"]) and s["best_rank"] == g["argmin"] and s["worst"] == F(g["worst"])
    assert float(np.median(ms)) == F(g["median"])
    assert close(s["sum"] / s["count"], F(g["mean"]), REL)
    assert close(math.exp(s["sum_log"] / s["count"]), F(g["geomean"]), REL)


def test_c3_heuristic_and_percentile():
    g = load("c3_full.json")
    h = g["heuristic_relabeled_t00"]
    order, ms, sims = _capi.heuristic_batch(durs(g["durs"])[None], np.arange(10, dtype=np.uint8)[None], 2,
                                            0.5, osim.SUM_MODE)
    assert order[0].tolist() == h["order"] and ms[0] == F(h["makespan"]) and sims[0] == h["n_sims"]


def test_c4_sampled_ranks_and_subrange():
    g = load("c4_sample.json")
    d = durs(g["durs"])
    perms = np.array([O.unrank(r, 12) for r in g["ranks"]], dtype=np.uint8)
    for sig, want in g["makespans"].items():
        s, ms = _capi.eval_perms(d, 2, float(sig), perms)
        assert ms.tolist() == fl(want)
        # a 1M-rank window of the 12! space against the oracle
        lo = 123_456_789
        s, _ = _capi.exhaustive(d, 2, float(sig), lo, lo + 1_000_000)
        o, _ = O.exhaustive(d, 2, float(sig), lo, lo + 1_000_000, threads=8)
        assert_summary_vs_oracle(s, o)


def _unrank_many(ranks, n):
    """Vectorized Lehmer unranking (lexicographic permutation index)."""
    ranks = np.asarray(ranks, dtype=np.int64).copy()
    avail = np.ones((len(ranks), n), dtype=bool)
    out = np.empty((len(ranks), n), dtype=np.uint8)
    for p in range(n):
        f = math.factorial(n - 1 - p)
        dgt = ranks // f
        ranks -= dgt * f
        pick = np.argmax(np.cumsum(avail, axis=1) == (dgt + 1)[:, None], axis=1)
        out[:, p] = pick
        avail[np.arange(len(ranks)), pick] = False
    return out


def test_c4_strided_ranks_bit_exact():
    # SURVEY 8(d) C4 parity bar: 10^6 strided ranks r = k * floor(12!/10^6)
    d = synth.c4_group()
    step = math.factorial(12) // 1_000_000
    perms = _unrank_many(np.arange(1_000_000) * step, 12)
    assert perms[1].tolist() == O.unrank(step, 12)
    cpus = os.cpu_count() or 4
    for sig in (0.5, 0.375):
        s, ms = _capi.eval_perms(d, 2, sig, perms)
        o, oms = O.eval_perms(d, 2, sig, perms, threads=cpus)
        assert np.array_equal(ms, oms)
        assert_summary_vs_oracle(s, o)
    s, ms = _capi.eval_perms(d, 1, 1.0, perms)
    o, oms = O.eval_perms(d, 1, 1.0, perms, threads=cpus)
    assert np.array_equal(ms, oms)


def test_c4_full_space_vs_oracle():
    # the whole 12! space of the headline group against the C restatement
    # (~1 min of host time on 16 threads)
    d = synth.c4_group()
    total = math.factorial(12)
    s, _ = _capi.exhaustive(d, 2, 0.5, 0, total)
    o, _ = O.exhaustive(d, 2, 0.5, 0, total, threads=os.cpu_count() or 4)
    assert_summary_vs_oracle(s, o)


def test_c4_full_space_consistency():
    d = synth.c4_group()
    total = math.factorial(12)
    whole, _ = _capi.exhaustive(d, 2, 0.5, 0, total)
    assert whole["count"] == total
    parts = [_capi.exhaustive(d, 2, 0.5, total * i // 4, total * (i + 1) // 4)[0] for i in range(4)]
    best = min(parts, key=lambda p: (p["best"], p["best_rank"]))
    assert whole["best"] == best["best"] and whole["best_rank"] == best["best_rank"]
    assert whole["worst"] == max(p["worst"] for p in parts)
    assert close(whole["sum"], sum(p["sum"] for p in parts), REL)
    # the argmin ordering re-simulates to the best makespan
    perm = np.array([osim.search.unrank(whole["best_rank"], 12)], dtype=np.uint8)
    _, ms = _capi.eval_perms(d, 2, 0.5, perm)
    assert ms[0] == whole["best"]
    r = O.simulate(d, perm[0].tolist(), 2, 0.5)
    assert r.makespan == whole["best"]


def test_c5_heuristic_rows_bit_exact():
    g = load("c5_sample.json")
    for p in g["profiles"]:
        rows = p["rows"]
        d = np.stack([durs(r["durs"]) for r in rows])
        ranks = np.array([r["id_rank"] for r in rows], dtype=np.uint8)
        order, ms, sims = _capi.heuristic_batch(d, ranks, p["dma"], F(p["sigma"]), g["meta"]["sum_mode"])
        for i, r in enumerate(rows):
            assert order[i].tolist() == r["order"], (p["profile"], r["b"])
            assert ms[i] == F(r["makespan"]) and sims[i] == r["n_sims"]


@pytest.mark.parametrize("profile", ["nvidia", "amd", "phi"])
def test_c5_heuristic_vs_oracle_many(profile):
    # SURVEY 8(d) C5 parity bar, at full size: all 10^6 groups of config 5
    # per profile (seeds 0..999999), order, makespan and simulation count
    # bit-exact (~6 s of oracle time on 16 host threads per profile)
    cpus = os.cpu_count() or 4
    d, r = synth.c5_batch(profile, 1_000_000, start=0, workers=min(cpus, 32))
    _, dma, sigma = synth.PROFILES[profile]
    order, ms, sims = _capi.heuristic_batch(d, r, dma, sigma, osim.SUM_MODE)
    o_order, o_ms, o_sims = O.reorder_batch(d, r, dma, sigma, osim.SUM_MODE, threads=cpus)
    assert np.array_equal(order, o_order)
    assert np.array_equal(ms, o_ms)
    assert np.array_equal(sims, o_sims)


_HR_CHILD = """
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1806_10113_b200 as osim
from paper_1806_10113_b200 import _capi, synth
for prof in ("nvidia", "amd", "phi"):
    d, r = synth.c5_batch_fast(prof, 50_000)
    _, dma, sigma = synth.PROFILES[prof]
    o, m, n = _capi.heuristic_batch(d, r, dma, sigma, osim.SUM_MODE)
    print(prof, hashlib.sha256(o.tobytes() + m.tobytes() + n.tobytes()).hexdigest())
"""


def test_heuristic_lane_htd_pair_fallback():
    """k_heuristic_lane reads each candidate's {t_htd, 1/t_htd} from pairs it
    staged in the launcher's aux buffer; without the buffer it loads and
    divides per candidate.  OSIM_HL_NO_HR=1 forces that path: same outputs."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("0", "1"):
        r = subprocess.run([sys.executable, "-c", _HR_CHILD, root], env=dict(os.environ, OSIM_HL_NO_HR=v),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append([ln for ln in r.stdout.splitlines() if ln.split(" ")[0] in ("nvidia", "amd", "phi")])
    assert len(outs[0]) == 3 and outs[0] == outs[1]


def test_heuristic_random_goldens():
    g = load("heuristic_random.json")
    for c in g["cases"]:
        order, ms, sims = _capi.heuristic_batch(durs(c["durs"])[None], np.array([c["id_rank"]], np.uint8),
                                                c["dma"], F(c["sigma"]), g["meta"]["sum_mode"])
        assert order[0].tolist() == c["order"], (c["profile"], c["n"], c["seed"])
        assert ms[0] == F(c["makespan"]) and sims[0] == c["n_sims"]


def test_null_stages_general_path_vs_oracle():
    rng = np.random.default_rng(11)
    for trial in range(40):
        n = int(rng.integers(2, 8))
        d = rng.integers(0, 5, (n, 3)).astype(np.float64)
        d[d.sum(1) == 0, 1] = 1.0
        dma = 1 + trial % 2
        sigma = [0.5, 0.375, 0.8, 1.0][trial % 4]
        s, ms = _capi.exhaustive(d, dma, sigma, 0, math.factorial(n), want_makespans=True)
        o, oms = O.exhaustive(d, dma, sigma, makespans=True)
        assert np.array_equal(ms, oms)
        assert_summary_vs_oracle(s, o)
        ids = [f"t{i}" for i in rng.permutation(n)]
        rk = np.array(sorted(range(n), key=lambda i: ids[i]), dtype=np.uint8).argsort().astype(np.uint8)
        order, hm, hs = _capi.heuristic_batch(d[None], rk[None], dma, sigma, osim.SUM_MODE)
        oo, om, osims = O.reorder(d, rk, dma, sigma, osim.SUM_MODE)
        assert order[0].tolist() == oo and hm[0] == om and hs[0] == osims


def test_sampled_mode_dropin():
    g = load("sampled.json")
    p = osim.DeviceProfile("2dma", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(g["sigma"]))
    for c in g["cases"]:
        tasks = [osim.TaskSpec(f"t{i}", fixed_durations=tuple(r)) for i, r in enumerate(durs(c["durs"]).tolist())]
        rep = osim.exhaustive_search(tasks, p, cap=c["cap"], seed=c["seed"])
        assert rep.exhaustive is False
        assert sha(np.array(rep.makespans)) == c["makespans_sha256"]
        assert rep.best == F(c["best"]) and rep.worst == F(c["worst"])
        assert rep.median == F(c["median"]) and rep.geomean == F(c["geomean"])
        assert [int(x[1:]) for x in rep.best_ordering] == c["best_ordering"]


def test_errors_map_to_reference_exceptions():
    d = np.ones((3, 3))
    with pytest.raises(ValueError):
        _capi.exhaustive(d, 3, 0.5, 0, 6)
    with pytest.raises(ValueError):
        _capi.exhaustive(d, 2, 1.5, 0, 6)
    with pytest.raises(ValueError):
        _capi.exhaustive(d, 2, 0.5, 0, 7)
    with pytest.raises(ValueError):
        _capi.exhaustive(np.ones((17, 3)), 2, 0.5, 0, 1)
    with pytest.raises(osim.UnresolvableDuration):
        _capi.exhaustive(np.zeros((2, 3)), 2, 0.5, 0, 2)
    with pytest.raises(Exception):
        _capi.exhaustive(d, 2, 0.5, 0, 6, n_dev=64)


def test_determinism_run_to_run():
    d = synth.c4_group()
    a, _ = _capi.exhaustive(d, 2, 0.375, 0, 50_000_000)
    b, _ = _capi.exhaustive(d, 2, 0.375, 0, 50_000_000)
    assert a == b


# ---- row f2: percentile count and exact median on the device ---------------

def test_c3_median_and_heuristic_percentile_on_device():
    g = load("c3_full.json")
    h = g["heuristic_relabeled_t00"]
    s, below, med = _capi.exhaustive_stats(durs(g["durs"]), 2, 0.5, 0, 3628800, threshold=F(h["makespan"]))
    assert med == F(g["median"])
    assert below == g["below_heuristic"]
    assert s["best_rank"] == g["argmin"] and s["best"] == F(g["best"])


def test_medians_match_numpy_goldens():
    for c in load("c1_bk.json")["cases"]:
        _, below, med = _capi.exhaustive_stats(durs(c["durs"]), c["dma"], F(c["sigma"]), 0, 24)
        assert med == F(c["report"]["median"]) and below == 0
    g = load("c2_tg.json")
    for tg in g["tgs"]:
        _, _, med = _capi.exhaustive_stats(durs(tg["durs"]), 2, 0.5, 0, 40320)
        assert med == F(tg["median"])


def test_c4_window_median_odd_and_even_vs_numpy():
    d = synth.c4_group()
    for lo, cnt in ((77_777_777, 1_000_001), (300_000_000, 999_998)):
        _, oms = O.exhaustive(d, 2, 0.375, lo, lo + cnt, threads=8, makespans=True)
        thr = float(np.quantile(oms, 0.3))
        s, below, med = _capi.exhaustive_stats(d, 2, 0.375, lo, lo + cnt, threshold=thr)
        assert med == float(np.median(oms))
        assert below == int((oms < thr).sum())
        assert s["count"] == cnt


def test_median_with_heavy_ties_vs_numpy():
    # integer stage times: makespans repeat massively (duplicate middle
    # values, narrow common prefix), odd and even windows, both DMA modes
    rng = np.random.default_rng(11)
    d = rng.integers(1, 6, (9, 3)).astype(np.float64)
    for dma, sigma in ((2, 0.5), (1, 1.0)):
        for lo, hi in ((0, 362880), (1000, 362880 - 7)):
            _, oms = O.exhaustive(d, dma, sigma, lo, hi, threads=8, makespans=True)
            _, below, med = _capi.exhaustive_stats(d, dma, sigma, lo, hi, threshold=float(np.median(oms)))
            assert med == float(np.median(oms)) and below == int((oms < np.median(oms)).sum())


def test_c4_full_space_median_is_an_order_statistic():
    d = synth.c4_group()
    total = math.factorial(12)
    s, below, med = _capi.exhaustive_stats(d, 2, 0.5, 0, total, threshold=float("inf"))
    assert below == total == s["count"]
    # even count: med = (v[k-1] + v[k]) / 2 with k = total/2 -> at most k values
    # lie strictly below it and at least k at or below it
    _, lt, _ = _capi.exhaustive_stats(d, 2, 0.5, 0, total, threshold=med, median=False)
    _, le, _ = _capi.exhaustive_stats(d, 2, 0.5, 0, total, threshold=float(np.nextafter(med, np.inf)),
                                      median=False)
    assert lt <= total // 2 <= le
    assert s["best"] <= med <= s["worst"]


def test_f2_median_bin_above_2_32():
    """13! = 6,227,020,800 makespans in HBM with one value held by 11/13 of
    them (5.27e9 > 2^32 in the median's bin): the selection histograms count
    in 64 bits.  Every kernel lane is busy from the first HtD on (t_k = 5 >=
    every transfer), so makespan = first HtD + 13 * 5 + last DtH (1): 66.5 if
    task 11 runs first, 69.0 if task 12 does, else 67.0 (sampled against the
    oracle below)."""
    d = np.array([[1.0, 5.0, 1.0]] * 11 + [[0.5, 5.0, 1.0], [3.0, 5.0, 1.0]])
    rng = np.random.default_rng(13)
    perms = np.array([rng.permutation(13) for _ in range(2000)], dtype=np.uint8)
    _, oms = O.eval_perms(d, 2, 0.5, perms, threads=os.cpu_count() or 1)
    first = perms[:, 0]
    assert set(oms[first == 11]) == {66.5} and set(oms[first == 12]) == {69.0}
    assert set(oms[(first != 11) & (first != 12)]) == {67.0}
    total, f12 = math.factorial(13), math.factorial(12)
    s, lt, med = _capi.exhaustive_stats(d, 2, 0.5, 0, total, threshold=67.0)
    assert s["count"] == total and s["best"] == 66.5 and s["best_rank"] == 11 * f12 and s["worst"] == 69.0
    assert med == 67.0
    _, le, _ = _capi.exhaustive_stats(d, 2, 0.5, 0, total, threshold=float(np.nextafter(67.0, np.inf)),
                                      median=False)
    assert lt == f12 and le == total - f12
    assert lt <= total // 2 <= le  # the order-statistic check
    assert le - lt > 2**32


def test_select_kth_counts_above_2_32():
    """A synthetic device array of 2^32 + 5 values (34 GB): 2^32 + 1 ones
    then four twos, and a constant array; 32-bit bin counts would wrap."""
    import torch

    _capi.set_device(0)
    n = 2**32 + 5
    v = torch.ones(n, dtype=torch.float64, device="cuda")
    v[-4:] = 2.0
    torch.cuda.synchronize()
    p = v.data_ptr()
    assert _capi.select_kth_dev(p, n, 0) == 1.0
    assert _capi.select_kth_dev(p, n, 2**32) == 1.0
    assert _capi.select_kth_dev(p, n, 2**32 + 1) == 2.0
    assert _capi.select_kth_dev(p, n, n - 1) == 2.0
    v.fill_(3.25)
    torch.cuda.synchronize()
    assert _capi.select_kth_dev(p, n, n // 2) == 3.25
    with pytest.raises(ValueError):
        _capi.select_kth_dev(p, n, n)
    del v
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [2, 4])
def test_virtual_multi_device_paths(k):
    """The C-ABI's in-process n_dev > 1 paths (sharding, per-device
    validation, host-side merges and the per-device histogram sums of the
    exact median) on one GPU: OSIM_VIRTUAL_DEVICES=k gives the library k
    device contexts on device 0 (tests/ndev_check.py, in a subprocess)."""
    import subprocess
    import sys

    env = dict(os.environ, OSIM_VIRTUAL_DEVICES=str(k))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "ndev_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert f"ndev ok {list(range(2, k + 1))}" in r.stdout


def test_heuristic_percentile_dropin():
    g = load("c3_full.json")
    p = osim.DeviceProfile("2dma", 2, 0.01, 6e6, 0.01, 6e6, overlap_sigma=0.5)
    tasks = [osim.TaskSpec(f"t{i:02d}", fixed_durations=tuple(r)) for i, r in enumerate(durs(g["durs"]).tolist())]
    hms, pct, st = osim.heuristic_percentile(tasks, p)
    h = g["heuristic_relabeled_t00"]
    assert hms == F(h["makespan"])
    assert st.below == g["below_heuristic"]
    assert pct == 100.0 * g["below_heuristic"] / 3628800
    assert st.median == F(g["median"])


def test_distributed_stats_single_rank_nccl():
    import os
    import socket

    import torch
    import torch.distributed as tdist

    from paper_1806_10113_b200 import dist as odist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = load("c3_full.json")
        h = g["heuristic_relabeled_t00"]
        summ, below, med = odist.exhaustive_stats_distributed(durs(g["durs"]), 2, 0.5, threshold=F(h["makespan"]))
        assert med == F(g["median"]) and below == g["below_heuristic"]
        assert summ.best_rank == g["argmin"] and summ.count == 3628800
    finally:
        tdist.destroy_process_group()



# ---- row f1: NoReorder interleavings (deps + 1-DMA waves) -----------------

def test_simulate_sequence_timelines_bit_exact():
    g = load("noreorder.json")
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
        assert ms == F(c["makespan"]) and idle.tolist() == fl(c["idle"])
        for t in range(T * N):
            for k in range(3):
                s = c["start"][t][k]
                if s is None:
                    assert st[t, k] == -1.0
                else:
                    assert st[t, k] == F(s) and en[t, k] == F(c["end"][t][k])


def test_noreorder_distributions_bit_exact():
    import hashlib

    from paper_1806_10113_b200 import noreorder as nr

    g = load("noreorder.json")
    for c in g["cases"]:
        d = np.array([[[F(x) for x in r] for r in row] for row in c["durs"]])
        labels, ms, summ, exhaustive = nr.distribution_durs(d, c["dma"], F(c["sigma"]), c["cap"], c["seed"])
        assert exhaustive == c["exhaustive"] and len(ms) == c["count"]
        assert hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest() == c["makespans_sha256"]
        assert summ["best_rank"] == c["argmin"] and summ["best"] == F(c["best"]) and summ["worst"] == F(c["worst"])
        assert float(np.median(ms)) == F(c["median"])


def test_noreorder_large_space_vs_oracle():
    # 4 workers x 3 tasks: 369,600 interleavings, 1-DMA waves and 2-DMA
    rng = np.random.default_rng(5)
    d = rng.uniform(0.2, 5.0, (4, 3, 3))
    total = 369600
    for dma, sigma in ((1, 1.0), (2, 0.375)):
        s, below, ms = _capi.interleavings(d.reshape(-1, 3), 4, 3, dma, sigma, 0, total, threshold=20.0,
                                           want_makespans=True)
        o, oms = O.interleavings(d.reshape(-1, 3), 4, 3, dma, sigma, threads=8, makespans=True)
        assert np.array_equal(ms, oms)
        assert_summary_vs_oracle(s, o)
        assert below == int((oms < 20.0).sum())


def test_noreorder_fast_path_4x4_vs_oracle():
    # 2-DMA, every stage non-null: the FastSim interleaving kernel (n = 16:
    # unshifted packing); a 300k window of the 63,063,000 interleavings
    d = synth.real_group("K20", 16, 41)[1]
    lo, hi = 31_000_000, 31_300_000
    cpus = os.cpu_count() or 4
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        # 1-DMA: the wave-split fast kernel (k_interleave_pfx1)
        s, below, ms = _capi.interleavings(d, 4, 4, dma, sigma, lo, hi, threshold=90.0, want_makespans=True)
        o, oms = O.interleavings(d, 4, 4, dma, sigma, lo, hi, threads=cpus, makespans=True)
        assert np.array_equal(ms, oms)
        assert_summary_vs_oracle(s, o)
        assert below == int((oms < 90.0).sum())


@pytest.mark.parametrize("T,N,lo,hi", [
    (3, 5, 0, 756756),          # n = 15: pre-shifted packing, the whole space
    (2, 8, 5, 12870 - 3),       # ragged ends
    (1, 16, 0, 1),              # one sequence: the run is the whole ordering
    (16, 1, 1_000_000_007, 1_000_000_007 + 20_011),  # 16! / 1 labels, prime-length window
    (4, 4, 62_000_001, 62_100_000),
    (4, 4, 7, 8),               # a single rank inside a run
])
def test_noreorder_prefix_runs_vs_oracle(T, N, lo, hi):
    # k_interleave_pfx / k_interleave_pfx1 (1-DMA waves): runs of consecutive
    # ranks share their label prefix; windows cut runs anywhere, shapes cover
    # both packings and T or N = 1
    d = synth.real_group("K20", T * N, 7 + T)[1]
    cpus = os.cpu_count() or 4
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        s, below, ms = _capi.interleavings(d, T, N, dma, sigma, lo, hi, threshold=60.0, want_makespans=True)
        o, oms = O.interleavings(d, T, N, dma, sigma, lo, hi, threads=cpus, makespans=True)
        assert np.array_equal(ms, oms)
        assert_summary_vs_oracle(s, o)
        assert below == int((oms < 60.0).sum())


def test_simulate_with_deps_dropin():
    p2 = osim.DeviceProfile("2dma", 2, 0.0, 1.0, 0.0, 1.0, overlap_sigma=0.5)
    p1 = osim.DeviceProfile("1dma", 1, 0.0, 1.0, 0.0, 1.0)
    tasks = [osim.TaskSpec(f"t{i}", fixed_durations=(1.0 + i, 2.0, 0.5 * i + 0.25)) for i in range(5)]
    deps = {"t3": "t1", "t4": "t0"}
    dep = [-1, -1, -1, 1, 0]
    for p in (p2, p1):
        if p.dma_engines == 2:
            tl = osim.simulate(tasks, p, deps=deps)
            r = O.simulate([t.fixed_durations for t in tasks], list(range(5)), 2, p.overlap_sigma, dep=dep)
            assert tl.makespan == r.makespan
        else:
            # one 1-DMA submit: HtD(t3) waits for DtH(t1), queued behind it ->
            # the reference stalls (engine.py:239-241), and so must we
            with pytest.raises(RuntimeError):
                osim.simulate(tasks, p, deps=deps)
            with pytest.raises(RuntimeError):
                O.simulate([t.fixed_durations for t in tasks], list(range(5)), 1, 1.0, dep=dep)
        seq_tl = osim.simulate_sequence(tasks, p, deps)
        rs = O.simulate_seq([t.fixed_durations for t in tasks], list(range(5)), p.dma_engines, p.overlap_sigma, dep)
        assert seq_tl.makespan == rs.makespan


# ---- row f4: micro-step tick oracle -----------------------------------------

def test_micro_bit_exact_vs_reference():
    g = load("micro.json")
    for c in g["cases"]:
        ms = _capi.micro(durs(c["durs"]), c["dma"], F(c["sigma"]), F(c["dt"]), 0, 24)
        assert ms.tolist() == fl(c["makespans"])
    for c in g["random"]:
        st, en, ms = _capi.micro_timeline(durs(c["durs"]), c["dma"], F(c["sigma"]), F(c["dt"]), c["order"])
        assert ms == F(c["makespan"])
        for t in range(c["n"]):
            for k in range(3):
                s = c["start"][t][k]
                if s is None:
                    assert st[t, k] == -1.0
                else:
                    assert st[t, k] == F(s) and en[t, k] == F(c["end"][t][k])


def test_micro_simulate_dropin_and_validate_sweep():
    c = load("micro.json")["random"][7]
    tasks = [osim.TaskSpec(f"t{i}", fixed_durations=tuple(r)) for i, r in enumerate(durs(c["durs"]).tolist())]
    ordered = [tasks[i] for i in c["order"]]
    p = osim.DeviceProfile("p", c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))
    tl = osim.micro_simulate(ordered, p, dt=F(c["dt"]))
    assert tl.makespan == F(c["makespan"])
    assert [tl.idle[k] for k in osim.KINDS] == fl(c["idle"])
    checked, dev, ok = osim.validate(dt=0.001)
    assert checked == 240 and ok and dev <= 0.002


def test_micro_c2_group_vs_oracle():
    d = synth.c2_batch(1)[0]
    ms = _capi.micro(d, 2, 0.5, 0.001, 0, 40320)
    for r in range(0, 40320, 997):
        assert ms[r] == O.micro(d, O.unrank(r, 8), 2, 0.5, 0.001)[0]


# ---- row f3: proxy-thread scenario harness ----------------------------------

def test_harness_batch_bit_exact():
    g = load("harness.json")
    groups = {}
    for c in g["cases"]:
        groups.setdefault((c["T"], c["N"], c["dma"], c["sigma"]), []).append(c)
    for (T, N, dma, sig), cs in groups.items():
        d = np.stack([durs(c["durs"]) for c in cs])
        r = np.array([c["id_rank"] for c in cs], dtype=np.uint8)
        ms, ng, sz, _, _ = _capi.harness_batch(d, r, T, N, dma, F(sig), g["meta"]["sum_mode"])
        for i, c in enumerate(cs):
            assert ms[i] == F(c["makespan"]), (T, N, c["bk"], c["seed"])
            assert sz[i, : ng[i]].tolist() == c["tg_sizes"]


def test_run_scenario_dropin():
    from paper_1806_10113_b200 import workload as wl

    g = load("harness.json")
    c = g["cases"][4]
    p = osim.DeviceProfile("p", c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))
    sc = wl.Scenario(c["T"], c["N"], wl.load_bk_benchmark(c["bk"]), c["seed"], p)
    res = wl.run_scenario(sc, evaluate_noreorder=c["T"] * c["N"] <= 8)
    assert res.heuristic_makespan == F(c["makespan"]) and res.tg_sizes == c["tg_sizes"]
    assert res.timeline.makespan == max(cmd.end for cmd in res.timeline.commands)
    if res.noreorder is not None:
        assert res.speedup_best >= res.speedup_median >= 1.0


def test_harness_many_scenarios_vs_oracle():
    import ctypes as C

    from paper_1806_10113_b200 import workload as wl

    L = O.lib()
    L.oracle_harness.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int,
                                 C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    T, N = 4, 3
    for pname, (dev, dma, sigma) in synth.PROFILES.items():
        S = 2000
        d = np.stack([synth.real_group(dev, T * N, 10_000 + s)[1] for s in range(S)])
        r = np.tile(np.argsort(np.argsort([f"w{w}.{j}" for w in range(T) for j in range(N)])).astype(np.uint8),
                    (S, 1))
        ms, ng, sz, _, _ = _capi.harness_batch(d, r, T, N, dma, sigma, osim.SUM_MODE)
        for s in range(0, S, 97):
            om, ong, osz = C.c_double(), C.c_int(), np.zeros(64, dtype=np.int32)
            rc = L.oracle_harness(np.ascontiguousarray(d[s]).ctypes.data_as(C.POINTER(C.c_double)),
                                  np.ascontiguousarray(r[s]).ctypes.data_as(C.POINTER(C.c_uint8)), T, N, dma, sigma,
                                  osim.SUM_MODE, C.byref(om), C.byref(ong), osz.ctypes.data_as(C.POINTER(C.c_int)))
            assert rc == 0 and ms[s] == om.value and sz[s, : ng[s]].tolist() == osz[: ong.value].tolist()


# ---- every instantiation: n = 1..16 windows, both DMA modes, sigma pow2 or not ---

@pytest.mark.parametrize("n", list(range(1, 17)))
def test_exhaustive_every_n_window_vs_oracle(n):
    rng = np.random.default_rng(100 + n)
    d = rng.uniform(0.05, 6.0, (n, 3))
    total = math.factorial(n)
    span = min(total, 60_000)
    lo = (total - span) // 3 + (7 if total > span + 7 else 0)
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        s, ms = _capi.exhaustive(d, dma, sigma, lo, lo + span, want_makespans=True)
        o, oms = O.exhaustive(d, dma, sigma, lo, lo + span, threads=8, makespans=True)
        assert np.array_equal(ms, oms), (n, dma, sigma)
        assert_summary_vs_oracle(s, o)


@pytest.mark.parametrize("n", list(range(1, 13)))
def test_batch_every_n_vs_oracle(n):
    rng = np.random.default_rng(200 + n)
    B = 2 if n >= 10 else 12
    d = rng.uniform(0.05, 6.0, (B, n, 3))
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        out = _capi.exhaustive_batch(d, dma, sigma)
        for b in range(B):
            got = {k: out[b][k].item() for k in out.dtype.names}
            if n <= 10:
                o, _ = O.exhaustive(d[b], dma, sigma, threads=8)
            else:  # 11!/12! per group: against the single-group kernel (oracle-tested on windows)
                o, _ = _capi.exhaustive(d[b], dma, sigma, 0, math.factorial(n))
            assert_summary_vs_oracle(got, o)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 9, 13, 16])
def test_heuristic_every_size_vs_oracle(n):
    rng = np.random.default_rng(300 + n)
    B = 200
    d = rng.uniform(0.05, 6.0, (B, n, 3))
    r = np.stack([rng.permutation(n) for _ in range(B)]).astype(np.uint8)
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        order, ms, sims = _capi.heuristic_batch(d, r, dma, sigma, osim.SUM_MODE)
        oo, om, osims = O.reorder_batch(d, r, dma, sigma, osim.SUM_MODE, threads=8)
        assert np.array_equal(order, oo) and np.array_equal(ms, om) and np.array_equal(sims, osims)


def test_out_of_fast_range_durations_take_the_general_path():
    # non-null stages outside [2^-60, 2^60] (and sigma = 1) select the IEEE-division path
    rng = np.random.default_rng(9)
    for scale in (1e-22, 1e22):
        d = rng.uniform(0.5, 4.0, (6, 3)) * scale
        assert not _capi.fast_eligible(d, 0.5)
        for dma, sigma in ((2, 0.5), (2, 0.3), (1, 1.0)):
            s, ms = _capi.exhaustive(d, dma, sigma, 0, 720, want_makespans=True)
            o, oms = O.exhaustive(d, dma, sigma, makespans=True)
            assert np.array_equal(ms, oms)
            assert_summary_vs_oracle(s, o)
            r = np.arange(6, dtype=np.uint8)
            order, hm, _ = _capi.heuristic_batch(d[None], r[None], dma, sigma, osim.SUM_MODE)
            oo, om, _ = O.reorder(d, r, dma, sigma, osim.SUM_MODE)
            assert order[0].tolist() == oo and hm[0] == om


def test_heuristic_large_batch_device_validation_and_fallback():
    # >= 2^17 groups: chunked two-stream pipeline, inputs validated on the
    # device while the fast kernel runs optimistically
    rng = np.random.default_rng(77)
    B, n = (1 << 17) + 5, 4
    d = rng.uniform(0.05, 6.0, (B, n, 3))
    r = np.stack([rng.permutation(n) for _ in range(64)]).astype(np.uint8)[rng.integers(0, 64, B)]
    # one group outside the fast range -> the whole shard reruns on the general kernel
    d[70001] *= 1e23
    for dma, sigma in ((2, 0.5), (1, 1.0)):
        order, ms, sims = _capi.heuristic_batch(d, r, dma, sigma, osim.SUM_MODE)
        oo, om, osims = O.reorder_batch(d, r, dma, sigma, osim.SUM_MODE, threads=16)
        assert np.array_equal(order, oo) and np.array_equal(ms, om) and np.array_equal(sims, osims)
    # invalid inputs in an interior chunk: the lowest offending task / group is reported
    bad = d.copy()
    bad[90000, 2, 1] = -1.0
    bad[100000, 1, 0] = np.nan
    with pytest.raises(ValueError, match=f"task {90000 * n + 2}:"):
        _capi.heuristic_batch(bad, r, 2, 0.5, osim.SUM_MODE)
    bad = d.copy()
    bad[120000, 3] = 0.0
    with pytest.raises(osim.UnresolvableDuration, match=f"task {120000 * n + 3} has"):
        _capi.heuristic_batch(bad, r, 2, 0.5, osim.SUM_MODE)
    rr = r.copy()
    rr[100001] = [0, 1, 1, 3]
    rr[110000] = [0, 1, 2, 9]
    with pytest.raises(ValueError, match="group 100001:"):
        _capi.heuristic_batch(d, rr, 2, 0.5, osim.SUM_MODE)
    # the context is clean afterwards
    order, ms, _ = _capi.heuristic_batch(d[:1000], r[:1000], 2, 0.5, osim.SUM_MODE)
    oo, om, _ = O.reorder_batch(d[:1000], r[:1000], 2, 0.5, osim.SUM_MODE, threads=8)
    assert np.array_equal(order, oo) and np.array_equal(ms, om)


def _gpu_shard_worker(rank, world, port, q):
    import torch.distributed as tdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1806_10113_b200.dist import exhaustive_summary_distributed

        s = exhaustive_summary_distributed(synth.c3_group(), 2, 0.5)  # shard on cuda:0 via the library
        q.put((rank, s.best, s.best_ordering, s.worst, s.mean, s.geomean))
    finally:
        tdist.destroy_process_group()


def test_two_rank_shards_through_the_library_combine_exactly():
    # the N>1 path's sharding and combine with real GPU shards: two ranks
    # (gloo for the 48-byte exchange) each reduce their half of 10! on the
    # device independently; no rank waits on another's kernels
    import socket

    import torch.multiprocessing as mp

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    whole = osim.exhaustive_summary_durs(synth.c3_group(), 2, 0.5)
    for _, best, order, worst, mean, geo in res:
        assert best == whole.best and tuple(order) == tuple(whole.best_ordering) and worst == whole.worst
        assert close(mean, whole.mean, REL) and close(geo, whole.geomean, REL)


def _nccl_worker(port, q):
    import torch
    import torch.distributed as tdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_1806_10113_b200.dist import exhaustive_summary_distributed

        s = exhaustive_summary_distributed(synth.c3_group(), 2, 0.5)  # NCCL all_gather of device tensors
        from paper_1806_10113_b200.dist import exhaustive_summary_batch_distributed, reorder_durs_distributed

        d5, r5 = synth.c5_batch_fast("nvidia", 5000)
        order, ms, sims = reorder_durs_distributed(d5, r5, 2, 0.5)
        summ = exhaustive_summary_batch_distributed(synth.c2_batch(300), 2, 0.5)
        q.put((s.best, s.best_ordering, s.worst, s.mean, s.count, order, ms, sims, summ))
    finally:
        tdist.destroy_process_group()


def test_nccl_exchange_single_rank():
    # the NCCL branch of the sharded combine (device tensors, all_gather over
    # NCCL) at world size 1 -- the bench's N>1 code path on the one GPU here
    import socket

    import torch.multiprocessing as mp

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(port, q))
    p.start()
    best, order, worst, mean, count, o5, m5, s5, summ = q.get(timeout=300)
    p.join(timeout=120)
    assert p.exitcode == 0
    whole = osim.exhaustive_summary_durs(synth.c3_group(), 2, 0.5)
    assert best == whole.best and tuple(order) == tuple(whole.best_ordering) and worst == whole.worst
    assert count == 3628800 and mean == whole.mean
    d5, r5 = synth.c5_batch_fast("nvidia", 5000)
    wo, wm, ws = _capi.heuristic_batch(d5, r5, 2, 0.5, osim.SUM_MODE)
    assert np.array_equal(o5, wo) and np.array_equal(m5, wm) and np.array_equal(s5, ws)
    assert summ.tobytes() == _capi.exhaustive_batch(synth.c2_batch(300), 2, 0.5).tobytes()


def test_sigma_at_the_fast_range_boundary():
    # sigma = 2^-60 is the smallest fast-path sigma; just below it the
    # general (IEEE division) path runs; both bit-exact with the oracle
    rng = np.random.default_rng(17)
    d = rng.uniform(0.5, 4.0, (6, 3))
    r = np.arange(6, dtype=np.uint8)
    for sigma in (2.0 ** -60, np.nextafter(2.0 ** -60, 0.0), 1e-20, 2.0 ** -59 * 3):
        assert _capi.fast_eligible(d, sigma) == (sigma >= 2.0 ** -60)
        s, ms = _capi.exhaustive(d, 2, sigma, 0, 720, want_makespans=True)
        o, oms = O.exhaustive(d, 2, sigma, makespans=True)
        assert np.array_equal(ms, oms)
        assert_summary_vs_oracle(s, o)
        order, hm, sims = _capi.heuristic_batch(d[None], r[None], 2, sigma, osim.SUM_MODE)
        oo, om, osims = O.reorder(d, r, 2, sigma, osim.SUM_MODE)
        assert order[0].tolist() == oo and hm[0] == om


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 10, 12, 14, 16])
def test_null_stage_fast_path_vs_oracle(n):
    # every stage either 0 (no command) or in the fast range: NullSim path
    rng = np.random.default_rng(400 + n)
    d = rng.uniform(0.1, 5.0, (n, 3))
    d[rng.random((n, 3)) < 0.25] = 0.0
    d[0, 0] = 0.0  # at least one null stage
    for t in range(n):  # a task keeps at least one command
        if not d[t].any():
            d[t, 1] = 1.5
    total = math.factorial(n)
    lo, hi = (0, total) if total <= 400_000 else (total // 3, total // 3 + 400_000)
    assert not _capi.fast_eligible(d, 0.5)
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        s, ms = _capi.exhaustive(d, dma, sigma, lo, hi, want_makespans=True)
        o, oms = O.exhaustive(d, dma, sigma, lo, hi, threads=os.cpu_count() or 4, makespans=True)
        assert np.array_equal(ms, oms), (n, dma, sigma)
        assert_summary_vs_oracle(s, o)


@pytest.mark.parametrize("n", [7, 8])
def test_batch_null_stages_vs_oracle(n):
    # batched groups with null stages in the fast range: one CTA per group, NullSim
    rng = np.random.default_rng(500 + n)
    B = 64
    d = rng.uniform(0.1, 5.0, (B, n, 3))
    d[rng.random((B, n, 3)) < 0.2] = 0.0
    d[(d == 0).all(axis=2), 1] = 2.0
    cpus = os.cpu_count() or 4
    for dma, sigma in ((2, 0.5), (2, 0.375), (1, 1.0)):
        out = _capi.exhaustive_batch(d, dma, sigma)
        for b in range(0, B, 3):
            o, _ = O.exhaustive(d[b], dma, sigma, threads=cpus)
            assert_summary_vs_oracle({k: out[b][k].item() for k in out.dtype.names}, o)


def test_concurrent_host_calls_from_threads():
    # ctypes releases the GIL: several Python threads drive the library at
    # once; the per-device mutex keeps scratch/streams consistent
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(23)
    groups = [rng.uniform(0.2, 4.0, (9, 3)) for _ in range(8)]
    expect = [_capi.exhaustive(g, 2, 0.5, 0, 362880)[0] for g in groups]
    hd, hr = synth.c5_batch_fast("amd", 4096, seed=5)
    h_expect = _capi.heuristic_batch(hd, hr, 2, 0.375, osim.SUM_MODE)

    def work(i):
        if i % 3 == 2:
            o, m, s_ = _capi.heuristic_batch(hd, hr, 2, 0.375, osim.SUM_MODE)
            return ("h", np.array_equal(o, h_expect[0]) and np.array_equal(m, h_expect[1]))
        g = i % len(groups)
        s, _ = _capi.exhaustive(groups[g], 2, 0.5, 0, 362880)
        return ("e", s == expect[g])

    with ThreadPoolExecutor(6) as ex:
        res = list(ex.map(work, range(36)))
    assert all(ok for _, ok in res)


@pytest.mark.parametrize("profile", ["nvidia", "amd", "phi"])
def test_heuristic_null_stages_vs_oracle(profile):
    # 16-task groups with null stages (the device check reroutes the batch to
    # the NullSim heuristic): order, makespan and simulation count bit-exact
    d, r = synth.c5_batch_fast(profile, 2000, seed=91)
    rng = np.random.default_rng(92)
    d = d.copy()
    d[rng.random(d.shape) < 0.1] = 0.0
    d[(d == 0).all(axis=2), 1] = 1.0
    _, dma, sigma = synth.PROFILES[profile]
    order, ms, sims = _capi.heuristic_batch(d, r, dma, sigma, osim.SUM_MODE)
    o_order, o_ms, o_sims = O.reorder_batch(d, r, dma, sigma, osim.SUM_MODE, threads=os.cpu_count() or 4)
    assert np.array_equal(order, o_order) and np.array_equal(ms, o_ms) and np.array_equal(sims, o_sims)


# ---- groups of 17..64 tasks (csrc/osim_wide.cuh; tests/golden/wide.json) -----

def _wide_check_timeline(st, en, c, n):
    for t in range(n):
        for k in range(3):
            s = c["start"][t][k]
            if s is None:
                assert st[t, k] == -1.0
            else:
                assert st[t, k] == F(s) and en[t, k] == F(c["end"][t][k])


def test_wide_timelines_bit_exact():
    g = load("wide.json")
    for c in g["timelines"]:
        st, en, ms, idle = _capi.timeline(durs(c["durs"]), c["dma"], F(c["sigma"]), c["order"])
        assert ms == F(c["makespan"]) and idle.tolist() == fl(c["idle"])
        _wide_check_timeline(st, en, c, c["n"])
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
        assert ms == F(c["makespan"]) and idle.tolist() == fl(c["idle"])
        _wide_check_timeline(st, en, c, T * N)


def test_wide_simulate_dropin():
    # engine.simulate on a 48-task group through the drop-in API
    c = [x for x in load("wide.json")["timelines"] if x["n"] >= 40][0]
    p = osim.DeviceProfile("g", c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))
    d = durs(c["durs"])
    tasks = [osim.TaskSpec(f"t{i}", fixed_durations=tuple(d[i])) for i in c["order"]]
    tl = osim.simulate(tasks, p)
    assert tl.makespan == F(c["makespan"]) and [tl.idle[k] for k in osim.KINDS] == fl(c["idle"])
    assert [osim.KINDS.index(x.kind) for x in tl.commands] == c["sorted_kinds"]
    assert [int(x.task_id[1:]) for x in tl.commands] == c["sorted_tasks"]


def test_wide_heuristic_goldens_and_batch_vs_oracle():
    g = load("wide.json")
    mode = g["meta"]["sum_mode"]
    assert mode == osim.SUM_MODE
    for c in g["heuristic"]:
        order, ms, sims = _capi.heuristic_batch(durs(c["durs"])[None], np.array(c["id_rank"], np.uint8)[None],
                                                c["dma"], F(c["sigma"]), mode)
        assert order[0].tolist() == c["order"] and ms[0] == F(c["makespan"]) and sims[0] == c["n_sims"]
    # batches of real-task groups (17..24 tasks) against the oracle
    cpus = os.cpu_count() or 4
    for prof, n, B in (("nvidia", 20, 384), ("amd", 17, 256), ("phi", 24, 192)):
        _, dma, sigma = synth.PROFILES[prof]
        dev = {"nvidia": "K20", "amd": "AMD", "phi": "PHI"}[prof]
        d = np.stack([synth.real_group(dev, n, 500 + b)[1] for b in range(B)])
        r = np.stack([np.random.default_rng(b).permutation(n) for b in range(B)]).astype(np.uint8)
        order, ms, sims = _capi.heuristic_batch(d, r, dma, sigma, mode)
        oo, om, osims = O.reorder_batch(d, r, dma, sigma, mode, threads=cpus)
        assert np.array_equal(order, oo) and np.array_equal(ms, om) and np.array_equal(sims, osims)


def test_wide_sampled_search_and_noreorder():
    import hashlib

    from paper_1806_10113_b200 import noreorder as nr
    from paper_1806_10113_b200.search import sample_permutations

    g = load("wide.json")
    for c in g["sampled"]:
        d = durs(c["durs"])
        p = osim.DeviceProfile("g", c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))
        tasks = [osim.TaskSpec(f"t{i}", fixed_durations=tuple(d[i])) for i in range(c["n"])]
        rep = osim.exhaustive_search(tasks, p, cap=c["cap"], seed=c["seed"])  # sampled mode (n! > cap)
        assert rep.exhaustive is False
        assert sha(np.array(rep.makespans)) == c["makespans_sha256"]
        assert [int(x[1:]) for x in rep.best_ordering] == c["best_ordering"]
        assert rep.best == F(c["best"]) and rep.median == F(c["median"]) and rep.worst == F(c["worst"])
        perms = sample_permutations(c["n"], c["cap"], c["seed"])
        s, ms = _capi.eval_perms(d, c["dma"], F(c["sigma"]), perms)
        assert s["best_rank"] == c["argmin"] and sha(ms) == c["makespans_sha256"]
    for c in g["noreorder"]:
        d = np.array([[[F(x) for x in r] for r in row] for row in c["durs"]])
        labels, ms, summ, exhaustive = nr.distribution_durs(d, c["dma"], F(c["sigma"]), c["cap"], c["seed"])
        assert exhaustive is False and len(ms) == c["count"]
        assert hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest() == c["makespans_sha256"]
        assert summ["best_rank"] == c["argmin"] and summ["best"] == F(c["best"]) and summ["worst"] == F(c["worst"])
        assert float(np.median(ms)) == F(c["median"])


def test_wide_eval_perms_64_tasks_vs_oracle():
    # the largest groups (64 tasks), null stages, both DMA modes
    rng = np.random.default_rng(64)
    d = rng.uniform(0.1, 4.0, (64, 3))
    d[rng.random((64, 3)) < 0.1] = 0.0
    d[:, 1] = np.maximum(d[:, 1], 0.05)  # every task keeps a command
    perms = np.stack([rng.permutation(64) for _ in range(4000)]).astype(np.uint8)
    for dma, sigma in ((2, 0.375), (1, 1.0)):
        s, ms = _capi.eval_perms(d, dma, sigma, perms)
        o, oms = O.eval_perms(d, dma, sigma, perms, threads=os.cpu_count() or 4)
        assert np.array_equal(ms, oms)
        assert_summary_vs_oracle(s, o)


def test_wide_harness_bit_exact_and_dropin():
    # the paper's scenario sizes (T = 6, 8 workers x N = 4 dependent tasks)
    g = load("wide.json")
    mode = g["meta"]["sum_mode"]
    for c in g["harness"]:
        d = durs(c["durs"])[None]
        r = np.array(c["id_rank"], dtype=np.uint8)[None]
        ms, ng, sz, st, en = _capi.harness_batch(d, r, c["T"], c["N"], c["dma"], F(c["sigma"]), mode, timeline=True)
        assert ms[0] == F(c["makespan"]) and sz[0, : ng[0]].tolist() == c["tg_sizes"], (c["T"], c["N"], c["bk"])
    from paper_1806_10113_b200 import workload as wl

    c = [x for x in g["harness"] if x["T"] == 8 and x["N"] == 4 and x["bk"] != "real"][0]
    p = osim.DeviceProfile("p", c["dma"], 0.0, 1.0, 0.0, 1.0, overlap_sigma=F(c["sigma"]))
    sc = wl.Scenario(8, 4, wl.load_bk_benchmark(c["bk"]), c["seed"], p)
    res = wl.run_scenario(sc, evaluate_noreorder=True, cap=500)  # NoReorder sampled over 32-task sequences
    assert res.heuristic_makespan == F(c["makespan"]) and res.tg_sizes == c["tg_sizes"]
    assert [res.timeline.idle[k] for k in osim.KINDS] == fl(c["idle"])
    assert res.noreorder is not None and len(res.noreorder.makespans) == 500
    assert res.speedup_best >= res.speedup_median


def _oracle_union(d, dma, sigma, ranges):
    from paper_1806_10113_b200 import dist as odist

    return odist.combine([O.exhaustive(d, dma, sigma, lo, hi, threads=8)[0] for lo, hi in ranges])


@pytest.mark.parametrize("n,world", [(8, 2), (8, 3), (8, 5), (7, 2), (9, 4)])
def test_interleaved_shard_partition_vs_oracle(n, world):
    # fast path: shard s of W = the 512-prefix calls s, s + W, ... of the
    # whole space, each 512 * L! consecutive ranks (n = 8: L = 3, 3072 ranks;
    # osim_exhaustive_shard, offsim_b200.h); dist.shard_ranges states it
    from paper_1806_10113_b200 import dist as odist

    d = synth.c2_batch(1)[0] if n == 8 else synth.c3_group()[:n].copy()
    for s in range(world):
        got = _capi.exhaustive_shard(d, 2, 0.5, s, world)
        want = _oracle_union(d, 2, 0.5, odist.shard_ranges(n, s, world))
        assert_summary_vs_oracle(got, want)


@pytest.mark.parametrize("case", ["c3", "c4_w8", "c4_sigma0.375", "c4_1dma", "null_stage", "general"])
def test_shards_combine_to_the_whole_space(case):
    from paper_1806_10113_b200 import dist as odist

    dma, sigma, world = 2, 0.5, 3
    if case == "c3":
        d = synth.c3_group()
    elif case == "c4_w8":
        d, world = synth.c4_group(), 8
    elif case == "c4_sigma0.375":
        d, sigma, world = synth.c4_group(), 0.375, 4
    elif case == "c4_1dma":
        d, dma, sigma, world = synth.c4_group(), 1, 1.0, 2
    elif case == "null_stage":  # NullSim path: contiguous shards
        d = synth.c3_group().copy()
        d[3, 0] = 0.0
    else:  # general path (a duration outside the fast range): contiguous shards
        d = synth.c3_group()[:9].copy()
        d[2, 1] = 2.0 ** 23
    whole, _ = _capi.exhaustive(d, dma, sigma, 0, math.factorial(d.shape[0]))
    parts = [_capi.exhaustive_shard(d, dma, sigma, s, world) for s in range(world)]
    assert sum(p["count"] for p in parts) == whole["count"]
    got = odist.combine(parts)
    assert got["best"] == whole["best"] and got["best_rank"] == whole["best_rank"]
    assert got["worst"] == whole["worst"] and got["count"] == whole["count"]
    assert close(got["sum"], whole["sum"], REL) and close(got["sum_log"], whole["sum_log"], REL)


def test_shard_arguments_are_checked():
    d = synth.c3_group()
    for s, w in ((0, 0), (-1, 2), (2, 2)):
        with pytest.raises(ValueError, match="shard"):  # OSIM_EINVAL, the reference's error type
            _capi.exhaustive_shard(d, 2, 0.5, s, w)
