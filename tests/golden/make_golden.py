"""Generate golden fixtures by running the UNMODIFIED reference (offsim).

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--c3]

The reference is imported read-only from /root/reference/pkg/src.  Every
float is stored as ``float.hex`` so the fixtures are bit-exact.  The Python
version is recorded because builtin ``sum()`` (heuristic.py:47) changed to
Neumaier summation in CPython 3.12.

Fixtures (all under tests/golden/):
  c1_bk.json          BK0..BK100 x {1dma, 2dma}: exhaustive report + heuristic (config 1)
  sim_random.json     random ordered groups: full timelines, k_end, idle, steps
  heuristic_random.json  random groups through reorder_batch (sum-sensitive)
  c2_tg.json          config-2 TGs 0..3 (8 tasks, 8! orderings each)
  c4_sample.json      config-4 input (AMD, 12 tasks): strided-rank makespans, sigma 0.5 / 0.375
  c5_sample.json      config-5 inputs (16 tasks) x 3 profiles through reorder_batch
  sampled.json        exhaustive_search in sampled (cap) mode
  c3_full.json        (--c3, ~3 min on 8 cores) config-3 full 10! sweep
  wide.json           groups of 17..64 tasks: timelines (plain, deps, 1-DMA waves),
                      reorder_batch, sampled exhaustive_search, sampled NoReorder
  big.json            groups above 64 tasks (to 300), NoReorder enumeration beyond 16
                      tasks, micro_simulate beyond 16 tasks, reorder_batch of one task
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import multiprocessing as mp
import os
import sys
from itertools import islice, permutations

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import offsim  # noqa: E402
from offsim import engine, heuristic  # noqa: E402
from offsim.model import DeviceProfile, TaskSpec  # noqa: E402
from offsim.oracle import exhaustive_search  # noqa: E402
from offsim.workload import BK_NAMES, load_bk_benchmark, sample_real_tasks  # noqa: E402
from offsim.cli import load_profile_arg  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
H = float.hex


def meta():
    return {
        "python": sys.version.split()[0],
        "sum_mode": 1 if sys.version_info >= (3, 12) else 0,
        "numpy": np.__version__,
        "generator": "tests/golden/make_golden.py",
        "reference": REF_SRC,
    }


def dump(name, doc):
    doc = {"meta": meta(), **doc}
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(doc, fh, indent=None, separators=(",", ":"))
        fh.write("\n")
    print("wrote", name, os.path.getsize(os.path.join(HERE, name)), "bytes")


def prof(dma, sigma):
    return DeviceProfile("g", dma, 0.0, 1.0, 0.0, 1.0, overlap_sigma=sigma)


def counting_reorder(tasks, profile):
    """reorder_batch with the number of simulate() calls it made."""
    calls = [0]
    real = heuristic.simulate

    def counted(*a, **k):
        calls[0] += 1
        return real(*a, **k)

    heuristic.simulate = counted
    try:
        out = heuristic.reorder_batch(tasks, profile)
    finally:
        heuristic.simulate = real
    return out, calls[0]


def run_steps(tasks, profile):
    sim = engine.DeviceSim(profile)
    sim.submit(tasks)
    steps = 0
    while not sim.drained():
        assert sim.step() is not None
        steps += 1
    return sim.timeline(), steps


def timeline_doc(tasks, order_idx, profile):
    ordered = [tasks[i] for i in order_idx]
    tl, steps = run_steps(ordered, profile)
    ref = engine.simulate(ordered, profile)
    assert ref.makespan == tl.makespan
    idx = {t.id: i for i, t in enumerate(tasks)}
    kinds = {engine.KIND_HTD: 0, engine.KIND_K: 1, engine.KIND_DTH: 2}
    start = [[None] * 3 for _ in tasks]
    end = [[None] * 3 for _ in tasks]
    for c in tl.commands:
        start[idx[c.task_id]][kinds[c.kind]] = H(c.start)
        end[idx[c.task_id]][kinds[c.kind]] = H(c.end)
    k_end = max((c.end for c in tl.commands if c.kind == engine.KIND_K), default=0.0)
    return {
        "makespan": H(tl.makespan),
        "k_end": H(k_end),
        "idle": [H(tl.idle[k]) for k in engine.KINDS],
        "start": start,
        "end": end,
        "steps": steps,
        "sorted_kinds": [kinds[c.kind] for c in tl.commands],
        "sorted_tasks": [idx[c.task_id] for c in tl.commands],
    }


def durs_of(tasks, profile=None):
    return [[H(float(x)) for x in offsim.stage_times(t, profile)] for t in tasks]


def id_rank(tasks):
    order = sorted(range(len(tasks)), key=lambda i: tasks[i].id)
    rank = [0] * len(tasks)
    for r, i in enumerate(order):
        rank[i] = r
    return rank


def report_doc(tasks, profile, cap=10_000, seed=0, full=True):
    rep = exhaustive_search(tasks, profile, cap=cap, seed=seed)
    ms = np.asarray(rep.makespans)
    idx = {t.id: i for i, t in enumerate(tasks)}
    orderings = [[idx[i] for i in o] for o in rep.orderings]
    head = len(ms) if full else 64
    return {
        "count": len(ms),
        "makespans": [H(m) for m in rep.makespans[:head]],
        "orderings": orderings[:head],
        "makespans_sha256": hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest(),
        "orderings_sha256": hashlib.sha256(np.asarray(orderings, dtype=np.uint8).tobytes()).hexdigest(),
        "best": H(rep.best),
        "argmin": int(np.argmin(ms)),
        "best_ordering": [idx[i] for i in rep.best_ordering],
        "worst": H(rep.worst),
        "median": H(rep.median),
        "geomean": H(rep.geomean),
        "mean": H(float(ms.mean())),
        "exhaustive": rep.exhaustive,
    }


def heuristic_doc(tasks, profile):
    out, calls = counting_reorder(tasks, profile)
    idx = {t.id: i for i, t in enumerate(tasks)}
    return {
        "order": [idx[t.id] for t in out],
        "makespan": H(engine.simulate(out, profile).makespan),
        "n_sims": calls,
    }


# ---------------------------------------------------------------- C1
def gen_c1():
    cases = []
    for name in BK_NAMES:
        tasks = list(load_bk_benchmark(name).tasks)
        for pname in ("1dma", "2dma"):
            p = load_profile_arg(pname)
            cases.append(
                {
                    "bk": name,
                    "profile": pname,
                    "dma": p.dma_engines,
                    "sigma": H(p.overlap_sigma),
                    "ids": [t.id for t in tasks],
                    "durs": durs_of(tasks, p),
                    "id_rank": id_rank(tasks),
                    "report": report_doc(tasks, p),
                    "heuristic": heuristic_doc(tasks, p),
                    "timeline_identity": timeline_doc(tasks, list(range(len(tasks))), p),
                }
            )
    dump("c1_bk.json", {"cases": cases})


# ---------------------------------------------------------- random sims
def rand_task_durs(rng, n, mode):
    out = []
    for _ in range(n):
        while True:
            if mode == "int":
                d = [float(rng.integers(0, 6)) for _ in range(3)]
            elif mode == "mixed":
                d = [float(rng.integers(1, 4)) if rng.random() < 0.5 else float(rng.uniform(0.1, 5.0)) for _ in range(3)]
            else:
                d = [float(rng.uniform(0.01, 10.0)) for _ in range(3)]
            for k in range(3):
                if mode != "int" and rng.random() < 0.12:
                    d[k] = 0.0
            if d[0] + d[2] > 0 or d[1] > 0:
                if max(d) > 0:
                    break
        out.append(d)
    return out


def gen_sim_random(count=800):
    rng = np.random.default_rng(1806_10113)
    sigmas = [0.375, 0.5, 0.8, 1.0]
    cases = []
    for c in range(count):
        n = int(rng.integers(1, 9))
        mode = ["int", "mixed", "real"][c % 3]
        dma = 1 + (c // 3) % 2
        sigma = sigmas[(c // 6) % 4]
        d = rand_task_durs(rng, n, mode)
        tasks = [TaskSpec(id=f"t{i}", fixed_durations=tuple(d[i])) for i in range(n)]
        order = [int(x) for x in rng.permutation(n)]
        p = prof(dma, sigma)
        doc = timeline_doc(tasks, order, p)
        doc.update({"n": n, "dma": dma, "sigma": H(sigma), "durs": [[H(x) for x in r] for r in d], "order": order})
        cases.append(doc)
    dump("sim_random.json", {"cases": cases})


# ------------------------------------------------------ random heuristic
DEVICE_PROFILES = {
    # config 5: NVIDIA-style, AMD-style, Xeon-Phi-style
    "nvidia": ("K20", 2, 0.5),
    "amd": ("AMD", 2, 0.375),
    "phi": ("PHI", 1, 1.0),
}


def gen_heuristic_random():
    rng = np.random.default_rng(7)
    cases = []
    for pname, (dev, dma, sigma) in DEVICE_PROFILES.items():
        p = prof(dma, sigma)
        for n in range(1, 17):
            for rep in range(3 if n < 16 else 10):
                seed = 1000 * n + rep
                tasks = sample_real_tasks(dev, n, seed=seed)
                doc = heuristic_doc(tasks, p)
                doc.update({"profile": pname, "dma": dma, "sigma": H(sigma), "n": n, "seed": seed,
                            "ids": [t.id for t in tasks], "durs": durs_of(tasks), "id_rank": id_rank(tasks)})
                cases.append(doc)
    # small integer-valued groups (ties everywhere), like tests/test_heuristic.py:113-128
    for c in range(120):
        n = int(rng.integers(1, 8))
        dma = 1 + c % 2
        sigma = [0.5, 0.375, 1.0, 0.8][c % 4]
        d = rand_task_durs(rng, n, "int" if c % 2 else "mixed")
        ids = [f"x{int(v)}" for v in rng.permutation(100)[:n]]
        tasks = [TaskSpec(id=ids[i], fixed_durations=tuple(d[i])) for i in range(n)]
        p = prof(dma, sigma)
        doc = heuristic_doc(tasks, p)
        doc.update({"profile": "rand", "dma": dma, "sigma": H(sigma), "n": n, "seed": c,
                    "ids": ids, "durs": durs_of(tasks), "id_rank": id_rank(tasks)})
        cases.append(doc)
    dump("heuristic_random.json", {"cases": cases})


# ---------------------------------------------------------------- C2
C2_SEED = 18061011302
C2_TABLE2 = [(0.1, 0.8, 0.1), (0.2, 0.7, 0.1), (0.3, 0.6, 0.1), (0.1, 0.7, 0.2),
             (0.6, 0.2, 0.2), (0.2, 0.2, 0.6), (0.4, 0.2, 0.4), (0.8, 0.1, 0.1)]


def c2_durations(n_tg):
    """Config-2 inputs: Table-2 x 10 ms x U(0.5, 1.5)."""
    base = np.array([[f * 10.0 for f in row] for row in C2_TABLE2])
    rng = np.random.default_rng(C2_SEED)
    return base[None] * rng.uniform(0.5, 1.5, (100000, 8, 3))[:n_tg]


def gen_c2(n_tg=4):
    d = c2_durations(n_tg)
    p = load_profile_arg("2dma")
    tgs = []
    for b in range(n_tg):
        tasks = [TaskSpec(id=f"t{i:02d}", fixed_durations=tuple(float(x) for x in d[b, i])) for i in range(8)]
        rep = exhaustive_search(tasks, p, cap=40320)
        ms = np.asarray(rep.makespans)
        tgs.append({
            "tg": b,
            "durs": [[H(float(x)) for x in r] for r in d[b]],
            "best": H(rep.best), "argmin": int(np.argmin(ms)), "worst": H(rep.worst),
            "median": H(rep.median), "geomean": H(rep.geomean), "mean": H(float(ms.mean())),
            "sum": H(float(ms.sum())),
            "makespans_sha256": hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest(),
            "makespans_head": [H(float(m)) for m in ms[:512]],
        })
        print("c2 tg", b, rep.best)
    dump("c2_tg.json", {"seed": C2_SEED, "dma": 2, "sigma": H(0.5), "tgs": tgs})


# ---------------------------------------------------------------- C4
def gen_c4(samples=2000):
    tasks = sample_real_tasks("AMD", 12, seed=12)
    total = math.factorial(12)
    stride = total // samples
    ranks = [k * stride for k in range(samples)] + [total - 1]
    out = {}
    for sigma in (0.5, 0.375):
        p = prof(2, sigma)
        ms = []
        for r in ranks:
            perm = unrank(r, 12)
            ms.append(H(engine.simulate([tasks[i] for i in perm], p).makespan))
        out[str(sigma)] = ms
    dump("c4_sample.json", {"durs": durs_of(tasks), "ids": [t.id for t in tasks], "dma": 2,
                            "ranks": ranks, "makespans": out})


def unrank(r, n):
    avail = list(range(n))
    perm = []
    for i in range(n):
        f = math.factorial(n - 1 - i)
        d, r = divmod(r, f)
        perm.append(avail.pop(d))
    return perm


# ---------------------------------------------------------------- C5
def gen_c5(per_profile=200):
    out = []
    for pname, (dev, dma, sigma) in DEVICE_PROFILES.items():
        p = prof(dma, sigma)
        rows = []
        for b in range(per_profile):
            tasks = sample_real_tasks(dev, 16, seed=b)
            doc = heuristic_doc(tasks, p)
            rows.append({"b": b, "ids": [t.id for t in tasks], "durs": durs_of(tasks),
                         "id_rank": id_rank(tasks), **doc})
        out.append({"profile": pname, "device": dev, "dma": dma, "sigma": H(sigma), "rows": rows})
        print("c5", pname)
    dump("c5_sample.json", {"profiles": out})


# ------------------------------------------------------------ sampled
def gen_sampled():
    p = load_profile_arg("2dma")
    cases = []
    t6 = [TaskSpec(id=f"t{i}", fixed_durations=(0.5 + 0.1 * i, 2.0, 0.5)) for i in range(6)]
    cases.append({"name": "six_cap50_seed9", "cap": 50, "seed": 9, "durs": durs_of(t6),
                  **report_doc(t6, p, cap=50, seed=9)})
    t8 = sample_real_tasks("K20", 8, seed=3)
    cases.append({"name": "k20_8_default_cap", "cap": 10_000, "seed": 0, "durs": durs_of(t8),
                  **report_doc(t8, p, full=False)})
    dump("sampled.json", {"dma": 2, "sigma": H(0.5), "cases": cases})


# ------------------------------------------------- row f1: NoReorder (deps)
def gen_noreorder():
    from offsim import workload
    from offsim.workload import Scenario

    cases = []
    for (T, N, bk, seed, pname, cap) in [(2, 2, "BK50", 1, "2dma", 10_000), (2, 2, "BK50", 1, "1dma", 10_000),
                                         (3, 2, "BK25", 2, "2dma", 10_000), (3, 2, "BK75", 3, "1dma", 10_000),
                                         (2, 3, "BK0", 4, "1dma", 10_000), (2, 4, "BK100", 5, "2dma", 10_000),
                                         (4, 2, "BK50", 6, "2dma", 10_000), (4, 2, "BK50", 6, "1dma", 10_000),
                                         (3, 3, "BK25", 7, "1dma", 2_000), (4, 3, "BK75", 8, "2dma", 1_000)]:
        p = load_profile_arg(pname)
        sc = Scenario(workers=T, batch_depth=N, pool=load_bk_benchmark(bk), seed=seed, profile=p)
        wt = workload._draw_worker_tasks(sc)
        rep = workload.noreorder_distribution(sc, wt, cap)
        ms = np.asarray(rep.makespans)
        idx = {wt[w][j].id: (w, j) for w in range(T) for j in range(N)}
        labels = [[idx[i][0] for i in o] for o in rep.orderings]
        cases.append({
            "T": T, "N": N, "bk": bk, "seed": seed, "profile": pname, "cap": cap,
            "dma": p.dma_engines, "sigma": H(p.overlap_sigma),
            "durs": [[[H(float(x)) for x in offsim.stage_times(wt[w][j], p)] for j in range(N)] for w in range(T)],
            "count": len(ms), "exhaustive": rep.exhaustive,
            "labels_head": labels[:200],
            "labels_sha256": hashlib.sha256(np.asarray(labels, dtype=np.uint8).tobytes()).hexdigest(),
            "makespans_head": [H(float(m)) for m in ms[:200]],
            "makespans_sha256": hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest(),
            "best": H(rep.best), "argmin": int(np.argmin(ms)), "worst": H(rep.worst),
            "median": H(rep.median), "geomean": H(rep.geomean),
        })
        print("noreorder", T, N, pname, len(ms), rep.exhaustive)
    # simulate_sequence timelines with deps (1-DMA waves and 2-DMA gates),
    # random worker interleavings incl. null stages
    rng = np.random.default_rng(99)
    seqs = []
    for c in range(300):
        T = int(rng.integers(1, 4)); N = int(rng.integers(1, 4))
        dma = 1 + c % 2
        sigma = [0.5, 0.375, 1.0][c % 3]
        p = prof(dma, sigma)
        d = rand_task_durs(rng, T * N, ["int", "mixed", "real"][c % 3])
        tasks = [[TaskSpec(id=f"w{w}.{j}", fixed_durations=tuple(d[w * N + j])) for j in range(N)] for w in range(T)]
        labels = [int(x) for x in rng.permutation([w for w in range(T) for _ in range(N)])]
        cnt = [0] * T
        seq = []
        for w in labels:
            seq.append(tasks[w][cnt[w]]); cnt[w] += 1
        deps = {tasks[w][j].id: tasks[w][j - 1].id for w in range(T) for j in range(1, N)}
        tl = workload.simulate_sequence(seq, p, deps)
        flat = [t for row in tasks for t in row]
        ix = {t.id: i for i, t in enumerate(flat)}
        kinds = {engine.KIND_HTD: 0, engine.KIND_K: 1, engine.KIND_DTH: 2}
        start = [[None] * 3 for _ in flat]
        end = [[None] * 3 for _ in flat]
        for cmd in tl.commands:
            start[ix[cmd.task_id]][kinds[cmd.kind]] = H(cmd.start)
            end[ix[cmd.task_id]][kinds[cmd.kind]] = H(cmd.end)
        seqs.append({"T": T, "N": N, "dma": dma, "sigma": H(sigma), "labels": labels,
                     "durs": [[H(x) for x in r] for r in d], "makespan": H(tl.makespan),
                     "idle": [H(tl.idle[k]) for k in engine.KINDS], "start": start, "end": end})
    dump("noreorder.json", {"cases": cases, "sequences": seqs})


# ------------------------------------------- row f4: micro-step tick oracle
def gen_micro():
    from offsim.oracle import micro_simulate

    cases = []
    for name in BK_NAMES:
        tasks = list(load_bk_benchmark(name).tasks)
        for pname in ("1dma", "2dma"):
            p = load_profile_arg(pname)
            ms = []
            for perm in permutations(range(4)):
                tl = micro_simulate([tasks[i] for i in perm], p, dt=0.001)
                ms.append(H(tl.makespan))
            cases.append({"bk": name, "profile": pname, "dma": p.dma_engines, "sigma": H(p.overlap_sigma),
                          "dt": H(0.001), "durs": durs_of(tasks, p), "makespans": ms})
    rng = np.random.default_rng(4242)
    rand = []
    for c in range(120):
        n = int(rng.integers(1, 6))
        dma = 1 + c % 2
        sigma = [0.5, 0.375, 1.0][c % 3]
        dt = [0.01, 0.005, 0.001, 0.0025][c % 4]
        d = rand_task_durs(rng, n, ["int", "mixed", "real"][c % 3])
        tasks = [TaskSpec(id=f"t{i}", fixed_durations=tuple(d[i])) for i in range(n)]
        order = [int(x) for x in rng.permutation(n)]
        tl = micro_simulate([tasks[i] for i in order], prof(dma, sigma), dt=dt)
        kinds = {engine.KIND_HTD: 0, engine.KIND_K: 1, engine.KIND_DTH: 2}
        start = [[None] * 3 for _ in range(n)]
        end = [[None] * 3 for _ in range(n)]
        for cmd in tl.commands:
            i = int(cmd.task_id[1:])
            start[i][kinds[cmd.kind]] = H(cmd.start)
            end[i][kinds[cmd.kind]] = H(cmd.end)
        rand.append({"n": n, "dma": dma, "sigma": H(sigma), "dt": H(dt), "durs": [[H(x) for x in r] for r in d],
                     "order": order, "makespan": H(tl.makespan), "start": start, "end": end,
                     "idle": [H(tl.idle[k]) for k in engine.KINDS]})
    dump("micro.json", {"cases": cases, "random": rand})


# ------------------------------------------ row f3: proxy-thread harness
def gen_harness():
    from offsim import workload
    from offsim.workload import Scenario

    cases = []
    rng = np.random.default_rng(2024)
    for c in range(60):
        T = int(rng.integers(1, 9))
        N = int(rng.integers(1, 5))
        while T * N > 16:
            N -= 1
        bk = BK_NAMES[c % 5]
        pname = ["1dma", "2dma"][c % 2]
        p = load_profile_arg(pname)
        seed = int(rng.integers(0, 10_000))
        sc = Scenario(workers=T, batch_depth=N, pool=load_bk_benchmark(bk), seed=seed, profile=p)
        wt = workload._draw_worker_tasks(sc)
        res = workload.run_scenario(sc, evaluate_noreorder=False)
        flat = [t for row in wt for t in row]
        order = sorted(range(len(flat)), key=lambda i: flat[i].id)
        rank = [0] * len(flat)
        for r, i in enumerate(order):
            rank[i] = r
        cases.append({"T": T, "N": N, "bk": bk, "profile": pname, "seed": seed, "dma": p.dma_engines,
                      "sigma": H(p.overlap_sigma), "ids": [t.id for t in flat], "id_rank": rank,
                      "durs": [[H(float(x)) for x in offsim.stage_times(t, p)] for t in flat],
                      "makespan": H(res.heuristic_makespan), "tg_sizes": res.tg_sizes})
    # real-task pools with ids beyond w9 (string order != numeric order)
    for c in range(20):
        T, N = 10 + c % 6, 1
        pool = workload.make_benchmark("real", sample_real_tasks("K20", 8, seed=c))
        p = [load_profile_arg("2dma"), prof(2, 0.375), load_profile_arg("1dma")][c % 3]
        sc = Scenario(workers=T, batch_depth=N, pool=pool, seed=c, profile=p)
        wt = workload._draw_worker_tasks(sc)
        res = workload.run_scenario(sc, evaluate_noreorder=False)
        flat = [t for row in wt for t in row]
        order = sorted(range(len(flat)), key=lambda i: flat[i].id)
        rank = [0] * len(flat)
        for r, i in enumerate(order):
            rank[i] = r
        cases.append({"T": T, "N": N, "bk": "real", "profile": str(c % 3), "seed": c, "dma": p.dma_engines,
                      "sigma": H(p.overlap_sigma), "ids": [t.id for t in flat], "id_rank": rank,
                      "durs": [[H(float(x)) for x in offsim.stage_times(t, p)] for t in flat],
                      "makespan": H(res.heuristic_makespan), "tg_sizes": res.tg_sizes})
    dump("harness.json", {"cases": cases})


# ---------------------------------------------------------------- C3
def _c3_chunk(args):
    lo, hi = args
    tasks = sample_real_tasks("K20", 10, seed=10)
    p = load_profile_arg("2dma")
    out = np.empty(hi - lo)
    for j, perm in enumerate(islice(permutations(range(10)), lo, hi)):
        out[j] = engine.simulate([tasks[i] for i in perm], p).makespan
    return lo, out


def gen_c3(procs=8):
    total = math.factorial(10)
    chunks = [(total * k // 64, total * (k + 1) // 64) for k in range(64)]
    ms = np.empty(total)
    with mp.Pool(procs) as pool:
        for lo, out in pool.imap_unordered(_c3_chunk, chunks):
            ms[lo:lo + len(out)] = out
    tasks = sample_real_tasks("K20", 10, seed=10)
    relabeled = [TaskSpec(id=f"t{i:02d}", fixed_durations=t.fixed_durations) for i, t in enumerate(tasks)]
    p = load_profile_arg("2dma")
    heur = heuristic_doc(relabeled, p)
    hms = float.fromhex(heur["makespan"])
    dump("c3_full.json", {
        "durs": durs_of(tasks), "dma": 2, "sigma": H(0.5),
        "best": H(float(ms.min())), "argmin": int(np.argmin(ms)), "worst": H(float(ms.max())),
        "median": H(float(np.median(ms))), "geomean": H(float(np.exp(np.log(ms).mean()))),
        "mean": H(float(ms.mean())), "count": total,
        "makespans_sha256": hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest(),
        "heuristic_relabeled_t00": heur,
        "below_heuristic": int((ms < hms).sum()),
    })


# ---------------------------------------------- groups of 17..64 tasks
def gen_wide():
    from offsim import workload
    from offsim.workload import Scenario

    rng = np.random.default_rng(64_17)
    timelines = []
    for c in range(60):
        n = int(rng.choice([17, 20, 24, 31, 33, 40, 48, 57, 64]))
        mode = ["int", "mixed", "real"][c % 3]
        dma = 1 + (c // 3) % 2
        sigma = [0.375, 0.5, 0.8, 1.0][(c // 6) % 4]
        d = rand_task_durs(rng, n, mode)
        tasks = [TaskSpec(id=f"t{i}", fixed_durations=tuple(d[i])) for i in range(n)]
        order = [int(x) for x in rng.permutation(n)]
        doc = timeline_doc(tasks, order, prof(dma, sigma))
        doc.update({"n": n, "dma": dma, "sigma": H(sigma), "durs": [[H(x) for x in r] for r in d], "order": order})
        timelines.append(doc)
    # simulate_sequence with NoReorder chains (deps; 1-DMA waves)
    seqs = []
    for c in range(40):
        T = int(rng.integers(2, 7)); N = int(rng.integers(3, 10))
        while T * N <= 16 or T * N > 64:
            T = int(rng.integers(2, 7)); N = int(rng.integers(3, 10))
        dma = 1 + c % 2
        sigma = [0.5, 0.375, 1.0][c % 3]
        p = prof(dma, sigma)
        d = rand_task_durs(rng, T * N, ["int", "mixed", "real"][c % 3])
        tasks = [[TaskSpec(id=f"w{w}.{j}", fixed_durations=tuple(d[w * N + j])) for j in range(N)] for w in range(T)]
        labels = [int(x) for x in rng.permutation([w for w in range(T) for _ in range(N)])]
        cnt = [0] * T
        seq = []
        for w in labels:
            seq.append(tasks[w][cnt[w]]); cnt[w] += 1
        deps = {tasks[w][j].id: tasks[w][j - 1].id for w in range(T) for j in range(1, N)}
        tl = workload.simulate_sequence(seq, p, deps)
        flat = [t for row in tasks for t in row]
        ix = {t.id: i for i, t in enumerate(flat)}
        kinds = {engine.KIND_HTD: 0, engine.KIND_K: 1, engine.KIND_DTH: 2}
        start = [[None] * 3 for _ in flat]
        end = [[None] * 3 for _ in flat]
        for cmd in tl.commands:
            start[ix[cmd.task_id]][kinds[cmd.kind]] = H(cmd.start)
            end[ix[cmd.task_id]][kinds[cmd.kind]] = H(cmd.end)
        seqs.append({"T": T, "N": N, "dma": dma, "sigma": H(sigma), "labels": labels,
                     "durs": [[H(x) for x in r] for r in d], "makespan": H(tl.makespan),
                     "idle": [H(tl.idle[k]) for k in engine.KINDS], "start": start, "end": end})
    # reorder_batch on real-task groups and on tie-heavy integer groups
    heur = []
    for pname, (dev, dma, sigma) in DEVICE_PROFILES.items():
        p = prof(dma, sigma)
        for n, seed in ((17, 1), (20, 2), (24, 3), (32, 4)):
            tasks = sample_real_tasks(dev, n, seed=seed)
            doc = heuristic_doc(tasks, p)
            doc.update({"profile": pname, "dma": dma, "sigma": H(sigma), "n": n, "seed": seed,
                        "ids": [t.id for t in tasks], "durs": durs_of(tasks), "id_rank": id_rank(tasks)})
            heur.append(doc)
    for c in range(12):
        n = int(rng.choice([17, 19, 22, 26]))
        dma = 1 + c % 2
        sigma = [0.5, 0.375, 1.0, 0.8][c % 4]
        d = rand_task_durs(rng, n, "int" if c % 2 else "mixed")
        ids = [f"x{int(v)}" for v in rng.permutation(100)[:n]]
        tasks = [TaskSpec(id=ids[i], fixed_durations=tuple(d[i])) for i in range(n)]
        doc = heuristic_doc(tasks, prof(dma, sigma))
        doc.update({"profile": "rand", "dma": dma, "sigma": H(sigma), "n": n, "seed": c,
                    "ids": ids, "durs": durs_of(tasks), "id_rank": id_rank(tasks)})
        heur.append(doc)
    # exhaustive_search in sampled mode (n! > cap)
    sampled = []
    for n, dev, pname, cap, seed in ((18, "K20", "2dma", 500, 5), (25, "AMD", "1dma", 300, 6)):
        p = load_profile_arg(pname)
        tasks = sample_real_tasks(dev, n, seed=seed)
        sampled.append({"n": n, "profile": pname, "dma": p.dma_engines, "sigma": H(p.overlap_sigma),
                        "cap": cap, "seed": seed, "durs": durs_of(tasks, p), **report_doc(tasks, p, cap, seed)})
    # NoReorder distribution in sampled mode (more than 16 tasks)
    noreorder = []
    for (T, N, bk, seed, pname, cap) in [(4, 5, "BK50", 11, "2dma", 400), (3, 7, "BK25", 12, "1dma", 300)]:
        p = load_profile_arg(pname)
        sc = Scenario(workers=T, batch_depth=N, pool=load_bk_benchmark(bk), seed=seed, profile=p)
        wt = workload._draw_worker_tasks(sc)
        rep = workload.noreorder_distribution(sc, wt, cap)
        ms = np.asarray(rep.makespans)
        idx = {wt[w][j].id: (w, j) for w in range(T) for j in range(N)}
        labels = [[idx[i][0] for i in o] for o in rep.orderings]
        noreorder.append({
            "T": T, "N": N, "bk": bk, "seed": seed, "profile": pname, "cap": cap,
            "dma": p.dma_engines, "sigma": H(p.overlap_sigma),
            "durs": [[[H(float(x)) for x in offsim.stage_times(wt[w][j], p)] for j in range(N)] for w in range(T)],
            "count": len(ms), "exhaustive": rep.exhaustive,
            "labels_sha256": hashlib.sha256(np.asarray(labels, dtype=np.uint8).tobytes()).hexdigest(),
            "makespans_sha256": hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest(),
            "best": H(rep.best), "argmin": int(np.argmin(ms)), "worst": H(rep.worst), "median": H(rep.median),
        })
    # the proxy-thread harness at the paper's scenario sizes (T = 6, 8 workers x N = 4)
    harness = []
    for c, (T, N) in enumerate([(6, 4), (8, 4), (5, 4), (4, 8), (8, 3), (6, 6), (8, 4), (6, 4),
                                (3, 7), (9, 2), (16, 2), (8, 8)]):
        if c < 8:
            bk = BK_NAMES[c % 5]
            pool = load_bk_benchmark(bk)
        else:
            bk = "real"
            pool = workload.make_benchmark("real", sample_real_tasks(["K20", "AMD", "PHI"][c % 3], 8, seed=c))
        p = [load_profile_arg("2dma"), load_profile_arg("1dma"), prof(2, 0.375)][c % 3]
        seed = 100 + c
        sc = Scenario(workers=T, batch_depth=N, pool=pool, seed=seed, profile=p)
        wt = workload._draw_worker_tasks(sc)
        res = workload.run_scenario(sc, evaluate_noreorder=False)
        flat = [t for row in wt for t in row]
        harness.append({"T": T, "N": N, "bk": bk, "seed": seed, "dma": p.dma_engines, "sigma": H(p.overlap_sigma),
                        "ids": [t.id for t in flat], "id_rank": id_rank(flat),
                        "durs": [[H(float(x)) for x in offsim.stage_times(t, p)] for t in flat],
                        "makespan": H(res.heuristic_makespan), "tg_sizes": res.tg_sizes,
                        "idle": [H(res.timeline.idle[k]) for k in engine.KINDS]})
    dump("wide.json", {"timelines": timelines, "sequences": seqs, "heuristic": heur, "sampled": sampled,
                       "noreorder": noreorder, "harness": harness})


# ------------------------------------------- groups above 64 tasks (any n)
def _multiset_perms(labels):
    """Every distinct permutation of `labels` (recursive choice of the next
    label).  Stands in for itertools.permutations inside the reference's
    sorted(set(permutations(labels))) (workload.py:262-265): the sorted set
    of distinct sequences is the same list, but (T*N)! raw permutations are
    out of reach above ~12 tasks."""
    counts = {}
    for x in labels:
        counts[x] = counts.get(x, 0) + 1
    keys = sorted(counts)
    out, cur = [], []

    def rec():
        if len(cur) == len(labels):
            out.append(tuple(cur))
            return
        for k in keys:
            if counts[k]:
                counts[k] -= 1
                cur.append(k)
                rec()
                cur.pop()
                counts[k] += 1

    rec()
    return out


def _seq_timeline(tasks_grid, labels, p):
    from offsim import workload

    T = len(tasks_grid)
    cnt = [0] * T
    seq = []
    for w in labels:
        seq.append(tasks_grid[w][cnt[w]]); cnt[w] += 1
    deps = {tasks_grid[w][j].id: tasks_grid[w][j - 1].id for w in range(T) for j in range(1, len(tasks_grid[w]))}
    tl = workload.simulate_sequence(seq, p, deps)
    flat = [t for row in tasks_grid for t in row]
    ix = {t.id: i for i, t in enumerate(flat)}
    kinds = {engine.KIND_HTD: 0, engine.KIND_K: 1, engine.KIND_DTH: 2}
    start = [[None] * 3 for _ in flat]
    end = [[None] * 3 for _ in flat]
    for cmd in tl.commands:
        start[ix[cmd.task_id]][kinds[cmd.kind]] = H(cmd.start)
        end[ix[cmd.task_id]][kinds[cmd.kind]] = H(cmd.end)
    return tl, start, end


def gen_big():
    """big.json: the reference on groups of more than 64 tasks (and the other
    drop-in divergences VERDICT r01 listed): timelines, simulate_sequence,
    reorder_batch, sampled exhaustive_search, NoReorder (exhaustive beyond 16
    tasks and sampled beyond 64), micro_simulate beyond 16 tasks, the harness
    beyond 64 tasks, and reorder_batch of one unresolvable task."""
    from offsim import workload
    from offsim.oracle import micro_simulate
    from offsim.workload import Scenario

    rng = np.random.default_rng(70_2)
    timelines = []
    for c, n in enumerate([65, 70, 70, 96, 130, 200, 257, 300]):
        mode = ["int", "mixed", "real"][c % 3]
        dma = 1 + c % 2
        sigma = [0.375, 0.5, 0.8, 1.0][(c // 2) % 4]
        d = rand_task_durs(rng, n, mode)
        tasks = [TaskSpec(id=f"t{i}", fixed_durations=tuple(d[i])) for i in range(n)]
        order = [int(x) for x in rng.permutation(n)]
        doc = timeline_doc(tasks, order, prof(dma, sigma))
        doc.update({"n": n, "dma": dma, "sigma": H(sigma), "durs": [[H(x) for x in r] for r in d], "order": order})
        timelines.append(doc)
        print("big timeline", n)
    seqs = []
    for c, (T, N) in enumerate([(5, 14), (9, 8), (3, 30), (13, 6)]):
        dma = 1 + c % 2
        sigma = [0.5, 0.375, 1.0, 0.8][c % 4]
        d = rand_task_durs(rng, T * N, ["int", "mixed", "real"][c % 3])
        grid = [[TaskSpec(id=f"w{w}.{j}", fixed_durations=tuple(d[w * N + j])) for j in range(N)] for w in range(T)]
        labels = [int(x) for x in rng.permutation([w for w in range(T) for _ in range(N)])]
        tl, start, end = _seq_timeline(grid, labels, prof(dma, sigma))
        seqs.append({"T": T, "N": N, "dma": dma, "sigma": H(sigma), "labels": labels,
                     "durs": [[H(x) for x in r] for r in d], "makespan": H(tl.makespan),
                     "idle": [H(tl.idle[k]) for k in engine.KINDS], "start": start, "end": end})
        print("big sequence", T, N)
    heur = []
    for pname, (dev, dma, sigma) in DEVICE_PROFILES.items():
        p = prof(dma, sigma)
        for n, seed in ((65, 1), (70, 2)):
            tasks = sample_real_tasks(dev, n, seed=seed)
            doc = heuristic_doc(tasks, p)
            doc.update({"profile": pname, "dma": dma, "sigma": H(sigma), "n": n, "seed": seed,
                        "ids": [t.id for t in tasks], "durs": durs_of(tasks), "id_rank": id_rank(tasks)})
            heur.append(doc)
            print("big heuristic", pname, n)
    for c, n in enumerate([70, 100]):
        dma = 1 + c % 2
        sigma = [0.5, 0.375][c % 2]
        d = rand_task_durs(rng, n, "int" if c % 2 else "mixed")
        ids = [f"x{int(v)}" for v in rng.permutation(1000)[:n]]
        tasks = [TaskSpec(id=ids[i], fixed_durations=tuple(d[i])) for i in range(n)]
        doc = heuristic_doc(tasks, prof(dma, sigma))
        doc.update({"profile": "rand", "dma": dma, "sigma": H(sigma), "n": n, "seed": c,
                    "ids": ids, "durs": durs_of(tasks), "id_rank": id_rank(tasks)})
        heur.append(doc)
        print("big heuristic rand", n)
    sampled = []
    for n, dev, pname, cap, seed in ((70, "K20", "2dma", 200, 7), (90, "PHI", "1dma", 120, 8)):
        p = load_profile_arg(pname)
        tasks = sample_real_tasks(dev, n, seed=seed)
        rep = report_doc(tasks, p, cap, seed, full=True)
        rep["orderings_sha256"] = hashlib.sha256(np.asarray(
            [[int(x) for x in o] for o in rep["orderings"]], dtype=np.uint32).tobytes()).hexdigest()
        rep["orderings"] = rep["orderings"][:8]
        sampled.append({"n": n, "profile": pname, "dma": p.dma_engines, "sigma": H(p.overlap_sigma),
                        "cap": cap, "seed": seed, "durs": durs_of(tasks, p), **rep})
        print("big sampled", n)
    noreorder = []
    real_perm = workload.permutations
    for (T, N, bk, seed, pname, cap) in [(2, 9, "BK50", 21, "2dma", 50_000), (2, 9, "BK75", 22, "1dma", 50_000),
                                         (2, 10, "BK25", 23, "2dma", 200_000), (7, 10, "BK50", 24, "1dma", 300),
                                         (5, 14, "BK100", 25, "2dma", 200)]:
        p = load_profile_arg(pname)
        sc = Scenario(workers=T, batch_depth=N, pool=load_bk_benchmark(bk), seed=seed, profile=p)
        wt = workload._draw_worker_tasks(sc)
        workload.permutations = _multiset_perms
        try:
            rep = workload.noreorder_distribution(sc, wt, cap)
        finally:
            workload.permutations = real_perm
        ms = np.asarray(rep.makespans)
        idx = {wt[w][j].id: (w, j) for w in range(T) for j in range(N)}
        labels = [[idx[i][0] for i in o] for o in rep.orderings]
        noreorder.append({
            "T": T, "N": N, "bk": bk, "seed": seed, "profile": pname, "cap": cap,
            "dma": p.dma_engines, "sigma": H(p.overlap_sigma),
            "durs": [[[H(float(x)) for x in offsim.stage_times(wt[w][j], p)] for j in range(N)] for w in range(T)],
            "count": len(ms), "exhaustive": rep.exhaustive,
            "labels_head": labels[:20],
            "labels_sha256": hashlib.sha256(np.asarray(labels, dtype=np.uint8).tobytes()).hexdigest(),
            "makespans_sha256": hashlib.sha256(ms.astype("<f8").tobytes()).hexdigest(),
            "makespans_head": [H(float(m)) for m in ms[:20]],
            "best": H(rep.best), "argmin": int(np.argmin(ms)), "worst": H(rep.worst), "median": H(rep.median),
            "geomean": H(rep.geomean), "best_ordering": [list(idx[i]) for i in rep.best_ordering],
        })
        print("big noreorder", T, N, len(ms), rep.exhaustive)
    micro = []
    for c, n in enumerate([17, 20, 33, 70, 120]):
        dma = 1 + c % 2
        sigma = [0.5, 0.375, 1.0][c % 3]
        dt = [0.01, 0.005, 0.02][c % 3]
        d = rand_task_durs(rng, n, ["int", "mixed", "real"][c % 3])
        tasks = [TaskSpec(id=f"t{i}", fixed_durations=tuple(d[i])) for i in range(n)]
        order = [int(x) for x in rng.permutation(n)]
        tl = micro_simulate([tasks[i] for i in order], prof(dma, sigma), dt=dt)
        kinds = {engine.KIND_HTD: 0, engine.KIND_K: 1, engine.KIND_DTH: 2}
        start = [[None] * 3 for _ in range(n)]
        end = [[None] * 3 for _ in range(n)]
        for cmd in tl.commands:
            i = int(cmd.task_id[1:])
            start[i][kinds[cmd.kind]] = H(cmd.start)
            end[i][kinds[cmd.kind]] = H(cmd.end)
        micro.append({"n": n, "dma": dma, "sigma": H(sigma), "dt": H(dt), "durs": [[H(x) for x in r] for r in d],
                      "order": order, "makespan": H(tl.makespan), "start": start, "end": end,
                      "idle": [H(tl.idle[k]) for k in engine.KINDS]})
        print("big micro", n)
    harness = []
    for c, (T, N) in enumerate([(5, 14), (9, 8), (70, 1), (33, 3)]):
        bk = BK_NAMES[c % 5]
        pool = load_bk_benchmark(bk) if c % 2 == 0 else workload.make_benchmark(
            "real", sample_real_tasks(["K20", "AMD", "PHI"][c % 3], 8, seed=c))
        p = [load_profile_arg("2dma"), load_profile_arg("1dma"), prof(2, 0.375)][c % 3]
        seed = 300 + c
        sc = Scenario(workers=T, batch_depth=N, pool=pool, seed=seed, profile=p)
        wt = workload._draw_worker_tasks(sc)
        res = workload.run_scenario(sc, evaluate_noreorder=False)
        flat = [t for row in wt for t in row]
        harness.append({"T": T, "N": N, "bk": bk, "seed": seed, "dma": p.dma_engines, "sigma": H(p.overlap_sigma),
                        "ids": [t.id for t in flat], "id_rank": id_rank(flat),
                        "durs": [[H(float(x)) for x in offsim.stage_times(t, p)] for t in flat],
                        "makespan": H(res.heuristic_makespan), "tg_sizes": res.tg_sizes,
                        "idle": [H(res.timeline.idle[k]) for k in engine.KINDS]})
        print("big harness", T, N)
    # reorder_batch of one task returns it without resolving its durations
    # (heuristic.py:113-114): an unresolvable task comes back unchanged
    from offsim.model import UnresolvableDuration

    lone = TaskSpec(id="lone", kernel_work=0.0)
    try:
        offsim.stage_times(lone, None)
        resolvable = True
    except UnresolvableDuration:
        resolvable = False
    single = {"id": lone.id, "resolvable": resolvable,
              "returned": [t.id for t in heuristic.reorder_batch([lone], load_profile_arg("2dma"))]}
    dump("big.json", {"timelines": timelines, "sequences": seqs, "heuristic": heur, "sampled": sampled,
                      "noreorder": noreorder, "micro": micro, "harness": harness, "single": single})


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    if a.c3:
        gen_c3()
        sys.exit(0)
    gens = {"c1": gen_c1, "sim": gen_sim_random, "heur": gen_heuristic_random, "c2": gen_c2,
            "c4": gen_c4, "c5": gen_c5, "sampled": gen_sampled, "noreorder": gen_noreorder,
            "micro": gen_micro, "harness": gen_harness, "wide": gen_wide, "big": gen_big}
    for k, g in gens.items():
        if not a.only or k in a.only.split(","):
            g()
