#!/usr/bin/env python3
"""Benchmark of the B200 hot path (BASELINE.json metric: orderings simulated
per second at N=10/12, heuristic TG decisions per second).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

Headline workload (BASELINE config 4): one 12-task group (the reference's
sample_real_tasks("AMD", 12, seed=12), 2-DMA, sigma 0.5); one step = the
exhaustive search of all 12! = 479,001,600 orderings -> best makespan,
lowest-rank argmin, worst, mean, geomean.  With N ranks rank r takes the
interleaved 512-prefix calls r, r + N, ... of the Lehmer-rank space (every
rank samples the whole space, so the per-rank work evens out) and the 48-byte
per-rank summaries are combined by one NCCL all_gather inside the step
(strong scaling).

`value` times the device-resident path (osim_exhaustive_shard_dev: inputs in HBM,
CUDA events on the launching stream, L2 flushed between steps and excluded).
`e2e` times the public host API (exhaustive_summary_durs /
dist.exhaustive_summary_distributed): host buffers, H2D + kernels + D2H +
combine per step.  `secondary` holds configs 3 (N=10), 2 (100k x 8! batch)
and 5 (10^6 x 16-task heuristic, three device profiles).
`--impl reference` times the CPU restatement of the reference algorithm
(oracle/osim_oracle.c, bit-exact with the reference) on all host cores on a
bounded sample of the same workload, stratified over the whole 12! space.
`cpu_baseline.python` times the unmodified Python reference itself
(baseline/_ref, tools/install_reference.sh) on strided C4 ranks, one process
per host core.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N12 = 12
TOTAL12 = math.factorial(12)
SIGMA = 0.5
DMA = 2
WORKLOAD = ("C4: one 12-task TG (reference sample_real_tasks('AMD', 12, seed=12)), 2-DMA, sigma 0.5; "
            "exhaustive search of all 12! = 479001600 orderings -> best/argmin/worst/mean/geomean")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def op_counts():
    with open(os.path.join(ROOT, "tests", "golden", "op_counts.json")) as fh:
        return json.load(fh)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 100 ms while the timed region runs."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        rows = []
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), f[5], f[6], f[7], f[8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- helpers
class Dist:
    def __init__(self, gpus):
        self.world = env_int("WORLD_SIZE", 1)
        self.rank = env_int("RANK", 0)
        self.local = env_int("LOCAL_RANK", 0)
        self.pg = None
        if gpus != self.world and self.world > 1:
            print(f"warning: --gpus {gpus} but WORLD_SIZE={self.world}", file=sys.stderr)

    def init(self):
        import torch

        torch.cuda.set_device(self.local)
        # OSIM_BENCH_FORCE_PG=1: the N>1 code path (NCCL process group, the
        # per-step all_gather, max-over-ranks) at world size 1, to exercise it
        # on a single-GPU box under torchrun --nproc-per-node 1
        if self.world > 1 or os.environ.get("OSIM_BENCH_FORCE_PG") == "1":
            import torch.distributed as tdist


            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            tdist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = tdist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t)
        return float(t.item())


def timed_steps(step, K, W, flush, sync):
    """W untimed warm-ups, then K steps each bracketed by CUDA events on
    the current stream; L2 flushed before every step (not timed)."""
    import torch

    for _ in range(W):
        step()
    sync()
    evs = []
    for _ in range(K):
        flush()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        step(e[1])
        e[2].record()
        evs.append(e)
    torch.cuda.synchronize()
    kern = sum(e[0].elapsed_time(e[1]) for e in evs) / 1e3
    total = sum(e[0].elapsed_time(e[2]) for e in evs) / 1e3
    return total, kern


# ---------------------------------------------------------------- our arm
def run_ours(a):
    import ctypes as C

    import torch

    # stdout carries exactly the one JSON line: native code that prints on
    # fd 1 (NCCL's version banner at process-group init) goes to stderr
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)

    from paper_1806_10113_b200 import _capi, dist as odist, search, synth

    D = Dist(a.gpus)
    D.init()
    _capi.set_device(D.local)
    L = _capi.load()
    dev = torch.device("cuda", D.local)
    # a dedicated (non-default) stream: the library maps a NULL stream to its
    # own stream, and torch's legacy default stream has handle 0
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    sp = C.c_void_p(stream.cuda_stream)
    assert stream.cuda_stream != 0
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.zero_()

    ops = op_counts()
    peak_tflops = _capi.fp64_peak_tflops()  # DFMA: 2 flops/instruction
    peak_ops = peak_tflops / 2.0  # FP64 pipe instructions/s (T/s)

    # ---- headline: C4 ------------------------------------------------------
    durs = synth.c4_group()
    fast = int(_capi.fast_eligible(durs, SIGMA))
    assert fast == 1, "the C4 group is fast-path eligible (every duration in [2^-60, 2^22) ms)"
    d_durs = torch.from_numpy(durs).to(dev)
    d_out = torch.zeros(6, dtype=torch.float64, device=dev)
    gathered = [torch.zeros(6, dtype=torch.float64, device=dev) for _ in range(D.world)]
    launches_per_step = 1 if fast == 1 else 2  # fast path: the kernel's last CTA does the final reduce

    # rank r's shard: the interleaved 512-prefix calls r, r + N, ... of 12!
    # (osim_exhaustive_shard_dev; at N = 1 the whole space, as osim_exhaustive_dev)
    def step(ev_kernel_done=None):
        _capi.check(L.osim_exhaustive_shard_dev(C.c_void_p(d_durs.data_ptr()), N12, DMA, SIGMA, D.rank, D.world,
                                                fast, C.c_void_p(d_out.data_ptr()), sp))
        if ev_kernel_done is not None:
            ev_kernel_done.record()
        if D.pg:
            D.pg.all_gather(gathered, d_out)

    D.barrier()
    torch.cuda.synchronize()
    with ClockSampler(D.local) as clk:
        t_total, t_kern = timed_steps(step, a.steps, a.warmup, flush, torch.cuda.synchronize)
    D.barrier()
    torch.cuda.synchronize()
    t_max = D.max(t_total)
    value = TOTAL12 * a.steps / t_max
    parts = [odist.unpack(g.cpu().numpy()) for g in gathered] if D.pg else [odist.unpack(d_out.cpu().numpy())]
    res = search.summary_from_dict(odist.combine(parts), N12)
    assert res.count == TOTAL12, res
    mine = odist.unpack(d_out.cpu().numpy())["count"]  # orderings this rank simulated per step

    ops_per = ops[f"c4_sigma{SIGMA}"]["ops"]
    kern_avg = t_kern / a.steps
    achieved = ops_per * mine / kern_avg / 1e12
    roof = {"bound": "fp64", "achieved": achieved, "peak": peak_ops, "unit": "TFLOP/s", "frac": achieved / peak_ops,
            "traffic": profile_traffic(),
            "definition": ("algorithmic FP64 ops per ordering (S+8R+2O = %.1f, tests/golden/op_counts.json, "
                           "DDIV counted as one op) x orderings per launch / CUDA-event launch time; peak = "
                           "measured DFMA instructions/s of this GPU (osim_fp64_peak, %.2f TFLOP/s at 2 "
                           "flops/DFMA), i.e. FP64-pipe issue capacity in ops/s" % (ops_per, peak_tflops)),
            "kernel": "k_exhaustive_pfx<12,2,sigma-pow2,L=4>", "launch_ms": kern_avg * 1e3,
            "ncu_executed": {k: v for k, v in profile_headline().items()
                             if k in ("issue_active_pct", "fp64_pipe_active_pct", "alu_pipe_active_pct",
                                      "warp_exec_efficiency", "achieved_occupancy_pct",
                                      "theoretical_occupancy_pct", "source")}}
    # the same against the nominal FP64 pipe rate (64 FP64 lanes per SM x SMs x
    # the SM clock sampled during the timed region): MEASURED_PEAKS.json has no
    # FP64 entry, so both denominators are reported
    sm_mhz_fp = clk.summary().get("sm_mhz")
    if sm_mhz_fp:
        sms_fp = torch.cuda.get_device_properties(dev).multi_processor_count
        nominal = 64.0 * sms_fp * sm_mhz_fp * 1e6 / 1e12
        roof["peak_nominal"] = nominal
        roof["frac_nominal"] = achieved / nominal
    # the issue roofline (SURVEY 8(d) ii): warp instructions the kernel executes
    # per launch (the committed ncu capture of the same kernel on the whole
    # 12! space, scaled to this rank's shard) over 4 issues/clk/SM x SMs x the
    # SM clock measured during the timed region
    wi = profile_headline().get("warp_instructions_per_launch")
    sm_mhz = clk.summary().get("sm_mhz")
    if wi and sm_mhz:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        ach = wi * mine / TOTAL12 / kern_avg
        peak_i = 4.0 * sms * sm_mhz * 1e6
        roof["issue"] = {"achieved_warp_instr_per_s": ach, "peak_warp_instr_per_s": peak_i, "frac": ach / peak_i,
                         "warp_instr_per_launch": wi * mine / TOTAL12, "sms": sms, "sm_mhz": sm_mhz}

    # ---- e2e through the public API (host buffers) ---------------------------
    e2e_steps = max(3, a.steps // 2)
    D.barrier()

    def e2e_call():
        if D.pg:
            return odist.exhaustive_summary_distributed(durs, DMA, SIGMA)
        return search.exhaustive_summary_durs(durs, DMA, SIGMA)

    e2e_call()
    torch.cuda.synchronize()
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        r = e2e_call()
    t_e2e = D.max(time.perf_counter() - t0)
    assert r.best == res.best and r.best_rank == res.best_rank
    e2e = {"value": TOTAL12 * e2e_steps / t_e2e, "unit": "orderings/s",
           "h2d_bytes_per_step": durs.nbytes + (48 if D.pg else 0),
           "d2h_bytes_per_step": 48 + (48 * D.world if D.pg else 0),
           "api": "search.exhaustive_summary_durs" if not D.pg else "dist.exhaustive_summary_distributed",
           "steps": e2e_steps}

    secondary = {} if a.no_secondary else run_secondary(a, D, torch, dev, sp, flush, ops, peak_ops, L)

    cpu = None
    if D.rank == 0 and D.world == 1 and not a.no_cpu:
        cpu = cpu_baseline(a.cpu_seconds)
        if secondary:
            secondary["cpu_port_c5_nvidia_decisions_per_s"] = cpu_heuristic_rate(4.0)
    if secondary and D.world == 1:
        secondary.update(run_rows(a, cpu=not a.no_cpu))

    if D.rank == 0:
        line = {
            "metric": "orderings simulated/sec", "value": value, "unit": "orderings/s", "n_gpus": D.world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": t_max / a.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(D.world, D.pg is not None),
            "result": {"best": res.best, "best_rank": res.best_rank, "best_ordering": list(res.best_ordering),
                       "worst": res.worst, "mean": res.mean, "geomean": res.geomean},
            "roofline": roof, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches_per_step * a.steps,
            "secondary": secondary,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        buf = (json.dumps(line) + "\n").encode()
        while buf:
            buf = buf[os.write(json_fd, buf):]
    if D.pg:
        D.pg.barrier()
        D.pg.destroy_process_group()


def profile_headline():
    """The committed ncu capture summary of the headline kernel (DRAM bytes
    per launch, issue / FP64-pipe utilization), if present."""
    p = os.path.join(ROOT, "profiles", "ncu_headline.json")
    try:
        with open(p) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def profile_traffic():
    return profile_headline().get("dram_bytes_per_launch")


def run_secondary(a, D, torch, dev, sp, flush, ops, peak_ops, L):
    import ctypes as C

    from paper_1806_10113_b200 import _capi, dist as odist, synth

    out = {}
    K, W = 3, 1
    sync = torch.cuda.synchronize

    # C3: one 10-task group, 10! orderings (strong over ranks)
    d3 = torch.from_numpy(synth.c3_group()).to(dev)
    o3 = torch.zeros(6, dtype=torch.float64, device=dev)
    t10 = math.factorial(10)
    g3 = [torch.zeros(6, dtype=torch.float64, device=dev) for _ in range(D.world)]
    reps = 20  # one step = 20 back-to-back searches (a single one is ~0.2 ms)

    def s3(ev=None):
        # every search is complete: its shard, then its own all_gather of the
        # 48-B summaries (N > 1), as dist.exhaustive_summary_distributed does
        for _ in range(reps):
            _capi.check(L.osim_exhaustive_shard_dev(C.c_void_p(d3.data_ptr()), 10, 2, 0.5, D.rank, D.world, 1,
                                                    C.c_void_p(o3.data_ptr()), sp))
            if D.pg:
                D.pg.all_gather(g3, o3)
        if ev is not None:
            ev.record()

    t, tk = timed_steps(s3, K, W, flush, sync)
    t = D.max(t)
    parts3 = [odist.unpack(g.cpu().numpy()) for g in g3] if D.pg else [odist.unpack(o3.cpu().numpy())]
    c3 = odist.combine(parts3)
    assert c3["count"] == t10 and c3["best_rank"] == 381558, c3  # SURVEY appendix C3 golden
    out["c3_orderings_per_s"] = {"value": t10 * reps * K / t, "unit": "orderings/s",
                                 "workload": "C3: K20 seed 10, 10 tasks, 10! orderings x20 per step, one "
                                             "all_gather per search at N > 1",
                                 "latency_us_per_search": t / (reps * K) * 1e6,
                                 "frac_fp64": ops["c3"]["ops"] * odist.unpack(o3.cpu().numpy())["count"] * reps * K
                                 / tk / 1e12 / peak_ops}

    # C4 variants: sigma 0.375 (true-divide path) and 1-DMA
    d4v = torch.from_numpy(synth.c4_group()).to(dev)
    o4v = torch.zeros(6, dtype=torch.float64, device=dev)
    lo4, hi4 = odist.shard(TOTAL12, D.rank, D.world)
    for name, dma_v, sig_v, opkey in (("c4_sigma0.375_orderings_per_s", 2, 0.375, "c4_sigma0.375"),
                                      ("c4_1dma_orderings_per_s", 1, 1.0, None)):
        def s4(ev=None, dma_v=dma_v, sig_v=sig_v):
            _capi.check(L.osim_exhaustive_dev(C.c_void_p(d4v.data_ptr()), 12, dma_v, sig_v, lo4, hi4, 1,
                                              C.c_void_p(o4v.data_ptr()), None, sp))
            if ev is not None:
                ev.record()

        t, tk = timed_steps(s4, K, W, flush, sync)
        t = D.max(t)
        out[name] = {"value": TOTAL12 * K / t, "unit": "orderings/s",
                     "workload": f"C4 group, {dma_v}-DMA sigma {sig_v}, all 12! orderings"}
        if opkey:
            out[name]["frac_fp64"] = ops[opkey]["ops"] * (hi4 - lo4) * K / tk / 1e12 / peak_ops

    # row f2 on the headline space: exact median + percentile count of all 12!
    # makespans kept in HBM (single GPU; multi-rank uses dist.exhaustive_stats_distributed)
    if D.world == 1:
        d4 = synth.c4_group()
        _capi.exhaustive_stats(d4, 2, 0.5, 0, TOTAL12, threshold=60.0)  # warm-up (allocates 3.8 GB)
        torch.cuda.synchronize()
        tw = float("inf")
        for _ in range(3):  # host wall clock of single calls: the best of three
            t0 = time.perf_counter()
            st4, below4, med4 = _capi.exhaustive_stats(d4, 2, 0.5, 0, TOTAL12, threshold=60.0)
            tw = min(tw, time.perf_counter() - t0)
        out["c4_full_stats"] = {"value": TOTAL12 / tw, "unit": "orderings/s", "seconds": tw,
                                "workload": "C4 12! with exact median (radix selection over 3.8 GB of makespans "
                                            "in HBM) and count below 60 ms, host API wall clock",
                                "median": med4, "below_60ms": below4}

    # C2: 100k x 8-task groups, 8! each (group-range shards, no collective)
    B2 = 100_000
    lo2, hi2 = odist.shard(B2, D.rank, D.world)
    d2 = torch.from_numpy(synth.c2_batch(B2)[lo2:hi2].copy()).to(dev)
    o2 = torch.zeros((hi2 - lo2) * 6, dtype=torch.float64, device=dev)

    def s2(ev=None):
        _capi.check(L.osim_exhaustive_batch_dev(C.c_void_p(d2.data_ptr()), hi2 - lo2, 8, 2, 0.5, 1,
                                                C.c_void_p(o2.data_ptr()), sp))
        if ev is not None:
            ev.record()

    t, tk = timed_steps(s2, K, W, flush, sync)
    t = D.max(t)
    # the credited device-resident output equals the host API's on the same groups
    assert o2.cpu().numpy().tobytes() == _capi.exhaustive_batch(synth.c2_batch(B2)[lo2:hi2], 2, 0.5).tobytes()
    out["c2_orderings_per_s"] = {"value": B2 * 40320 * K / t, "unit": "orderings/s",
                                 "workload": "C2: 100000 x 8-task TGs (Table-2 x U(0.5,1.5)), 8! each, 2-DMA 0.5",
                                 "frac_fp64": ops["c2"]["ops"] * (hi2 - lo2) * 40320 * K / tk / 1e12 / peak_ops}
    del d2, o2

    # C5: 10^6 x 16-task groups through the heuristic, three device profiles
    B5 = 1_000_000
    lo5, hi5 = odist.shard(B5, D.rank, D.world)
    m = hi5 - lo5
    for prof, (_, dma, sigma) in synth.PROFILES.items():
        dh, rh = synth.c5_batch_fast(prof, B5)
        dd = torch.from_numpy(dh[lo5:hi5].copy()).to(dev)
        rr = torch.from_numpy(rh[lo5:hi5].copy()).to(dev)
        oo = torch.empty((m, 16), dtype=torch.uint8, device=dev)
        mm = torch.empty(m, dtype=torch.float64, device=dev)
        ns = torch.empty(m, dtype=torch.int32, device=dev)

        def s5(ev=None):
            _capi.check(L.osim_heuristic_batch_dev(C.c_void_p(dd.data_ptr()), C.c_void_p(rr.data_ptr()), m, 16,
                                                   dma, sigma, 1 if sys.version_info >= (3, 12) else 0, 1,
                                                   C.c_void_p(oo.data_ptr()), C.c_void_p(mm.data_ptr()),
                                                   C.c_void_p(ns.data_ptr()), sp))
            if ev is not None:
                ev.record()

        t, tk = timed_steps(s5, K, W, flush, sync)
        t = D.max(t)
        # the credited device-resident output equals the host API's on the same groups
        ho, hm, hn = _capi.heuristic_batch(dh[lo5:hi5], rh[lo5:hi5], dma, sigma,
                                           1 if sys.version_info >= (3, 12) else 0)
        assert np.array_equal(oo.cpu().numpy(), ho) and mm.cpu().numpy().tobytes() == hm.tobytes()
        assert np.array_equal(ns.cpu().numpy().view(np.uint32), hn)
        out[f"c5_{prof}_decisions_per_s"] = {
            "value": B5 * K / t, "unit": "TG decisions/s",
            "workload": f"C5: 10^6 x 16-task TGs, {prof}-style ({dma}-DMA, sigma {sigma}), reorder_batch",
            "frac_fp64": ops[f"c5_{prof}"]["ops"] * m * K / tk / 1e12 / peak_ops}
        if prof == "nvidia" and D.world == 1:
            # e2e through the public array API with host buffers (pinned)
            pd = torch.from_numpy(dh).pin_memory()
            pr = torch.from_numpy(rh).pin_memory()
            po = torch.empty((B5, 16), dtype=torch.uint8).pin_memory()
            pm = torch.empty(B5, dtype=torch.float64).pin_memory()
            pn = torch.empty(B5, dtype=torch.int32).pin_memory()
            args = (pd.numpy(), pr.numpy(), dma, sigma, 1 if sys.version_info >= (3, 12) else 0)
            _capi.heuristic_batch(*args, order=po.numpy(), makespan=pm.numpy(), n_sims=pn.numpy().view(np.uint32))
            t0 = time.perf_counter()
            for _ in range(K):
                _capi.heuristic_batch(*args, order=po.numpy(), makespan=pm.numpy(),
                                      n_sims=pn.numpy().view(np.uint32))
            te = time.perf_counter() - t0
            out["c5_nvidia_decisions_per_s"]["e2e"] = {
                "value": B5 * K / te, "unit": "TG decisions/s", "api": "_capi.heuristic_batch (pinned host buffers)",
                "h2d_bytes_per_step": dh.nbytes + rh.nbytes, "d2h_bytes_per_step": B5 * (16 + 8 + 4)}
        del dd, rr, oo, mm, ns
    return out


# ---------------------------------------------------------------- rows f1, f3, f4
def run_rows(a, cpu):
    """SURVEY 8(f) rows through the public C-ABI wrappers with host buffers
    (wall clock, best of 3 after a warm-up), each beside the CPU oracle on a
    bounded sample when `cpu` (rank 0, N = 1: the cpu_baseline leg)."""
    import ctypes as C

    from paper_1806_10113_b200 import _capi, synth

    def best(f, k=3):
        f()
        ts = []
        for _ in range(k):
            t0 = time.perf_counter()
            f()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    out = {}
    threads = os.cpu_count() or 1
    # f1: NoReorder interleavings, 4 workers x 4 tasks (16!/(4!^4) = 63,063,000)
    W, T = 4, 4
    d1 = synth.real_group("K20", W * T, 41)[1]
    tot1 = 63_063_000
    t = best(lambda: _capi.interleavings(d1, W, T, 2, 0.5, 0, tot1))
    out["f1_noreorder_interleavings_per_s"] = {
        "value": tot1 / t, "unit": "interleavings/s",
        "workload": "f1: all 63,063,000 interleavings of 4 workers x 4 in-order tasks (K20-style, 2-DMA, "
                    "sigma 0.5) -> summary; osim_interleavings host call"}
    # f3: proxy-thread scenario harness, 10^5 scenarios of 4 workers x 3 tasks
    S3, W3, T3 = 100_000, 4, 3
    d3 = np.stack([synth.real_group("K20", W3 * T3, 20_000 + s)[1] for s in range(2000)])
    d3 = np.ascontiguousarray(np.tile(d3, (S3 // 2000, 1, 1)))
    r3 = np.tile(np.argsort(np.argsort([f"w{w}.{j}" for w in range(W3) for j in range(T3)])).astype(np.uint8), (S3, 1))
    sm = 1 if sys.version_info >= (3, 12) else 0
    t = best(lambda: _capi.harness_batch(d3, r3, W3, T3, 2, 0.5, sm))
    out["f3_harness_scenarios_per_s"] = {
        "value": S3 / t, "unit": "scenarios/s",
        "workload": "f3: 10^5 proxy-thread scenarios (4 workers x 3 tasks, K20-style, 2-DMA, sigma 0.5, "
                    "Algorithm 1 per submitted group); osim_harness_batch host call"}
    # f4: micro-step tick oracle, all 8! orderings of a config-2 group at dt = 1 us
    d4 = synth.c2_batch(1)[0]
    t = best(lambda: _capi.micro(d4, 2, 0.5, 0.001, 0, 40320), 2)
    out["f4_micro_orderings_per_s"] = {
        "value": 40320 / t, "unit": "orderings/s",
        "workload": "f4: fixed-dt (1 us) tick simulation of all 8! orderings of a config-2 group "
                    "(2-DMA, sigma 0.5); osim_micro host call"}
    if cpu:
        from oracle import oracle as O

        m1 = 400_000
        t0 = time.perf_counter()
        O.interleavings(d1, W, T, 2, 0.5, 0, m1, threads=threads)
        out["f1_noreorder_interleavings_per_s"]["cpu_port"] = {
            "value": m1 / (time.perf_counter() - t0), "cores": threads,
            "sample": f"interleavings [0, {m1}) through oracle_interleavings"}
        L = O.lib()
        L.oracle_harness.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]
        om, ong, osz = C.c_double(), C.c_int(), np.zeros(64, dtype=np.int32)
        m3 = 2000
        t0 = time.perf_counter()
        for s_ in range(m3):
            L.oracle_harness(d3[s_].ctypes.data_as(C.POINTER(C.c_double)),
                             r3[s_].ctypes.data_as(C.POINTER(C.c_uint8)), W3, T3, 2, 0.5, sm, C.byref(om),
                             C.byref(ong), osz.ctypes.data_as(C.POINTER(C.c_int)))
        out["f3_harness_scenarios_per_s"]["cpu_port"] = {
            "value": m3 / (time.perf_counter() - t0), "cores": 1,
            "sample": f"{m3} scenarios through oracle_harness, one thread"}
        m4 = 40
        t0 = time.perf_counter()
        for r_ in range(m4):
            O.micro(d4, O.unrank(r_ * 1000, 8), 2, 0.5, 0.001)
        out["f4_micro_orderings_per_s"]["cpu_port"] = {
            "value": m4 / (time.perf_counter() - t0), "cores": 1,
            "sample": f"{m4} orderings through oracle_micro, one thread"}
    return out


# ---------------------------------------------------------------- CPU legs
STRATA = 64  # rank windows per CPU step, evenly spaced over all of 12!


def strata(m, k=0):
    """`m` C4 ranks as STRATA equal windows starting at i * 12!/STRATA,
    shifted by step index k (every window samples a different first task)."""
    w = max(1, m // STRATA)
    base = TOTAL12 // STRATA
    return [(i * base + k * w, i * base + (k + 1) * w) for i in range(STRATA)], w * STRATA


def port_windows(d, windows, threads):
    from oracle import oracle as O

    for lo, hi in windows:
        O.exhaustive(d, DMA, SIGMA, lo, hi, threads=threads)


def cpu_rate(seconds):
    """CPU restatement (oracle/, all host threads) on C4 ranks in STRATA
    windows spread over the whole 12! space, sized to ~`seconds`."""
    from oracle import oracle as O
    from paper_1806_10113_b200 import synth

    threads = os.cpu_count() or 1
    d = synth.c4_group()
    probe = 2000 * threads
    t0 = time.perf_counter()
    O.exhaustive(d, DMA, SIGMA, 0, probe, threads=threads)
    rate = probe / (time.perf_counter() - t0)
    wins, m = strata(int(max(probe, min(TOTAL12 // 2, rate * seconds))))
    t0 = time.perf_counter()
    port_windows(d, wins, threads)
    el = time.perf_counter() - t0
    return m / el, threads, m, wins


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _py_ref_worker(ranks):
    """Unmodified reference (baseline/_ref offsim): engine.simulate of each
    ordering, the body of exhaustive_search's loop (oracle.py:132-135)."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from offsim import engine
    from offsim.cli import load_profile_arg
    from offsim.workload import sample_real_tasks

    tasks = sample_real_tasks("AMD", 12, seed=12)
    prof = load_profile_arg("2dma")
    out = []
    for r in ranks:
        avail = list(range(N12))
        perm = []
        for i in range(N12, 0, -1):  # Lehmer unrank (itertools.permutations order)
            f = math.factorial(i - 1)
            perm.append(avail.pop(r // f))
            r %= f
        out.append(engine.simulate([tasks[i] for i in perm], prof).makespan)
    return out


def python_reference_rate(seconds):
    """The unmodified Python reference (tools/install_reference.sh ->
    baseline/_ref) on C4 ranks strided over all of 12!, one process per host
    core; its makespans are checked against the oracle port on the same ranks."""
    if not os.path.isdir(os.path.join(REF_DIR, "offsim")):
        return {"unavailable": "baseline/_ref/offsim missing (run tools/install_reference.sh)"}
    import multiprocessing as mp

    from oracle import oracle as O
    from paper_1806_10113_b200 import synth

    procs = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_py_ref_worker, [[0]] * procs)  # imports and warm-up outside the timed region
        t0 = time.perf_counter()
        pool.map(_py_ref_worker, [[7 * k] for k in range(20 * procs)])
        per = (time.perf_counter() - t0) / 20  # ~ seconds per ordering per process
        m = int(max(procs * 10, min(2_000_000, procs * seconds / max(per, 1e-6))))
        stride = TOTAL12 // m
        ranks = [k * stride for k in range(m)]
        chunks = [ranks[i::procs] for i in range(procs)]
        t0 = time.perf_counter()
        res = pool.map(_py_ref_worker, chunks)
        el = time.perf_counter() - t0
    ms = np.empty(m)
    for i in range(procs):
        ms[i::procs] = res[i]
    perms = np.array([O.unrank(r, N12) for r in ranks], dtype=np.uint8)
    _, oms = O.eval_perms(synth.c4_group(), DMA, SIGMA, perms, threads=procs)
    return {"value": m / el, "unit": "orderings/s", "cores": procs, "kind": "python",
            "sample": f"{m} C4 ranks k*{stride} (strided over all of 12!) through the unmodified reference "
                      f"(baseline/_ref offsim.engine.simulate), {procs} processes",
            "bit_exact_vs_port": bool(np.array_equal(ms, oms))}


def cpu_heuristic_rate(seconds):
    """CPU port of reorder_batch (oracle/, all host threads) on config-5
    groups (NVIDIA-style profile), sized to ~`seconds`."""
    from oracle import oracle as O
    from paper_1806_10113_b200 import synth

    threads = os.cpu_count() or 1
    d, r = synth.c5_batch_fast("nvidia", 400_000, seed=77)
    probe = 16 * threads
    t0 = time.perf_counter()
    O.reorder_batch(d[:probe], r[:probe], 2, 0.5, 1, threads=threads)
    rate = probe / (time.perf_counter() - t0)
    m = int(min(len(d), max(probe, rate * seconds)))
    t0 = time.perf_counter()
    O.reorder_batch(d[:m], r[:m], 2, 0.5, 1, threads=threads)
    el = time.perf_counter() - t0
    return {"value": m / el, "unit": "TG decisions/s", "cores": threads, "kind": "port",
            "sample": f"{m} config-5 16-task groups (NVIDIA-style) through oracle/osim_oracle.c reorder"}


def cpu_baseline(seconds):
    v, threads, m, wins = cpu_rate(seconds)
    return {"value": v, "unit": "orderings/s", "cores": threads, "kind": "port",
            "sample": f"{m} C4 ranks in {len(wins)} windows of {wins[0][1] - wins[0][0]} at i*12!/{len(wins)} "
                      f"through oracle/osim_oracle.c (C restatement of engine.py/oracle.py) on {threads} threads",
            "python": python_reference_rate(min(seconds, 10.0))}


def arm_config(world, pg):
    """The workload both arms report (the reference arm times a bounded
    sample of it per step, described in its cpu_baseline.sample)."""
    return {"workload": WORKLOAD, "orderings_per_step": TOTAL12, "n_tasks": N12,
            "parallelism": f"interleaved Lehmer-rank shards x{world}" + (" + NCCL all_gather of 48-B summaries"
                                                                         if pg else ""),
            "l2": "256 MiB buffer zeroed before every timed step (excluded from timing); inputs 288 B",
            "fast_path": True}


def run_reference(a):
    if env_int("RANK", 0) != 0:
        return
    from paper_1806_10113_b200 import synth

    threads = os.cpu_count() or 1
    d = synth.c4_group()
    v, _, m, _ = cpu_rate(float(os.environ.get("OSIM_REF_STEP_SECONDS", "2.0")))  # each step ~2 s
    for k in range(a.warmup):
        port_windows(d, strata(m // 4, 1000 + k)[0], threads)
    t0 = time.perf_counter()
    for k in range(a.steps):  # step k: the STRATA windows shifted by k (distinct ranks every step)
        port_windows(d, strata(m, k)[0], threads)
    el = time.perf_counter() - t0
    value = m * a.steps / el
    sample = (f"{a.steps} steps of {m} C4 orderings, each in {STRATA} rank windows spread over all of 12! "
              f"(window i of step k at i*12!/{STRATA} + k*{m // STRATA}), through oracle/osim_oracle.c on "
              f"{threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": "orderings simulated/sec", "value": value, "unit": "orderings/s",
        "n_gpus": env_int("WORLD_SIZE", 1), "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": el / a.steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": arm_config(env_int("WORLD_SIZE", 1), env_int("WORLD_SIZE", 1) > 1),
        "cpu_baseline": {"value": value, "unit": "orderings/s", "cores": threads, "kind": "port", "sample": sample,
                         "orderings_per_step": m},
        "e2e": {"value": value, "unit": "orderings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    a = ap.parse_args()
    if a.warmup < 3:
        print("note: --warmup raised to 3 (timing rules)", file=sys.stderr)
        a.warmup = 3
    if env_int("WORLD_SIZE", 1) > 1 or os.environ.get("OSIM_BENCH_FORCE_PG") == "1":
        # NCCL's init lines (communicator size, transport) on stderr, so the
        # run log shows every rank joined one communicator; set before torch
        # (and with it NCCL) is first imported
        # (the GPU image sets NCCL_DEBUG=VERSION, which prints only the banner)
        if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION", "WARN"):
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
