"""Per-rank shard times for the multi-GPU configs, measured on ONE GPU.

For W = 1, 2, 4, 8 and every rank r < W this times, on cuda:0, exactly the
work rank r does inside bench.py's step (for C4/C3 both the contiguous
dist.shard range and the interleaved 512-prefix calls of
osim_exhaustive_shard_dev that bench.py runs; the group range for C2/C5),
each shard on its own: W warm-up
launches, then K launches bracketed by CUDA events on the launching stream,
L2 flushed (256 MiB) before every timed launch.  Shards run one after another,
never concurrently, so no kernel waits on another rank.  The predicted W-GPU
step is the slowest shard (the max over ranks bench.py takes); it leaves out
the one 48-byte NCCL all_gather of C4/C3 (the driver's N>1 bench measures
that).  Output: one JSON document (default gpurun_out/shard_speed.json).
"""
import argparse
import ctypes as C
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1806_10113_b200 import _capi, dist as odist, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/shard_speed.json")
    a = ap.parse_args()

    L = _capi.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(st)
    sp = C.c_void_p(st.cuda_stream)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sum_mode = 1 if sys.version_info >= (3, 12) else 0

    def time_launch(fn):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(a.steps):
            flush_buf.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / a.steps / 1e3  # seconds per launch

    res = {"gpu": torch.cuda.get_device_name(dev), "steps": a.steps, "warmup": a.warmup, "configs": {}}

    # C4 / C3: Lehmer-rank shards of one group
    for name, n, durs in (("C4", 12, synth.c4_group()), ("C3", 10, synth.c3_group())):
        d = torch.from_numpy(durs).to(dev)
        o = torch.zeros(6, dtype=torch.float64, device=dev)
        fast = int(_capi.fast_eligible(durs, 0.5))
        total = math.factorial(n)
        rows = {}
        for W in (1, 2, 4, 8):
            ts = []
            for r in range(W):
                lo, hi = odist.shard(total, r, W)
                ts.append(time_launch(lambda lo=lo, hi=hi: _capi.check(L.osim_exhaustive_dev(
                    C.c_void_p(d.data_ptr()), n, 2, 0.5, lo, hi, fast, C.c_void_p(o.data_ptr()), None, sp))))
            rows[W] = {"shard_ms": [t * 1e3 for t in ts], "step_ms": max(ts) * 1e3,
                       "orderings_per_s": total / max(ts)}
        for W in rows:
            rows[W]["efficiency_vs_1"] = rows[1]["step_ms"] / (W * rows[W]["step_ms"])
        res["configs"][name + "_contiguous"] = {"unit": "orderings/s", "total": total, "by_world": rows}
        rows = {}
        for W in (1, 2, 4, 8):  # interleaved 512-prefix calls (osim_exhaustive_shard_dev, what bench.py runs)
            ts = []
            for r in range(W):
                ts.append(time_launch(lambda r=r, W=W: _capi.check(L.osim_exhaustive_shard_dev(
                    C.c_void_p(d.data_ptr()), n, 2, 0.5, r, W, fast, C.c_void_p(o.data_ptr()), sp))))
            rows[W] = {"shard_ms": [t * 1e3 for t in ts], "step_ms": max(ts) * 1e3,
                       "orderings_per_s": total / max(ts)}
        for W in rows:
            rows[W]["efficiency_vs_1"] = rows[1]["step_ms"] / (W * rows[W]["step_ms"])
        res["configs"][name + "_interleaved"] = {"unit": "orderings/s", "total": total, "by_world": rows}

    # C2: 10^5 x 8-task groups, group-range shards
    B2 = 100_000
    full2 = synth.c2_batch(B2)
    rows = {}
    for W in (1, 2, 4, 8):
        ts = []
        for r in range(W):
            lo, hi = odist.shard(B2, r, W)
            d2 = torch.from_numpy(full2[lo:hi].copy()).to(dev)
            o2 = torch.zeros((hi - lo) * 6, dtype=torch.float64, device=dev)
            ts.append(time_launch(lambda d2=d2, o2=o2, m=hi - lo: _capi.check(L.osim_exhaustive_batch_dev(
                C.c_void_p(d2.data_ptr()), m, 8, 2, 0.5, 1, C.c_void_p(o2.data_ptr()), sp))))
            del d2, o2
        rows[W] = {"shard_ms": [t * 1e3 for t in ts], "step_ms": max(ts) * 1e3,
                   "orderings_per_s": B2 * 40320 / max(ts)}
    for W in rows:
        rows[W]["efficiency_vs_1"] = rows[1]["step_ms"] / (W * rows[W]["step_ms"])
    res["configs"]["C2"] = {"unit": "orderings/s", "total_groups": B2, "by_world": rows}
    del full2

    # C5: 10^6 x 16-task heuristic, NVIDIA-style profile, group-range shards
    B5 = 1_000_000
    _, dma, sigma = synth.PROFILES["nvidia"]
    dh, rh = synth.c5_batch_fast("nvidia", B5)
    rows = {}
    for W in (1, 2, 4, 8):
        ts = []
        for r in range(W):
            lo, hi = odist.shard(B5, r, W)
            m = hi - lo
            dd = torch.from_numpy(dh[lo:hi].copy()).to(dev)
            rr = torch.from_numpy(rh[lo:hi].copy()).to(dev)
            oo = torch.empty((m, 16), dtype=torch.uint8, device=dev)
            mm = torch.empty(m, dtype=torch.float64, device=dev)
            ns = torch.empty(m, dtype=torch.int32, device=dev)
            ts.append(time_launch(lambda dd=dd, rr=rr, oo=oo, mm=mm, ns=ns, m=m: _capi.check(
                L.osim_heuristic_batch_dev(C.c_void_p(dd.data_ptr()), C.c_void_p(rr.data_ptr()), m, 16, dma, sigma,
                                           sum_mode, 1, C.c_void_p(oo.data_ptr()), C.c_void_p(mm.data_ptr()),
                                           C.c_void_p(ns.data_ptr()), sp))))
            del dd, rr, oo, mm, ns
        rows[W] = {"shard_ms": [t * 1e3 for t in ts], "step_ms": max(ts) * 1e3, "decisions_per_s": B5 / max(ts)}
    for W in rows:
        rows[W]["efficiency_vs_1"] = rows[1]["step_ms"] / (W * rows[W]["step_ms"])
    res["configs"]["C5_nvidia"] = {"unit": "TG decisions/s", "total_groups": B5, "by_world": rows}

    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1)
    for k, v in res["configs"].items():
        print(k, {W: (round(r["step_ms"], 3), round(r["efficiency_vs_1"], 3)) for W, r in v["by_world"].items()})


if __name__ == "__main__":
    main()
