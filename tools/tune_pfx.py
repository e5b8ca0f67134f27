"""Time the exhaustive kernels for the suffix length in $OSIM_PFX_L.

    OSIM_PFX_L=4 python tools/tune_pfx.py
"""
import ctypes as C
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main():
    _capi.set_device(0)
    L = _capi.load()
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    sp = C.c_void_p(st.cuda_stream)
    out = torch.zeros(6, dtype=torch.float64, device="cuda")
    res = {"L": os.environ.get("OSIM_PFX_L", "default")}
    for name, d, n, sig in (("c4", synth.c4_group(), 12, 0.5), ("c4s375", synth.c4_group(), 12, 0.375),
                            ("c3", synth.c3_group(), 10, 0.5)):
        dd = torch.from_numpy(d).cuda()
        tot = math.factorial(n)
        t = timeit(lambda: _capi.check(L.osim_exhaustive_dev(C.c_void_p(dd.data_ptr()), n, 2, sig, 0, tot, 1,
                                                             C.c_void_p(out.data_ptr()), None, sp)))
        res[name] = tot / t
    d2 = torch.from_numpy(synth.c2_batch(100_000)).cuda()
    o2 = torch.zeros(100_000 * 6, dtype=torch.float64, device="cuda")
    t = timeit(lambda: _capi.check(L.osim_exhaustive_batch_dev(C.c_void_p(d2.data_ptr()), 100_000, 8, 2, 0.5, 1,
                                                               C.c_void_p(o2.data_ptr()), sp)), reps=2)
    res["c2"] = 100_000 * 40320 / t
    for prof in ("nvidia", "amd", "phi"):
        _, dma, sigma = synth.PROFILES[prof]
        dh, rh = synth.c5_batch_fast(prof, 200_000)
        dd, rr = torch.from_numpy(dh).cuda(), torch.from_numpy(rh).cuda()
        oo = torch.empty((200_000, 16), dtype=torch.uint8, device="cuda")
        mm = torch.empty(200_000, dtype=torch.float64, device="cuda")
        t = timeit(lambda: _capi.check(L.osim_heuristic_batch_dev(
            C.c_void_p(dd.data_ptr()), C.c_void_p(rr.data_ptr()), 200_000, 16, dma, sigma, 1, 1,
            C.c_void_p(oo.data_ptr()), C.c_void_p(mm.data_ptr()), None, sp)), reps=2)
        res["c5_" + prof] = 200_000 / t
    print(json.dumps({k: (f"{v:.4g}" if isinstance(v, float) else v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
