"""Device-resident exhaustive rates (C4 sigma 0.5 / 0.375 / 1-DMA, C3, C2) of
the library at OSIM_LIB (A/B of tuning builds); CUDA events, L2 flushed."""
import ctypes as C
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def main():
    _capi.set_device(0)
    L = _capi.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(st)
    sp = C.c_void_p(st.cuda_stream)
    fl = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = torch.zeros(6, dtype=torch.float64, device=dev)
    res = {}

    def timed(fn, k=5):
        fn()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(k):
            fl.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1) / 1e3
        return tot / k

    for name, d, n, dma, sg in (("c4", synth.c4_group(), 12, 2, 0.5), ("c4_375", synth.c4_group(), 12, 2, 0.375),
                                ("c4_1dma", synth.c4_group(), 12, 1, 1.0), ("c3", synth.c3_group(), 10, 2, 0.5)):
        dd = torch.from_numpy(d).to(dev)
        tot = math.factorial(n)
        t = timed(lambda: _capi.check(L.osim_exhaustive_dev(C.c_void_p(dd.data_ptr()), n, dma, sg, 0, tot, 1,
                                                            C.c_void_p(out.data_ptr()), None, sp)))
        res[name] = tot / t / 1e9
    B = 100_000
    d2 = torch.from_numpy(synth.c2_batch(B)).to(dev)
    o2 = torch.zeros(B * 6, dtype=torch.float64, device=dev)
    t = timed(lambda: _capi.check(L.osim_exhaustive_batch_dev(C.c_void_p(d2.data_ptr()), B, 8, 2, 0.5, 1,
                                                             C.c_void_p(o2.data_ptr()), sp)), 3)
    res["c2"] = B * 40320 / t / 1e9
    print(json.dumps({k: round(v, 3) for k, v in res.items()}))


if __name__ == "__main__":
    main()
