"""Exactly bench.py's timed C5 launch (osim_heuristic_batch_dev, B = 10^6
16-task groups, one device profile), once after one warm-up launch, for an
ncu capture of the credited kernel:

    ncu --set full -k regex:k_heuristic -s 1 -c 1 python tools/c5_launch.py nvidia
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1806_10113_b200 import _capi, synth  # noqa: E402


def main(prof="nvidia", B=1_000_000, reps=2):
    _capi.set_device(0)
    L = _capi.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(st)
    _, dma, sigma = synth.PROFILES[prof]
    d, r = synth.c5_batch_fast(prof, B)
    dd, rr = torch.from_numpy(d).to(dev), torch.from_numpy(r).to(dev)
    oo = torch.empty((B, 16), dtype=torch.uint8, device=dev)
    mm = torch.empty(B, dtype=torch.float64, device=dev)
    ns = torch.empty(B, dtype=torch.int32, device=dev)
    sm = 1 if sys.version_info >= (3, 12) else 0
    for _ in range(reps):
        _capi.check(L.osim_heuristic_batch_dev(C.c_void_p(dd.data_ptr()), C.c_void_p(rr.data_ptr()), B, 16, dma,
                                               sigma, sm, 1, C.c_void_p(oo.data_ptr()), C.c_void_p(mm.data_ptr()),
                                               C.c_void_p(ns.data_ptr()), C.c_void_p(st.cuda_stream)))
    torch.cuda.synchronize()
    print(prof, "order[0]", oo[0].tolist(), "makespan[0]", float(mm[0]), "n_sims[0]", int(ns[0]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "nvidia")
