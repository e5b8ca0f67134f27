"""Device-resident C5 heuristic rate (osim_heuristic_batch_dev, CUDA events)
for the three device profiles; tuning aid."""
import ctypes as C
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
    B = 1_000_000
    null = "--null" in sys.argv  # one null DtH per group: the NullSim checkpoint kernel
    for prof in ("nvidia", "amd", "phi"):
        _, dma, sigma = synth.PROFILES[prof]
        d, r = synth.c5_batch_fast(prof, B)
        if null:
            d[:, 5, 2] = 0.0
        dd, rr = torch.from_numpy(d).to(dev), torch.from_numpy(r).to(dev)
        oo = torch.empty((B, 16), dtype=torch.uint8, device=dev)
        mm = torch.empty(B, dtype=torch.float64, device=dev)
        ns = torch.empty(B, dtype=torch.int32, device=dev)

        def run():
            _capi.check(L.osim_heuristic_batch_dev(C.c_void_p(dd.data_ptr()), C.c_void_p(rr.data_ptr()), B, 16, dma,
                                                   sigma, 1, 2 if null else 1, C.c_void_p(oo.data_ptr()),
                                                   C.c_void_p(mm.data_ptr()),
                                                   C.c_void_p(ns.data_ptr()), C.c_void_p(st.cuda_stream)))
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        print(f"{prof}{' (null stages)' if null else ''}: {5 * B / (e0.elapsed_time(e1) / 1e3) / 1e6:.1f} M decisions/s", flush=True)


if __name__ == "__main__":
    main()
