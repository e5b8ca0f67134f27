"""A/B of the heuristic kernels (k_heuristic_fast / k_heuristic_nullck vs
k_heuristic_lane / k_heuristic_null_lane, OSIM_HEUR_LANE=0/1; AB_NULL=1: one
null DtH per group, the null-stage kernels): device-resident rate on the C5 batch
(10^6 x 16 tasks, three device profiles) and a hash of the outputs, which
must be identical.

    python tools/heur_ab.py            (both, in subprocesses)
"""
import ctypes as C
import hashlib
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child():
    import torch

    from paper_1806_10113_b200 import _capi, synth

    _capi.set_device(0)
    L = _capi.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(st)
    B = int(os.environ.get("AB_B", 1_000_000))
    out = {}
    for prof in ("nvidia", "amd", "phi"):
        _, dma, sigma = synth.PROFILES[prof]
        d, r = synth.c5_batch_fast(prof, B)
        if os.environ.get("AB_NULL") == "1":  # one null DtH per group: the null-stage kernels
            d[:, 5, 2] = 0.0
        dd, rr = torch.from_numpy(d).to(dev), torch.from_numpy(r).to(dev)
        oo = torch.empty((B, 16), dtype=torch.uint8, device=dev)
        mm = torch.empty(B, dtype=torch.float64, device=dev)
        ns = torch.empty(B, dtype=torch.int32, device=dev)

        def run():
            mode = 2 if os.environ.get("AB_NULL") == "1" else 1
            _capi.check(L.osim_heuristic_batch_dev(C.c_void_p(dd.data_ptr()), C.c_void_p(rr.data_ptr()), B, 16, dma,
                                                   sigma, 1, mode, C.c_void_p(oo.data_ptr()), C.c_void_p(mm.data_ptr()),
                                                   C.c_void_p(ns.data_ptr()), C.c_void_p(st.cuda_stream)))
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        h = hashlib.sha256(oo.cpu().numpy().tobytes() + mm.cpu().numpy().tobytes() + ns.cpu().numpy().tobytes())
        out[prof] = {"M_decisions_per_s": 5 * B / (e0.elapsed_time(e1) / 1e3) / 1e6, "sha": h.hexdigest()[:16]}
    print(json.dumps(out))


def main():
    res = {}
    for v in sys.argv[1:] or ["0", "1"]:
        env = dict(os.environ, OSIM_HEUR_LANE=v)
        p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        if p.returncode:
            print(p.stderr[-3000:])
            sys.exit(1)
        res[v] = json.loads(p.stdout.strip().splitlines()[-1])
        print("OSIM_HEUR_LANE", v, res[v], flush=True)
    if len(res) > 1:
        a, b = list(res.values())[:2]
        print("identical outputs:", all(a[p]["sha"] == b[p]["sha"] for p in a))


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
    else:
        main()
