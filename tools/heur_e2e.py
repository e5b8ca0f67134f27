"""C5 end-to-end rate through the host API with pinned buffers (the bench's
e2e leg), for chunk counts in $OSIM_HCHUNKS (run once per value)."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one():
    import numpy as np
    import torch

    from paper_1806_10113_b200 import _capi, synth
    B = 1_000_000
    dh, rh = synth.c5_batch_fast("nvidia", B)
    pd, pr = torch.from_numpy(dh).pin_memory(), torch.from_numpy(rh).pin_memory()
    po = torch.empty((B, 16), dtype=torch.uint8).pin_memory()
    pm = torch.empty(B, dtype=torch.float64).pin_memory()
    pn = torch.empty(B, dtype=torch.int32).pin_memory()
    args = (pd.numpy(), pr.numpy(), 2, 0.5, 1)
    kw = dict(order=po.numpy(), makespan=pm.numpy(), n_sims=pn.numpy().view(np.uint32))
    _capi.heuristic_batch(*args, **kw)
    t = time.perf_counter()
    for _ in range(5):
        _capi.heuristic_batch(*args, **kw)
    print(os.environ.get("OSIM_HCHUNKS", "default"), f"{5 * B / (time.perf_counter() - t) / 1e6:.1f} M decisions/s e2e",
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        for k in (sys.argv[1:] or ["4", "8", "16", "32"]):
            subprocess.run([sys.executable, __file__, "one"], env={**os.environ, "OSIM_HCHUNKS": k}, check=True)
