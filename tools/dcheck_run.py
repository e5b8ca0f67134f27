"""The kernels with their device-side bounds / invariant checks compiled in
(OSIM_DEBUG_CHECKS, see osim_sim.cuh; compute-sanitizer is closed on the GPU
pool).  Builds nothing: run on the GPU box with the checking build,

    python -m paper_1806_10113_b200._build --variant dcheck -DOSIM_DEBUG_CHECKS   (here)
    OSIM_LIB=$PWD/paper_1806_10113_b200/liboffsim_b200_dcheck.so python tools/dcheck_run.py

It runs tools/sanitize_run.py (every kernel family, oracle-checked) and the
race-sensitive prefix kernel over whole spaces at several residencies
(OSIM_CTAS_PER_SM = 1..4 change which CTAs share an SM and how the
barrier-free phase overlap interleaves); every run must be bit-identical."""
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    from paper_1806_10113_b200 import _capi, dist as odist, synth

    _capi.set_device(0)
    out = {}
    for name, d, n in (("c3", synth.c3_group(), 10), ("c4", synth.c4_group(), 12)):
        s, _ = _capi.exhaustive(d, 2, 0.5, 0, math.factorial(n))
        out[name] = odist.pack(s).tobytes().hex()
        out[name + "_375"] = odist.pack(_capi.exhaustive(d, 2, 0.375, 0, math.factorial(n))[0]).tobytes().hex()
        out[name + "_shards"] = [odist.pack(_capi.exhaustive_shard(d, 2, 0.5, r, 8)).tobytes().hex() for r in range(8)]
    st, below, med = _capi.exhaustive_stats(synth.c3_group(), 2, 0.5, 0, math.factorial(10), threshold=69.0)
    out["c3_stats"] = [odist.pack(st).tobytes().hex(), below, med.hex()]
    d5, r5 = synth.c5_batch_fast("nvidia", 20_000)
    o, m, _ = _capi.heuristic_batch(d5, r5, 2, 0.5, 1)
    out["c5"] = [o.tobytes().hex()[:64], m.tobytes().hex()[:64], __import__("hashlib").sha256(o.tobytes() + m.tobytes()).hexdigest()]
    print(json.dumps(out))


def main():
    lib = os.environ.get("OSIM_LIB", "")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], capture_output=True, text=True)
    print("sanitize_run under", lib or "default build", "rc", r.returncode, r.stdout.strip()[-200:], r.stderr[-2000:])
    assert r.returncode == 0
    runs = {}
    for k in ("1", "2", "3", "4"):
        env = dict(os.environ, OSIM_CTAS_PER_SM=k)
        p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        assert p.returncode == 0, p.stderr[-3000:]
        runs[k] = json.loads(p.stdout.strip().splitlines()[-1])
        print("ctas/sm", k, "ok")
    ref = runs["4"]
    same = all(runs[k] == ref for k in runs)
    print(json.dumps({"lib": lib, "identical_across_residencies": same, "c4": ref["c4"], "c3_stats": ref["c3_stats"]}))
    assert same


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
    else:
        main()
