import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1806_10113_b200 import _capi, synth
d = synth.c4_group().copy()
d[3, 0] = 0.0  # one null HtD -> general path
assert not _capi.fast_eligible(d, 0.5)
total = 479001600
for lo, hi in ((0, 20_000_000),):
    _capi.exhaustive(d, 2, 0.5, lo, lo + 1_000_000)
    t = time.perf_counter(); _capi.exhaustive(d, 2, 0.5, lo, hi); dt = time.perf_counter() - t
    print(f"general path C4 with a null stage: {(hi-lo)/dt/1e9:.2f} G orderings/s")
d2 = synth.c4_group() * 1e23  # out of fast range
t = time.perf_counter(); _capi.exhaustive(d2, 2, 0.5, 0, 20_000_000); dt = time.perf_counter() - t
print(f"general path C4 scaled 1e23: {20e6/dt/1e9:.2f} G orderings/s")
