"""Algorithmic FP64 op counts per unit for the roofline.

ops per ordering = S + 8R + 2O with S = steps, R = running-command-steps,
O = running transfer-steps at rate sigma != 1 (DDIV counted as one op,
x/1.0 and x*1.0 excluded).  Counted with the pinned CPU oracle's
instrumentation; deterministic per input.  Writes tests/golden/op_counts.json,
which bench.py reads (it never runs the oracle for this).

    python tests/golden/make_opcounts.py
"""

import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1806_10113_b200 import synth  # noqa: E402


def per_unit(S, R, Ov, units):
    return {"S": S / units, "R": R / units, "O": Ov / units, "ops": (S + 8 * R + 2 * Ov) / units,
            "units_counted": int(units)}


def main():
    out = {"formula": "S + 8R + 2O FP64 ops per unit (SURVEY.md 8(d))"}
    t12 = math.factorial(12)
    for sig in (0.5, 0.375):
        stride = t12 // 400_000
        s = O.op_stats(synth.c4_group(), 2, sig, 0, t12, stride)
        out[f"c4_sigma{sig}"] = {**per_unit(*s, len(range(0, t12, stride))), "sampling": f"every {stride}th rank"}
    s = O.op_stats(synth.c3_group(), 2, 0.5, 0, math.factorial(10), 1)
    out["c3"] = {**per_unit(*s, math.factorial(10)), "sampling": "exact, all 10! orderings"}
    d = synth.c2_batch(64)
    acc = np.zeros(3, dtype=np.int64)
    for b in range(64):
        acc += O.op_stats(d[b], 2, 0.5, 0, 40320, 1)
    out["c2"] = {**per_unit(*acc, 64 * 40320), "sampling": "exact over TGs 0..63"}
    for prof, (dev, dma, sigma) in synth.PROFILES.items():
        dd, rr = synth.c5_batch(prof, 400)
        acc = np.zeros(4, dtype=np.int64)
        for b in range(400):
            acc += O.reorder_op_stats(dd[b], rr[b], dma, sigma, 1)
        out[f"c5_{prof}"] = {**per_unit(*acc[:3], 400), "sims_per_decision": acc[3] / 400,
                             "sampling": "TGs 0..399 (per decision incl. the final evaluation)"}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "op_counts.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
