"""Loading helpers for the reference-generated fixtures in tests/golden/."""

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F = float.fromhex


@functools.lru_cache(maxsize=None)
def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def durs(rows):
    return np.array([[F(x) for x in r] for r in rows], dtype=np.float64)


def fl(xs):
    return [F(x) for x in xs]


def sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b))
