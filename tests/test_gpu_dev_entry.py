"""The device-resident entry points that produce bench.py's credited rates
(osim_exhaustive_shard_dev for C4/C3, osim_exhaustive_batch_dev for C2,
osim_heuristic_batch_dev for C5) against the host API on the bench's own
inputs: byte-identical outputs (oracle.py:111-136, heuristic.py:105-125)."""

import ctypes as C
import math
import sys

import numpy as np
import pytest

from paper_1806_10113_b200 import _capi, dist as odist, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    _capi.set_device(0)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(device=dev)
    return torch, dev, st, _capi.load()


def _shard_dev(env, durs, n, dma, sigma, shard, shards, fast):
    torch, dev, st, L = env
    dd = torch.from_numpy(durs).to(dev)
    out = torch.zeros(6, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    _capi.check(L.osim_exhaustive_shard_dev(C.c_void_p(dd.data_ptr()), n, dma, sigma, shard, shards, fast,
                                            C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)))
    st.synchronize()
    return odist.unpack(out.cpu().numpy())


@pytest.mark.parametrize("W", range(1, 9))
def test_c4_shard_dev_equals_host_api(env, W):
    # the bench's headline launch at every world size: each rank's
    # device-resident shard equals the host API's shard byte for byte, and the
    # combined shards equal the whole-space host search (best / argmin /
    # worst / count exact; the sums within 1e-12: partition-dependent order)
    d = synth.c4_group()
    fast = int(_capi.fast_eligible(d, 0.5))
    assert fast == 1
    parts = []
    for r in range(W):
        dv = _shard_dev(env, d, 12, 2, 0.5, r, W, fast)
        host = _capi.exhaustive_shard(d, 2, 0.5, r, W)
        assert odist.pack(dv).tobytes() == odist.pack(host).tobytes()
        parts.append(dv)
    whole, _ = _capi.exhaustive(d, 2, 0.5, 0, math.factorial(12))
    comb = odist.combine(parts)
    for k in ("best", "best_rank", "worst", "count"):
        assert comb[k] == whole[k]
    for k in ("sum", "sum_log"):
        assert abs(comb[k] - whole[k]) <= 1e-12 * abs(whole[k])


def test_c3_shard_dev_equals_host_api(env):
    d = synth.c3_group()
    for W in (1, 2, 8):
        for r in range(W):
            dv = _shard_dev(env, d, 10, 2, 0.5, r, W, 1)
            assert odist.pack(dv).tobytes() == odist.pack(_capi.exhaustive_shard(d, 2, 0.5, r, W)).tobytes()


def test_c2_batch_dev_equals_host_api(env):
    torch, dev, st, L = env
    B = 100_000
    d = synth.c2_batch(B)
    dd = torch.from_numpy(d).to(dev)
    o = torch.zeros(B * 6, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    _capi.check(L.osim_exhaustive_batch_dev(C.c_void_p(dd.data_ptr()), B, 8, 2, 0.5, 1, C.c_void_p(o.data_ptr()),
                                            C.c_void_p(st.cuda_stream)))
    st.synchronize()
    host = _capi.exhaustive_batch(d, 2, 0.5)
    assert o.cpu().numpy().tobytes() == host.tobytes()


@pytest.mark.parametrize("prof", ["nvidia", "amd", "phi"])
def test_c5_heuristic_dev_equals_host_api(env, prof):
    torch, dev, st, L = env
    B = 1_000_000
    _, dma, sigma = synth.PROFILES[prof]
    dh, rh = synth.c5_batch_fast(prof, B)
    dd, rr = torch.from_numpy(dh).to(dev), torch.from_numpy(rh).to(dev)
    oo = torch.empty((B, 16), dtype=torch.uint8, device=dev)
    mm = torch.empty(B, dtype=torch.float64, device=dev)
    ns = torch.empty(B, dtype=torch.int32, device=dev)
    sm = 1 if sys.version_info >= (3, 12) else 0
    torch.cuda.synchronize()
    _capi.check(L.osim_heuristic_batch_dev(C.c_void_p(dd.data_ptr()), C.c_void_p(rr.data_ptr()), B, 16, dma, sigma,
                                           sm, 1, C.c_void_p(oo.data_ptr()), C.c_void_p(mm.data_ptr()),
                                           C.c_void_p(ns.data_ptr()), C.c_void_p(st.cuda_stream)))
    st.synchronize()
    o, m, n = _capi.heuristic_batch(dh, rh, dma, sigma, sm)
    assert np.array_equal(oo.cpu().numpy(), o)
    assert mm.cpu().numpy().tobytes() == m.tobytes()
    assert np.array_equal(ns.cpu().numpy().view(np.uint32), n)
    assert set(np.unique(n).tolist()) == {16 * 15 // 2 - 1}
