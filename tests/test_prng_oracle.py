"""PRNG sampler variants (north_star pcg32 / sfc64 / xoshiro256pp): the
oracle's generators against public known answers, and the native host
forms against the oracle.  The variants are not in the reference, so the
sampler semantics are this repo's definition."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import prng_oracle as po


def test_pcg32_published_vector():
    g = po.Pcg32(42, 54)  # pcg32-demo: pcg32_srandom_r(&rng, 42u, 54u)
    assert [g.next32() for _ in range(6)] == [0xa15c02b7, 0x7b47f409, 0xba1d3330, 0x83d2f293,
                                              0xbfa4784b, 0xcbed606e]


def test_sfc64_step_matches_numpy():
    g = po.Sfc64(0x1234, 0x5678)
    bg = np.random.SFC64(0)
    st = bg.state
    st["state"]["state"] = np.array([g.a, g.b, g.c, g.w], dtype=np.uint64)
    st["has_uint32"] = 0
    bg.state = st
    assert [g.next64() for _ in range(16)] == [int(x) for x in bg.random_raw(16)]


def test_xoshiro256pp_definition():
    g = po.Xoshiro256pp(0, 0, state=[1, 2, 3, 4])
    assert g.next64() == (5 << 23) + 1
    s0, s3 = 7, 6 << 45  # state after one step, from the recurrence
    assert g.next64() == (po._rotl(s0 + s3, 23) + s0) & po.M64


@pytest.mark.parametrize("kind", ["pcg32", "sfc64", "xoshiro256pp"])
def test_native_streams_and_floyd_match_oracle(kind):
    from paper_2505_10806_b200 import _lib

    code = _lib.PRNG_KINDS[kind]
    out = np.zeros(40, dtype=np.uint64)
    _lib.host_call("rg_prng_raw", code, 0xDEADBEEF, 0x12345, 40, out.ctypes.data)
    g = po.KINDS[kind](0xDEADBEEF, 0x12345)
    want = [g.next32() if kind == "pcg32" else g.next64() for _ in range(40)]
    assert out.tolist() == want
    rng = np.random.default_rng(3)
    for _ in range(50):
        D = int(rng.integers(1, 5000))
        T = int(rng.integers(0, min(D, 40) + 1))
        nk, sd = (int(x) for x in rng.integers(0, 2**63, size=2))
        pos = np.zeros(max(T, 1), dtype=np.int32)
        _lib.host_call("rg_prng_select", code, nk, sd, D, T, pos.ctypes.data)
        want = po.floyd(po.KINDS[kind](nk, sd), D, T)
        assert pos[:T].tolist() == want
        assert len(set(want)) == T and all(0 <= p < D for p in want)


def test_floyd_is_uniform_subset():
    from scipy import stats

    counts = np.zeros(20, dtype=np.int64)
    for s in range(4000):
        for p in po.floyd(po.Xoshiro256pp(s, 7), 20, 5):
            counts[p] += 1
    assert stats.chisquare(counts)[1] > 0.01


def test_prng_block_small_graph(small_graph_arrays):
    g = small_graph_arrays
    for kind in ("pcg32", "sfc64", "xoshiro256pp"):
        fr, ed = po.block(g.indptr, g.indices, np.arange(12), [3, 5], 99, kind)
        for inner, outer in zip(fr, fr[1:]):
            assert np.all(np.isin(inner, outer))
        for (src, dst), F in zip(ed, [5, 3]):
            assert np.all(np.bincount(np.searchsorted(fr[0 if F == 5 else 1], dst)) <= F)
