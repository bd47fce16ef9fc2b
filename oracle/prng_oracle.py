"""CPU ORACLE for the PRNG sampler variants — test infrastructure only.

north_star asks for pcg32 / sfc64 / xoshiro256pp neighbour sampling; the
reference has none of them (only SplitMix64 keys,
rng.py:1-62; its test_multi_prng_*.json fixtures are unidentified), so
parity for these variants is UNPINNED against the reference.  The
semantics are defined in paper_2505_10806_b200/csrc/rg_prng.cuh and
restated here in plain Python integers:

  D <= F                 -> every neighbour (as sampler.py:102-113)
  D  > F                 -> generator seeded from the reference's node key
                            nk = mix((v+1)G ^ s_d) and the step seed s_d;
                            Floyd's algorithm draws F distinct positions
                            with Lemire bounded integers
  edges, frontiers       -> exactly sample_block's (dst, src) sort and union

The raw generators are pinned to public known answers where one exists:
pcg32 to pcg-c-basic's srandom(42, 54) vector, sfc64's step to
numpy.random.SFC64 (state injected), xoshiro256++ to its defining
recurrence.
"""

from __future__ import annotations

import numpy as np

from . import gnn_oracle as orc

M64 = (1 << 64) - 1
M32 = (1 << 32) - 1
G = orc.GOLDEN


def splitmix_next(x: int) -> tuple[int, int]:
    x = (x + G) & M64
    z = x
    z = ((z ^ (z >> 30)) * orc.MIX1) & M64
    z = ((z ^ (z >> 27)) * orc.MIX2) & M64
    return x, z ^ (z >> 31)


def _rotl(x: int, k: int) -> int:
    return ((x << k) | (x >> (64 - k))) & M64


def _lemire64(gen, n: int) -> int:
    x = gen.next64()
    m = x * n
    lo = m & M64
    if lo < n:
        t = ((1 << 64) - n) % n
        while lo < t:
            x = gen.next64()
            m = x * n
            lo = m & M64
    return m >> 64


class Pcg32:
    """pcg_basic.c: pcg32_srandom_r / pcg32_random_r."""

    def __init__(self, initstate: int, initseq: int):
        self.state = 0
        self.inc = ((initseq << 1) | 1) & M64
        self.next32()
        self.state = (self.state + initstate) & M64
        self.next32()

    def next32(self) -> int:
        old = self.state
        self.state = (old * 6364136223846793005 + self.inc) & M64
        xorshifted = (((old >> 18) ^ old) >> 27) & M32
        rot = old >> 59
        return ((xorshifted >> rot) | (xorshifted << ((32 - rot) & 31))) & M32

    def bounded(self, n: int) -> int:
        m = self.next32() * n
        lo = m & M32
        if lo < n:
            t = ((1 << 32) - n) % n
            while lo < t:
                m = self.next32() * n
                lo = m & M32
        return m >> 32


class Sfc64:
    def __init__(self, k0: int, k1: int, state=None):
        if state is not None:
            self.a, self.b, self.c, self.w = state
            return
        x, self.a = splitmix_next(k0 & M64)
        x, self.b = splitmix_next(x)
        self.c = k1 & M64
        self.w = 1
        for _ in range(12):
            self.next64()

    def next64(self) -> int:
        tmp = (self.a + self.b + self.w) & M64
        self.w = (self.w + 1) & M64
        self.a = self.b ^ (self.b >> 11)
        self.b = (self.c + (self.c << 3)) & M64
        self.c = (_rotl(self.c, 24) + tmp) & M64
        return tmp

    def bounded(self, n: int) -> int:
        return _lemire64(self, n)


class Xoshiro256pp:
    def __init__(self, k0: int, k1: int, state=None):
        if state is not None:
            self.s = list(state)
            return
        x = (k0 ^ k1) & M64
        self.s = []
        for _ in range(4):
            x, z = splitmix_next(x)
            self.s.append(z)

    def next64(self) -> int:
        s = self.s
        result = (_rotl((s[0] + s[3]) & M64, 23) + s[0]) & M64
        t = (s[1] << 17) & M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def bounded(self, n: int) -> int:
        return _lemire64(self, n)


KINDS = {"pcg32": Pcg32, "sfc64": Sfc64, "xoshiro256pp": Xoshiro256pp}


def floyd(gen, D: int, T: int) -> list[int]:
    """Floyd's T-subset of range(D), positions in draw order."""
    chosen: list[int] = []
    seen: set[int] = set()
    for j in range(D - T, D):
        t = gen.bounded(j + 1)
        pick = j if t in seen else t
        seen.add(pick)
        chosen.append(pick)
    return chosen


def pick_neighbors(indptr, indices, frontier, fanout: int, seed_d: int, kind: str):
    """One expansion step with a PRNG variant -> (src, dst), unsorted."""
    src, dst = [], []
    for v in np.asarray(frontier, dtype=np.int64).tolist():
        a, b = int(indptr[v]), int(indptr[v + 1])
        D = b - a
        if D <= fanout:
            pos = range(D)
        else:
            nk = orc.mix((((v + 1) * G) & M64) ^ (seed_d & M64))
            pos = sorted(floyd(KINDS[kind](nk, seed_d), D, fanout))
        for p in pos:
            src.append(int(indices[a + p]))
            dst.append(v)
    return np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64)


def block(indptr, indices, seeds, fanouts, rng_seed: int, kind: str):
    """sample_block (sampler.py:116-152) with a PRNG variant -> (frontiers, edges)."""
    if kind == "splitmix":
        return orc.block(indptr, indices, seeds, fanouts, rng_seed)
    L = len(fanouts)
    fr = np.unique(np.asarray(seeds, dtype=np.int64))
    frontiers, edges = [fr], []
    for d in range(L):
        seed_d = orc.mix(rng_seed ^ (((d + 1) * G) & M64))
        src, dst = pick_neighbors(indptr, indices, fr, fanouts[L - 1 - d], seed_d, kind)
        o = np.lexsort((src, dst))
        src, dst = src[o], dst[o]
        edges.append((src, dst))
        fr = np.union1d(fr, src)
        frontiers.append(fr)
    return frontiers, edges
