"""CPU ORACLE — test infrastructure, not product code.

A numpy restatement of the reference hot path (gnnpipe, arxiv 2505.10806's
desk-scale re-creation at /root/reference/pkg/src/gnnpipe).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module; the product path (paper_2505_10806_b200) never does.

Parity pinning: every function here is checked against golden vectors the
reference itself produced (tests/golden/make_golden.py imports gnnpipe from
/root/reference and records its outputs), including the pinned REPLAY run of
the reference's own acceptance suite (pkg/test_output.txt:196).

Each function cites the reference file:line it restates.  Arithmetic is
numpy uint64 wrap-around exactly as in the reference; the neighbour
selection is formulated per (node, position) key so that it can be checked
independently of the reference's lexsort implementation.
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
SHUFFLE_TAG = 0x73687566  # sampler.py:20

_U = np.uint64


def mix(x: int) -> int:
    """SplitMix64 finalizer, scalar (rng.py:28-33)."""
    x &= MASK64
    x = ((x ^ (x >> 30)) * MIX1) & MASK64
    x = ((x ^ (x >> 27)) * MIX2) & MASK64
    return x ^ (x >> 31)


def mix_v(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finalizer over a uint64 array (rng.py:36-44)."""
    y = np.array(x, dtype=np.uint64, copy=True)
    with np.errstate(over="ignore"):
        y ^= y >> _U(30)
        y *= _U(MIX1)
        y ^= y >> _U(27)
        y *= _U(MIX2)
        y ^= y >> _U(31)
    return y


def counter_stream(master: int, count: int) -> np.ndarray:
    """key_j = mix((j+1)*GOLDEN + master) (rng.py:47-50)."""
    j = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix_v(j * _U(GOLDEN) + _U(master & MASK64))


def batch_seed(s0: int, e: int, i: int) -> int:
    """seed_for without the range check (sampler.py:32-40)."""
    return mix(s0 ^ ((e << 32) | i))


def epoch_order(train_nodes: np.ndarray, s0: int, e: int) -> np.ndarray:
    """Permuted train ids of epoch e (sampler.py:55-56, rng.py:53-62):
    stable ascending sort of the per-position counter keys."""
    master = mix(batch_seed(s0, e, 0) ^ SHUFFLE_TAG)
    keys = counter_stream(master, len(train_nodes))
    return np.asarray(train_nodes, dtype=np.int64)[np.argsort(keys, kind="stable")]


def epoch_chunks(train_nodes: np.ndarray, batch_size: int, s0: int, e: int) -> list[np.ndarray]:
    """epoch_batches (sampler.py:43-57)."""
    perm = epoch_order(train_nodes, s0, e)
    return [perm[k:k + batch_size] for k in range(0, len(perm), batch_size)]


def pick_neighbors(indptr, indices, frontier: np.ndarray, fanout: int, seed_d: int):
    """One expansion step (sampler.py:86-113): for each v in frontier keep
    the min(deg, fanout) positions with the smallest mix(nk_v + (p+1)G),
    nk_v = mix((v+1)G ^ seed_d).  Returns (src, dst), not yet sorted."""
    fr = np.asarray(frontier, dtype=np.int64)
    lo = indptr[fr]
    deg = (indptr[fr + 1] - lo).astype(np.int64)
    if deg.sum() == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    owner_row = np.repeat(np.arange(len(fr)), deg)
    first = np.repeat(np.cumsum(deg) - deg, deg)
    p = np.arange(owner_row.size, dtype=np.int64) - first
    with np.errstate(over="ignore"):
        nk = mix_v((fr.astype(np.uint64) + _U(1)) * _U(GOLDEN) ^ _U(seed_d & MASK64))
        key = mix_v(nk[owner_row] + (p.astype(np.uint64) + _U(1)) * _U(GOLDEN))
    # rank of each key inside its node: sort by (row, key), then position
    # within the row's run is the rank
    order = np.lexsort((key, owner_row))
    rank = np.empty_like(p)
    rank[order] = p  # sorted runs start at `first` as the unsorted ones do
    keep = rank < np.minimum(deg, fanout)[owner_row]
    src = np.asarray(indices)[lo[owner_row[keep]] + p[keep]].astype(np.int64)
    dst = fr[owner_row[keep]]
    return src, dst


def block(indptr, indices, seeds, fanouts, rng_seed: int):
    """sample_block (sampler.py:116-152) -> (frontiers, edges)."""
    if len(fanouts) == 0:
        raise ValueError("fanouts must be nonempty")
    seeds = np.asarray(seeds, dtype=np.int64)
    if len(seeds) == 0:
        raise ValueError("seeds must be nonempty")
    L = len(fanouts)
    fr = np.unique(seeds)
    frontiers, edges = [fr], []
    for d in range(L):
        seed_d = mix(rng_seed ^ (((d + 1) * GOLDEN) & MASK64))
        src, dst = pick_neighbors(indptr, indices, fr, fanouts[L - 1 - d], seed_d)
        o = np.lexsort((src, dst))
        src, dst = src[o], dst[o]
        edges.append((src, dst))
        fr = np.union1d(fr, src)
        frontiers.append(fr)
    return frontiers, edges


def access_counts(input_sets, owner: np.ndarray, my_part: int):
    """collect_access over the given input sets (plan.py:108-130):
    (sorted remote ids, per-batch appearance counts)."""
    parts = [ids[owner[ids] != my_part] for ids in input_sets]
    merged = np.concatenate(parts) if parts else np.empty(0, np.int64)
    return np.unique(merged, return_counts=True)


def hot_set(ids: np.ndarray, counts: np.ndarray, n_hot: int) -> np.ndarray:
    """top_hot (plan.py:133-141), as the count-threshold rule of SURVEY.md
    Appendix A.4: every count > c*, then the lowest ids at count == c*."""
    if n_hot < 0:
        raise ValueError("n_hot must be >= 0")
    ids = np.asarray(ids, dtype=np.int64)
    if n_hot >= len(ids):
        return ids.copy()
    if n_hot == 0:
        return np.empty(0, np.int64)
    c_star = np.sort(counts)[::-1][n_hot - 1]
    above = counts > c_star
    quota = n_hot - int(above.sum())
    tie = np.flatnonzero(counts == c_star)[:quota]  # ids ascending
    sel = above.copy()
    sel[tie] = True
    return ids[sel]


def route_counts(input_nodes, owner, my_part: int, hot_ids):
    """Per-bundle provenance and fallback accounting (prefetch.py:57-79,
    cache.py:66-72, store.py:179-195): (n_local, n_hit, n_fallback, rpcs)."""
    ids = np.asarray(input_nodes, dtype=np.int64)
    own = owner[ids]
    local = own == my_part
    remote = ~local
    hot = np.zeros(len(ids), dtype=bool)
    if hot_ids is not None and len(hot_ids):
        pos = np.minimum(np.searchsorted(hot_ids, ids), len(hot_ids) - 1)
        hot = remote & (hot_ids[pos] == ids)
    fb = remote & ~hot
    rpcs = len(np.unique(own[fb]))
    return int(local.sum()), int(hot.sum()), int(fb.sum()), rpcs


def mean_aggregate(h: np.ndarray, src_front, dst_front, src, dst):
    """SAGE mean aggregation (model.py:72-81): in-order fp32 sums / max(cnt,1)
    and the self rows.  Returns (mean, h_self)."""
    sp = np.searchsorted(src_front, src)
    dp = np.searchsorted(dst_front, dst)
    cnt = np.bincount(dp, minlength=len(dst_front)).astype(h.dtype)
    acc = np.zeros((len(dst_front), h.shape[1]), dtype=h.dtype)
    np.add.at(acc, dp, h[sp])
    mean = acc / np.maximum(cnt, 1)[:, None]
    return mean, h[np.searchsorted(src_front, dst_front)]


def mean_aggregate_bwd(dself, dmean, n_src, src_front, dst_front, src, dst):
    """Backward scatter of the aggregation (model.py:126-135)."""
    sp = np.searchsorted(src_front, src)
    dp = np.searchsorted(dst_front, dst)
    cnt = np.bincount(dp, minlength=len(dst_front)).astype(dmean.dtype)
    dh = np.zeros((n_src, dmean.shape[1]), dtype=dmean.dtype)
    np.add.at(dh, np.searchsorted(src_front, dst_front), dself)
    np.add.at(dh, sp, (dmean / np.maximum(cnt, 1)[:, None])[dp])
    return dh
