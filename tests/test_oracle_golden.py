"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by
importing gnnpipe from /root/reference).  These run without a GPU."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import fixture_graph, load_case
from oracle import gnn_oracle as orc


def _graph_for(meta, small):
    return small if meta["graph"] == "small" else fixture_graph(meta["graph"])


def test_mix64_known_values():
    assert orc.mix(0) == 0
    v = np.array([0, 1, 2**63, 2**64 - 1], dtype=np.uint64)
    assert [int(x) for x in orc.mix_v(v)] == [orc.mix(int(x)) for x in v]


def test_sample_cases_match_reference(golden, small_npz, small_graph_arrays):
    for c in golden["sample_cases"]:
        meta, seeds, fr, ed = load_case(small_npz, golden, c["name"])
        g = _graph_for(meta, small_graph_arrays)
        got_fr, got_ed = orc.block(g.indptr, g.indices, seeds, meta["fanouts"], int(meta["seed"]))
        assert len(got_fr) == len(fr), c["name"]
        for a, b in zip(got_fr, fr):
            assert np.array_equal(a, b), c["name"]
        for (s1, d1), (s2, d2) in zip(got_ed, ed):
            assert np.array_equal(s1, s2) and np.array_equal(d1, d2), c["name"]


def test_epoch_permutations(golden, small_npz, small_graph_arrays):
    train = np.flatnonzero(small_graph_arrays.train_mask)
    for e in range(3):
        assert np.array_equal(np.concatenate(orc.epoch_chunks(train, 64, 7, e)),
                              small_npz[f"perm_e{e}"])
    big = orc.epoch_chunks(np.arange(153_431), 1000, 1, 0)
    g = golden["epoch_153431"]
    assert len(big) == g["n_batches"] == 154 and len(big[-1]) == g["last"] == 431
    flat = np.concatenate(big)
    assert flat[:16].tolist() == g["head"]
    assert hashlib.blake2b(flat.astype("<i8").tobytes(), digest_size=16).hexdigest() == g["hash"]


def _oracle_plan(g, train, fanouts, batch, epochs, s0):
    h = hashlib.blake2b(digest_size=8)
    sets = []
    for e in range(epochs):
        se = []
        for i, seeds in enumerate(orc.epoch_chunks(train, batch, s0, e)):
            fr, _ = orc.block(g.indptr, g.indices, seeds, fanouts, orc.batch_seed(s0, e, i))
            se.append(fr[-1])
            h.update(np.array([e, i], dtype="<u8").tobytes())
            h.update(fr[-1].astype("<u8").tobytes())
        sets.append(se)
    return sets, f"{int.from_bytes(h.digest(), 'little'):016x}"


def test_plan_digest_and_input_sets(golden, small_npz, small_graph_arrays):
    g = small_graph_arrays
    train = np.flatnonzero(g.train_mask)
    sets, digest = _oracle_plan(g, train, [3, 5], 64, 3, 7)
    assert digest == golden["plan_small"]["digest"]
    for e in range(3):
        off = small_npz[f"plan_off_e{e}"]
        flat = small_npz[f"plan_in_e{e}"]
        for i, s in enumerate(sets[e]):
            assert np.array_equal(s, flat[off[i]:off[i + 1]])


def test_access_counts_and_top_hot(small_npz):
    owner = small_npz["owner2"]
    sets = []
    for e in range(3):
        off, flat = small_npz[f"plan_off_e{e}"], small_npz[f"plan_in_e{e}"]
        sets.append([flat[off[i]:off[i + 1]] for i in range(len(off) - 1)])
    for p in range(2):
        for scope in (None, 0, 1, 2):
            chosen = [s for e in range(3) if scope in (None, e) for s in sets[e]]
            ids, cnt = orc.access_counts(chosen, owner, p)
            tag = f"p{p}_{'all' if scope is None else 'e%d' % scope}"
            assert np.array_equal(ids, small_npz[f"freq_ids_{tag}"])
            assert np.array_equal(cnt, small_npz[f"freq_cnt_{tag}"])
            for n_hot in (0, 1, 5, 20, 80, len(ids) - 1, len(ids), len(ids) + 5):
                key = f"hot_{tag}_{n_hot}"
                if key in small_npz.files:
                    assert np.array_equal(orc.hot_set(ids, cnt, n_hot), small_npz[key]), key


def test_top_hot_kats():
    # plan.py tests (test_plan.py:92-105)
    assert orc.hot_set(np.array([2, 5, 9, 11]), np.array([4, 1, 7, 4]), 2).tolist() == [2, 9]
    assert orc.hot_set(np.array([3, 8, 12]), np.array([5, 5, 5]), 2).tolist() == [3, 8]
    assert orc.hot_set(np.array([1, 2]), np.array([1, 2]), 10).tolist() == [1, 2]
    assert orc.hot_set(np.array([1, 2]), np.array([1, 2]), 0).tolist() == []
    with pytest.raises(ValueError):
        orc.hot_set(np.array([1]), np.array([1]), -1)


def test_bundle_accounting(golden, small_npz):
    owner = small_npz["owner2"]
    off, flat = small_npz["plan_off_e0"], small_npz["plan_in_e0"]
    sets0 = [flat[off[i]:off[i + 1]] for i in range(len(off) - 1)]
    for rec in golden["bundles_small"]:
        p = rec["part"]
        ids, cnt = orc.access_counts(sets0, owner, p)
        hot = orc.hot_set(ids, cnt, rec["n_hot"]) if rec["n_hot"] else None
        got = orc.route_counts(sets0[rec["batch"]], owner, p, hot)
        assert got == (rec["n_local"], rec["n_hit"], rec["n_fallback"], rec["account"][0])
        assert rec["account"][1] == rec["n_fallback"]
        assert rec["account"][2] == rec["n_fallback"] * 4 * 8


@pytest.mark.slow
def test_replay_run_pulls_match_reference_log(golden):
    """The pinned REPLAY config (test_acceptance.py:27-30): per-worker,
    per-epoch fallback pulls/RPCs/hits of rapid and baseline mode, through
    the oracle, equal the reference run (and test_output.txt:196)."""
    from paper_2505_10806_b200.graph import synth_powerlaw
    from paper_2505_10806_b200.partition import partition_edgecut

    cfg = golden["replay"]["config"]
    g = synth_powerlaw(cfg["gen_nodes"], cfg["gen_edges_per_node"], cfg["feat_dim"],
                       cfg["num_classes"], cfg["s0"], with_features=False)
    owner = partition_edgecut(g, cfg["partitions"]).owner
    train = np.flatnonzero(g.train_mask)
    sets, digest = _oracle_plan(g, train, cfg["fanouts"], cfg["batch_size"], cfg["epochs"],
                                cfg["s0"])
    assert digest == "31a0e51d3b2d9a8c" == golden["replay"]["rapid"][0]["digest"]
    totals_rapid, totals_base = [0] * cfg["epochs"], [0] * cfg["epochs"]
    for p in range(cfg["partitions"]):
        all_ids, _ = orc.access_counts([s for se in sets for s in se], owner, p)
        n_hot = int(len(all_ids) * 15.0 / 100.0)
        rec_r = golden["replay"]["rapid"][p]["epochs"]
        rec_b = golden["replay"]["baseline"][p]["epochs"]
        for e in range(cfg["epochs"]):
            ids, cnt = orc.access_counts(sets[e], owner, p)
            hot = orc.hot_set(ids, cnt, n_hot)
            fb = rpc = hits = base = base_rpc = 0
            for s in sets[e]:
                _, h, f, r = orc.route_counts(s, owner, p, hot)
                fb, rpc, hits = fb + f, rpc + r, hits + h
                _, _, f0, r0 = orc.route_counts(s, owner, p, None)
                base, base_rpc = base + f0, base_rpc + r0
            assert [rpc, fb, hits] == [rec_r[e][0], rec_r[e][1], rec_r[e][3]]
            assert [base_rpc, base] == [rec_b[e][0], rec_b[e][1]]
            totals_rapid[e] += fb
            totals_base[e] += base
    # the reference's own pytest log, pkg/test_output.txt:196
    assert totals_rapid == [326975, 326783, 326665, 326985, 327409]
    assert totals_base == [406701, 406553, 406308, 406717, 407090]


def test_mean_aggregation_oracle_in_order():
    rng = np.random.default_rng(0)
    src_front = np.array([1, 3, 4, 7, 9])
    dst_front = np.array([3, 7])
    src = np.array([1, 4, 9, 3, 4])
    dst = np.array([3, 3, 3, 7, 7])
    h = rng.standard_normal((5, 6)).astype(np.float32)
    mean, hs = orc.mean_aggregate(h, src_front, dst_front, src, dst)
    exp0 = ((np.float32(0) + h[0]) + h[2] + h[4]) / np.float32(3)
    assert np.array_equal(mean[0], exp0.astype(np.float32))
    assert np.array_equal(hs, h[[1, 3]])


def _h16(*arrays) -> str:
    m = hashlib.blake2b(digest_size=16)
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()


@pytest.mark.parametrize("name", ["small", "replay", "c1",
                                  pytest.param("products", marks=pytest.mark.slow)])
def test_c_oracle_generator_matches_reference(golden, name):
    """oracle/oracle_graph.c (the bench reference arm's inputs, no product
    library) reproduces gnnpipe's synth_powerlaw + partition_edgecut: CSR,
    features and masks hashes, and the LDG owner arrays."""
    from oracle import graph_oracle as go

    rec = golden["generator"][name]
    n, m, d, _c, s = rec["args"]
    g = go.synth_powerlaw(n, m, d, s)
    want = rec["hash"]
    assert _h16(g.indptr.astype("<i8")) == want["indptr"]
    assert _h16(g.indices.astype("<i4")) == want["indices"]
    assert _h16(g.features.astype("<f4")) == want["features"]
    assert _h16(g.train_mask.astype("u1"), g.val_mask.astype("u1"),
                g.test_mask.astype("u1")) == want["masks"]
    for k, hk in rec["owner"].items():
        assert _h16(go.partition_edgecut(g, int(k)).astype("<i8")) == hk, k
