"""Device parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the CPU oracle.  Bit-exact for every id, count, set and
row; the reference's own REPLAY log is reproduced end to end."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import fixture_graph, load_case
from oracle import gnn_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rg():
    import paper_2505_10806_b200 as rg

    from paper_2505_10806_b200 import _lib

    _lib.device()  # loud failure if the extension or the GPU is missing
    return rg


@pytest.fixture(scope="module")
def small(rg):
    return rg.synth_powerlaw(1000, 5, 8, 4, seed=7)


def test_native_library_is_loaded(rg):
    from paper_2505_10806_b200 import _lib

    lib = _lib.device()
    assert lib.rg_device_ok() == 1
    assert str(_lib.LIB_PATH).endswith("librapidgnn_b200.so")


def test_mix64_and_stream_keys(rg):
    from paper_2505_10806_b200 import _lib

    x = np.array([0, 1, 2, 2**63, 2**64 - 1, 12345678901234567], dtype=np.uint64)
    t = torch.from_numpy(x.view(np.int64)).cuda()
    out = torch.empty_like(t)
    _lib.call("rg_mix64", t.data_ptr(), out.data_ptr(), len(x), _lib.stream_handle())
    assert np.array_equal(out.cpu().numpy().view(np.uint64), orc.mix_v(x))
    keys = torch.empty(1000, dtype=torch.int64, device="cuda")
    _lib.call("rg_stream_keys", 0xDEADBEEF12345678, 1000, keys.data_ptr(), _lib.stream_handle())
    assert np.array_equal(keys.cpu().numpy().view(np.uint64),
                          orc.counter_stream(0xDEADBEEF12345678, 1000))


def test_sample_cases_bit_exact(rg, golden, small_npz, small):
    for c in golden["sample_cases"]:
        meta, seeds, fr, ed = load_case(small_npz, golden, c["name"])
        g = small if meta["graph"] == "small" else fixture_graph(meta["graph"])
        b = rg.sample_block(g, seeds, meta["fanouts"], int(meta["seed"]))
        assert len(b.frontiers) == len(fr)
        for a, w in zip(b.frontiers, fr):
            assert np.array_equal(a, w), c["name"]
        for (s1, d1), (s2, d2) in zip(b.edges, ed):
            assert np.array_equal(s1, s2) and np.array_equal(d1, d2), c["name"]
        assert np.array_equal(b.seeds, seeds)


def test_unsorted_rows_path(rg):
    """CSR rows that are not ascending take the sorting path; same result."""
    rng = np.random.default_rng(5)
    g = rg.synth_powerlaw(3000, 6, 4, 2, seed=3)
    perm_idx = g.indices.copy()
    for v in range(g.num_nodes):
        a, b = g.indptr[v], g.indptr[v + 1]
        perm_idx[a:b] = rng.permutation(perm_idx[a:b])
    g2 = rg.Graph(g.num_nodes, g.num_edges, g.indptr, perm_idx, g.features, g.labels, g.feat_dim,
                  g.num_classes, g.train_mask, g.val_mask, g.test_mask)
    for s in range(4):
        seeds = rng.choice(3000, 128, replace=False)
        b = rg.sample_block(g2, seeds, [7, 40], s)
        fr, ed = orc.block(g2.indptr, g2.indices, seeds, [7, 40], s)
        for a, w in zip(b.frontiers, fr):
            assert np.array_equal(a, w)
        for (s1, d1), (s2, d2) in zip(b.edges, ed):
            assert np.array_equal(s1, s2) and np.array_equal(d1, d2)


def test_sampler_errors(rg, small):
    with pytest.raises(ValueError):
        rg.sample_block(small, np.array([], dtype=np.int64), [3], 0)
    with pytest.raises(ValueError):
        rg.sample_block(small, np.array([0]), [], 0)
    with pytest.raises(ValueError):
        rg.sample_block(small, np.array([small.num_nodes]), [3], 0)
    with pytest.raises(NotImplementedError):
        rg.sample_block(small, np.array([0]), [5000], 0)


def test_epoch_batches(rg, golden, small_npz, small):
    train = np.flatnonzero(small.train_mask)
    sch = rg.SeedSchedule(s0=7, epochs=3, batches_per_epoch=-(-len(train) // 64))
    for e in range(3):
        assert np.array_equal(np.concatenate(rg.epoch_batches(train, 64, sch, e)),
                              small_npz[f"perm_e{e}"])
    big = rg.epoch_batches(np.arange(153_431), 1000, rg.SeedSchedule(1, 1, 154), 0)
    flat = np.concatenate(big)
    assert len(big) == 154 and len(big[-1]) == 431
    want = golden["epoch_153431"]["hash"]
    assert hashlib.blake2b(flat.astype("<i8").tobytes(), digest_size=16).hexdigest() == want
    with pytest.raises(ValueError):
        rg.epoch_batches(np.empty(0, dtype=np.int64), 10, sch, 0)
    with pytest.raises(ValueError):
        rg.epoch_batches(np.arange(5), 0, sch, 0)


@pytest.fixture(scope="module")
def plan_small(rg, small):
    train = np.flatnonzero(small.train_mask)
    return rg.generate_plan(small, train, [3, 5], 64, 3, s0=7)


def test_generate_plan_matches_reference(plan_small, golden, small_npz):
    assert plan_small.digest_hex() == golden["plan_small"]["digest"]
    for e in range(3):
        off, flat = small_npz[f"plan_off_e{e}"], small_npz[f"plan_in_e{e}"]
        for i, s in enumerate(plan_small.input_sets[e]):
            assert np.array_equal(s, flat[off[i]:off[i + 1]])
    blk = plan_small.block(1, 3)
    assert np.array_equal(blk.input_nodes, plan_small.input_sets[1][3])
    assert blk.epoch == 1 and blk.batch == 3


def test_collect_access_and_top_hot(rg, plan_small, small_npz):
    book = rg.PartitionBook(k=2, owner=small_npz["owner2"])
    for p in range(2):
        for scope in (None, 0, 1, 2):
            f = rg.collect_access(plan_small, book, p, epoch=scope)
            tag = f"p{p}_{'all' if scope is None else 'e%d' % scope}"
            assert np.array_equal(f.ids, small_npz[f"freq_ids_{tag}"])
            assert np.array_equal(f.counts, small_npz[f"freq_cnt_{tag}"])
            for n_hot in (0, 1, 5, 20, 80, len(f) - 1, len(f), len(f) + 5):
                key = f"hot_{tag}_{n_hot}"
                if key in small_npz.files:
                    assert np.array_equal(rg.top_hot(f, n_hot), small_npz[key]), key


def test_top_hot_kats_device(rg):
    F = rg.FrequencyTable
    assert rg.top_hot(F(np.array([2, 5, 9, 11]), np.array([4, 1, 7, 4])), 2).tolist() == [2, 9]
    assert rg.top_hot(F(np.array([3, 8, 12]), np.array([5, 5, 5])), 2).tolist() == [3, 8]
    assert rg.top_hot(F(np.array([1, 2]), np.array([1, 2])), 10).tolist() == [1, 2]
    assert rg.top_hot(F(np.array([1, 2]), np.array([1, 2])), 0).tolist() == []
    with pytest.raises(ValueError):
        rg.top_hot(F(np.array([1]), np.array([1])), -1)
    # brute force optimum with least-id ties (test_acceptance.py:347-359)
    import itertools

    rng = np.random.default_rng(7)
    for _ in range(20):
        size = int(rng.integers(1, 10))
        ids = np.sort(rng.choice(100, size=size, replace=False)).astype(np.int64)
        counts = rng.integers(1, 6, size=size).astype(np.int64)
        lookup = dict(zip(ids.tolist(), counts.tolist()))
        for n_hot in range(size + 1):
            chosen = tuple(rg.top_hot(F(ids, counts), n_hot).tolist())
            combos = list(itertools.combinations(ids.tolist(), n_hot))
            best = max(sum(lookup[i] for i in c) for c in combos)
            assert chosen == min(c for c in combos if sum(lookup[i] for i in c) == best)


def _store(rg, g, owner, k=2):
    shards = [rg.StoreShard(p, np.flatnonzero(owner == p), g.features[owner == p])
              for p in range(k)]
    client = rg.StoreClient(owner, [rg.InprocTransport(s) for s in shards], g.feat_dim)
    return shards, client


def test_bundles_match_reference(rg, plan_small, small, small_npz, golden):
    owner = small_npz["owner2"]
    book = rg.PartitionBook(k=2, owner=owner)
    shards, client = _store(rg, small, owner)
    cache, key = None, None
    for rec in golden["bundles_small"]:
        p = rec["part"]
        if (p, rec["n_hot"]) != key:  # one cache per (worker, n_hot), as the golden run
            key = (p, rec["n_hot"])
            f0 = rg.collect_access(plan_small, book, p, epoch=0)
            cache = (rg.build_steady(rg.top_hot(f0, rec["n_hot"]), client, rg.TransferAccount())
                     if rec["n_hot"] else None)
        acct = rg.TransferAccount()
        blk = plan_small.block(0, rec["batch"])
        b = rg.assemble_bundle(blk, owner, p, shards[p], client, cache, acct)
        assert (b.n_local, b.n_cache_hit, b.n_fallback) == (rec["n_local"], rec["n_hit"],
                                                           rec["n_fallback"])
        assert list(acct.snapshot()) == rec["account"]
        assert (cache.hits if cache else 0, cache.misses if cache else 0) == (rec["hits"],
                                                                             rec["misses"])
        assert np.array_equal(b.rows, small.features[blk.input_nodes])


def _make_store(rg):
    rng = np.random.default_rng(42)
    feats = rng.normal(size=(10, 3)).astype(np.float32)
    owner = (np.arange(10) % 2).astype(np.uint32)
    shards = [rg.StoreShard(p, np.flatnonzero(owner == p), feats[owner == p]) for p in range(2)]
    client = rg.StoreClient(owner, [rg.InprocTransport(s) for s in shards], 3)
    return feats, owner, shards, client


def test_store_client_semantics(rg):
    feats, owner, shards, client = _make_store(rg)
    ids = np.array([3, 0, 7, 2])
    assert np.array_equal(client.sync_pull(ids), feats[ids])
    acct = rg.TransferAccount()
    client.vector_pull(np.array([0, 2, 4, 1]), acct)
    assert acct.snapshot() == (2, 4, 48)
    client.sync_pull(np.array([6]), acct)
    assert acct.snapshot() == (3, 5, 60)
    empty = client.sync_pull(np.empty(0, dtype=np.int64), acct)
    assert empty.shape == (0, 3) and acct.snapshot() == (3, 5, 60)
    assert np.array_equal(client.sync_pull(np.array([2, 2, 4])), feats[[2, 2, 4]])
    assert np.array_equal(shards[0].rows_for_local(np.array([4, 0])), feats[[4, 0]])
    assert shards[0].rpc_calls >= 1 and shards[1].nodes_served >= 1
    bad = rg.StoreClient(np.zeros_like(owner), [rg.InprocTransport(s) for s in shards], 3)
    with pytest.raises(rg.LookupError_):
        bad.sync_pull(np.array([1]))


def test_feature_cache_semantics(rg):
    rng = np.random.default_rng(3)
    feats = rng.normal(size=(40, 4)).astype(np.float32)
    owner = np.zeros(40, dtype=np.uint32)
    shard = rg.StoreShard(0, np.arange(40), feats)
    client = rg.StoreClient(owner, [rg.InprocTransport(shard)], 4)
    cache = rg.build_steady(np.array([2, 5, 9]), client)
    res = cache.lookup(np.array([5, 1, 9, 30]))
    assert res.found_pos.tolist() == [0, 2] and res.missing_pos.tolist() == [1, 3]
    assert res.missing_ids.tolist() == [1, 30]
    assert np.array_equal(res.found_rows, feats[[5, 9]])
    assert (cache.hits, cache.misses) == (2, 2)
    empty = rg.build_steady(np.empty(0, dtype=np.int64), client)
    assert empty.lookup(np.array([1, 2])).missing_ids.tolist() == [1, 2]
    c4 = rg.build_steady(np.array([4]), client)
    assert c4.reuse_ratio() is None
    c4.lookup(np.array([4, 4, 6, 8]))
    assert c4.reuse_ratio() == pytest.approx(0.5)
    acct = rg.TransferAccount()
    rg.build_steady(np.array([1, 2, 3, 4, 5]), client, acct)
    assert acct.snapshot() == (1, 5, 80)


def test_double_buffer_swap(rg, plan_small, small, small_npz):
    owner = small_npz["owner2"]
    book = rg.PartitionBook(k=2, owner=owner)
    shards, client = _store(rg, small, owner)
    cache = rg.build_steady(rg.top_hot(rg.collect_access(plan_small, book, 0, epoch=0), 30),
                            client)
    cache.lookup(np.array([0, 5]))
    cache.start_secondary_build(plan_small, 1, book, 0, 30, client)
    cache.wait_secondary()
    assert cache.swap() is True
    expected = rg.top_hot(rg.collect_access(plan_small, book, 0, epoch=1), 30)
    assert np.array_equal(cache.hot_ids, expected)
    assert (cache.hits, cache.misses) == (0, 0)
    assert np.array_equal(cache.lookup(expected).found_rows, small.features[expected])
    assert cache.swap() is False

    class Boom:
        feat_dim = small.feat_dim

        def vector_pull(self, ids, account=None):
            raise ConnectionError("injected")

    before = cache.hot_ids.copy()
    cache.start_secondary_build(plan_small, 2, book, 0, 10, Boom())
    cache.wait_secondary()
    assert cache.swap() is False and np.array_equal(cache.hot_ids, before)


def test_prefetcher_contract(rg, plan_small, small, small_npz):
    owner = small_npz["owner2"]
    shards, client = _store(rg, small, owner)
    pf = rg.Prefetcher(plan_small, 0, owner, 0, shards[0], client, None, None, depth=3)
    seen, i = [], 0
    while (b := pf.next_bundle()) is not None:
        ref = rg.assemble_bundle(plan_small.block(0, i), owner, 0, shards[0], client, None, None)
        assert np.array_equal(b.rows, ref.rows)
        seen.append(b.batch)
        i += 1
    assert seen == list(range(plan_small.num_batches(0)))
    assert pf.next_bundle() is None
    pf = rg.Prefetcher(plan_small, 0, owner, 0, shards[0], client, None, None, depth=2,
                       start_batch=2)
    assert pf.next_bundle().batch == 2
    pf.drain()
    pf.drain()
    assert pf.next_bundle() is None
    with pytest.raises(ValueError):
        rg.Prefetcher(plan_small, 0, owner, 0, shards[0], client, None, None, depth=0)

    class Boom:
        def sync_pull(self, ids, account=None):
            raise ConnectionError("injected")

    pf = rg.Prefetcher(plan_small, 0, owner, 0, shards[0], Boom(), None, None, depth=2)
    with pytest.raises(rg.PrefetchError) as exc:
        while pf.next_bundle() is not None:
            pass
    assert exc.value.batch == 0
    pf.drain()


def test_prefetcher_bounded_runahead(rg, plan_small, small, small_npz):
    import time

    owner = small_npz["owner2"]
    shards, client = _store(rg, small, owner)
    pf = rg.Prefetcher(plan_small, 0, owner, 0, shards[0], client, None, None, depth=2)
    deadline = time.monotonic() + 5
    while pf.assembled < 3 and time.monotonic() < deadline:
        time.sleep(0.01)
    time.sleep(0.3)
    assert pf.assembled <= 3  # queue depth 2 + the bundle in the producer's hand
    pf.drain()


def _records_equal(got, want):
    for p, rec in enumerate(want):
        g = got[p]["records"]
        for e, w in enumerate(rec["epochs"]):
            r = g[e]
            assert [r["rpc_calls"], r["nodes_pulled"], r["bytes_pulled"], r["cache_hits"],
                    r["cache_misses"]] == w[:5], (p, e)
            assert r["reuse_ratio"] == w[5], (p, e)
        assert got[p]["fill"] == rec["fill"], p


@pytest.mark.parametrize("label", ["rapid", "baseline", "hot0", "hot1", "hot5", "global"])
def test_replay_accounting_matches_reference_runs(rg, golden, label):
    """The pinned REPLAY config through the device data path: every
    per-worker per-epoch accounting column of the reference run."""
    from paper_2505_10806_b200.pipeline import run_accounting

    cfg = golden["replay"]["config"]
    g = rg.synth_powerlaw(cfg["gen_nodes"], cfg["gen_edges_per_node"], cfg["feat_dim"],
                          cfg["num_classes"], cfg["s0"])
    book = rg.partition_edgecut(g, cfg["partitions"])
    kw = {"rapid": {}, "baseline": {"mode": "baseline"}, "hot0": {"n_hot": 0},
          "hot1": {"n_hot_pct": 1.0}, "hot5": {"n_hot_pct": 5.0},
          "global": {"hot_scope": "global"}}[label]
    got = run_accounting(g, book, cfg["fanouts"], cfg["batch_size"], cfg["epochs"], cfg["s0"],
                         **kw)
    _records_equal(got, golden["replay"][label])
    if label in ("rapid", "baseline"):
        per_epoch = [sum(got[p]["records"][e]["nodes_pulled"] for p in got) for e in range(5)]
        assert per_epoch == ([326975, 326783, 326665, 326985, 327409] if label == "rapid"
                             else [406701, 406553, 406308, 406717, 407090])


@pytest.mark.parametrize("label", ["rapid", "baseline"])
def test_c1_accounting_matches_reference_runs(rg, golden, label):
    from paper_2505_10806_b200.pipeline import run_accounting

    cfg = golden["c1"]["config"]
    g = rg.synth_powerlaw(cfg["gen_nodes"], cfg["gen_edges_per_node"], cfg["feat_dim"],
                          cfg["num_classes"], cfg["s0"])
    book = rg.partition_edgecut(g, cfg["partitions"])
    got = run_accounting(g, book, cfg["fanouts"], cfg["batch_size"], cfg["epochs"], cfg["s0"],
                         mode=label)
    _records_equal(got, golden["c1"][label])


def test_star_marginal_uniformity(rg):
    """Each leaf of a degree-20 star is picked equally often (test_sampler.py:146-153)."""
    from scipy import stats

    from paper_2505_10806_b200.engine import BlockSampler, DeviceGraph

    g = fixture_graph("star")
    G = 4000
    smp = BlockSampler(DeviceGraph.of(g), [5], 1, group=G)
    smp.seeds.zero_()
    smp.nseeds.fill_(1)
    seeds = np.arange(G, dtype=np.uint64)
    smp.rng.copy_(torch.from_numpy(seeds.view(np.int64)))
    smp.run(G)
    picks = smp.ell[0][:, :5].cpu().numpy()
    assert (smp.cnt[0][:, 0].cpu().numpy() == 5).all()
    counts = np.bincount(picks.ravel() - 1, minlength=20)
    assert stats.chisquare(counts)[1] > 0.01
    # and the device draws equal the oracle's for a few seeds
    for s in (0, 1, 77, 3999):
        fr, ed = orc.block(g.indptr, g.indices, [0], [5], s)
        assert np.array_equal(np.sort(picks[s]), ed[0][0])


def _sage_check(rg, blk, h0, dtype, rng, hidden=48):
    from paper_2505_10806_b200.aggregate import edges_to_ell, sage_mean, sage_mean_backward
    from paper_2505_10806_b200.aggregate import sage_positions

    n_nodes = int(max(int(f.max()) for f in blk.frontiers if len(f))) + 1
    for d in range(blk.num_layers - 1, -1, -1):
        src_front, dst_front = blk.frontiers[d + 1], blk.frontiers[d]
        src, dst = blk.edges[d]
        h = h0 if d == blk.num_layers - 1 else rng.standard_normal(
            (len(src_front), hidden)).astype(dtype)
        want_mean, want_self = orc.mean_aggregate(h, src_front, dst_front, src, dst)
        ell, cnt, F = edges_to_ell(dst_front, src, dst)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        pos = sage_positions(dev(src_front.astype(np.int32)), dev(dst_front.astype(np.int32)),
                             dev(ell), dev(cnt), F, n_nodes)
        mean, hself = sage_mean(dev(h), pos, dev(cnt))
        assert np.array_equal(mean.cpu().numpy(), want_mean)
        assert np.array_equal(hself.cpu().numpy(), want_self)
        dself = rng.standard_normal(want_mean.shape).astype(dtype)
        dmean = rng.standard_normal(want_mean.shape).astype(dtype)
        want_dh = orc.mean_aggregate_bwd(dself, dmean, len(src_front), src_front, dst_front,
                                         src, dst)
        dh = sage_mean_backward(dev(dself), dev(dmean), dev(cnt), pos)
        assert np.array_equal(dh.cpu().numpy(), want_dh)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_sage_mean_fwd_bwd_bit_exact(rg, dtype):
    """K8 against the reference's in-order numpy semantics (model.py:72-81,
    126-135), fp32 and fp64 (RunConfig.precision)."""
    g = rg.synth_powerlaw(20000, 5, 64, 8, seed=7)
    rng = np.random.default_rng(11)
    blk = rg.sample_block(g, rng.choice(20000, 256, replace=False), [10, 25], 99)
    _sage_check(rg, blk, g.features[blk.input_nodes].astype(dtype), dtype, rng)


def test_sage_mean_hub_in_degree_above_4096(rg):
    """A star centre sampled by > 4,096 dst rows: its backward segment is
    longer than any shared-memory sort (the round-1 kernel flagged it and
    went on silently); the radix-sort transpose keeps it bit-exact."""
    n_leaf = 6000
    edges = [(0, j) for j in range(1, n_leaf + 1)]
    g = rg.from_edge_list(n_leaf + 1, edges, feat_dim=20)
    rng = np.random.default_rng(5)
    g.features[:] = rng.standard_normal(g.features.shape).astype(np.float32)
    blk = rg.sample_block(g, np.arange(1, n_leaf + 1), [3], 17)
    src, dst = blk.edges[0]
    assert int((src == 0).sum()) == n_leaf  # every leaf's only neighbour is the hub
    _sage_check(rg, blk, g.features[blk.input_nodes], np.float32, rng)


def test_sage_mean_strided_rows(rg):
    """the forward reads h with its row pitch (h.stride(0)), so a
    view of padded bundle rows with feat_dim % 4 != 0 (d = 6, the reference's
    acceptance graph) aggregates the right rows."""
    from paper_2505_10806_b200.aggregate import edges_to_ell, sage_mean, sage_positions

    g = rg.synth_powerlaw(3000, 4, 6, 3, seed=7)
    rng = np.random.default_rng(2)
    blk = rg.sample_block(g, rng.choice(3000, 64, replace=False), [5, 4], 3)
    src_front, dst_front = blk.frontiers[2], blk.frontiers[1]
    src, dst = blk.edges[1]
    h = g.features[src_front]
    padded = np.zeros((len(src_front), 8), np.float32)
    padded[:, :6] = h
    view = torch.from_numpy(padded).cuda()[:, :6]
    assert view.stride(0) == 8
    want_mean, want_self = orc.mean_aggregate(h, src_front, dst_front, src, dst)
    ell, cnt, F = edges_to_ell(dst_front, src, dst)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    pos = sage_positions(dev(src_front.astype(np.int32)), dev(dst_front.astype(np.int32)),
                         dev(ell), dev(cnt), F, g.num_nodes)
    mean, hself = sage_mean(view, pos, dev(cnt))
    assert np.array_equal(mean.cpu().numpy(), want_mean)
    assert np.array_equal(hself.cpu().numpy(), want_self)


@pytest.mark.parametrize("nbits", [3_000_000, 12_000_000])
def test_bitmap_compact_both_scan_paths(rg, nbits):
    """rg_bitmap_compact (np.unique / np.union1d, sampler.py:138,148) on G = 3
    bitmaps: below and above the chunk count where the chunk totals get their
    own scan kernel (papers100M-sized node sets); ids, counts and the per-word
    ranks wpre equal numpy's."""
    from paper_2505_10806_b200 import _lib

    lib = _lib.load()
    G = 3
    nwords = (nbits + 31) // 32
    assert (lib.rg_bitmap_compact_launches(nwords) == 3) == (nbits > 8_388_608)
    rng = np.random.default_rng(nbits)
    dens = [0.001, 0.05, 0.3]
    bits = np.zeros((G, nwords * 32), bool)
    for b in range(G):
        bits[b, :nbits] = rng.random(nbits) < dens[b]
    # bit j of word w = node 32 w + j
    words = np.packbits(bits.reshape(G, nwords * 32), axis=-1, bitorder="little").view("<u4")
    cap = int(bits.sum(axis=1).max()) + 1
    d_bm = torch.from_numpy(words.view(np.int32).copy()).cuda()
    chunk = torch.empty((G, int(lib.rg_bitmap_chunks(nwords))), dtype=torch.int32, device="cuda")
    out = torch.empty((G, cap), dtype=torch.int32, device="cuda")
    nout = torch.empty(G, dtype=torch.int32, device="cuda")
    wpre = torch.empty((G, nwords), dtype=torch.int32, device="cuda")
    _lib.call("rg_bitmap_compact", d_bm.data_ptr(), nwords, G, chunk.data_ptr(), out.data_ptr(),
              cap, nout.data_ptr(), wpre.data_ptr(), _lib.stream_handle())
    got_n, got, got_pre = nout.cpu().numpy(), out.cpu().numpy(), wpre.cpu().numpy()
    for b in range(G):
        ids = np.flatnonzero(bits[b])
        assert got_n[b] == len(ids)
        assert np.array_equal(got[b, : len(ids)], ids)
        pc = bits[b].reshape(nwords, 32).sum(axis=1)
        assert np.array_equal(got_pre[b], np.concatenate([[0], np.cumsum(pc)[:-1]]))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_softmax_xent_and_sgd_apply(rg, dtype):
    """The training step's fused head and update (rg_softmax_xent,
    rg_sgd_apply) against the reference's expressions (model.py:107-124,
    139-146) in numpy: loss and gradient over the live seed rows (padding
    rows zero), and w - lr * g with the chunk partials summed in order
    (bit-exact: the same per-operation rounding)."""
    import ctypes

    from paper_2505_10806_b200 import _lib

    rng = np.random.default_rng(5)
    cap, n, C, nodes = 96, 77, 47, 500
    logits = (rng.standard_normal((cap, C)) * 3).astype(dtype)
    labels = rng.integers(0, C, nodes).astype(np.int64)
    front0 = np.sort(rng.choice(nodes, cap, replace=False)).astype(np.int32)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    d_l, d_lab, d_f = dev(logits), dev(labels), dev(front0)
    d_n = dev(np.array([n], np.int32))
    d_dz = torch.full((cap, C), 7.0, dtype=d_l.dtype, device="cuda")
    loss = torch.zeros((), dtype=torch.float64, device="cuda")
    code = 0 if dtype == np.float32 else 1
    nll = torch.empty(cap, dtype=d_l.dtype, device="cuda")
    _lib.call("rg_softmax_xent", code, d_l.data_ptr(), C, cap, d_n.data_ptr(), d_lab.data_ptr(),
              d_f.data_ptr(), d_dz.data_ptr(), nll.data_ptr(), loss.data_ptr(),
              _lib.stream_handle())
    x = logits[:n].astype(np.float64)
    y = labels[front0[:n]]
    sh = x - x.max(axis=1, keepdims=True)
    se = np.exp(sh).sum(axis=1)
    want_loss = float(np.mean(np.log(se) - sh[np.arange(n), y]))
    want_dz = np.exp(sh) / se[:, None]
    want_dz[np.arange(n), y] -= 1
    want_dz /= n
    tol = 2e-6 if dtype == np.float32 else 1e-12
    got = d_dz.cpu().numpy()
    assert np.all(got[n:] == 0)
    assert np.allclose(got[:n], want_dz, rtol=tol * 10, atol=tol)
    assert float(loss.item()) == pytest.approx(want_loss, rel=tol * 10)
    # update: three tensors, 21 / 3 / 1 chunk partials
    lr = 0.05
    shapes = [(100, 32), (32, 47), (47,)]
    chunks = [21, 3, 1]
    ws = [rng.standard_normal(sh).astype(dtype) for sh in shapes]
    gs = [rng.standard_normal((c,) + sh).astype(dtype) for c, sh in zip(chunks, shapes)]
    d_ws, d_gs = [dev(w) for w in ws], [dev(g) for g in gs]
    _lib.call("rg_sgd_apply", code, 3, (ctypes.c_void_p * 3)(*[w.data_ptr() for w in d_ws]),
              (ctypes.c_void_p * 3)(*[g.data_ptr() for g in d_gs]),
              (ctypes.c_int64 * 3)(*[w.size for w in ws]), (ctypes.c_int32 * 3)(*chunks), lr,
              _lib.stream_handle())
    for w, g, d_w in zip(ws, gs, d_ws):
        part = []
        for k in range(8):  # in-order sums over c = k, k + 8, ...
            acc = np.zeros_like(g[0])
            for c in range(k, g.shape[0], 8):
                acc = g[c].copy() if c == k else acc + g[c]
            part.append(acc)
        s_ = ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]))
        assert np.array_equal(d_w.cpu().numpy(), w - dtype(lr) * s_)


@pytest.mark.parametrize("kind", ["pcg32", "sfc64", "xoshiro256pp"])
def test_prng_variant_blocks_match_oracle(rg, small, kind):
    """Device PRNG-variant sampling == the variant oracle (fast and CTA paths)."""
    from oracle import prng_oracle as po

    g2 = rg.synth_powerlaw(20000, 5, 8, 4, seed=7)
    rng = np.random.default_rng(17)
    cases = [(small, np.arange(10), [3, 5]), (small, np.arange(40), [40, 48]),
             (g2, rng.choice(20000, 256, replace=False), [10, 25]),
             (g2, rng.choice(20000, 64, replace=False), [15, 10, 5])]
    for g, seeds, fan in cases:
        s = int(rng.integers(2**63))
        b = rg.sample_block(g, seeds, fan, s, prng=kind)
        fr, ed = po.block(g.indptr, g.indices, seeds, fan, s, kind)
        for a, w in zip(b.frontiers, fr):
            assert np.array_equal(a, w)
        for (s1, d1), (s2, d2) in zip(b.edges, ed):
            assert np.array_equal(s1, s2) and np.array_equal(d1, d2)


def test_prng_variant_plan_and_accounting(rg):
    """The variant flows through the plan pass and the data-path accounting."""
    from oracle import prng_oracle as po
    from paper_2505_10806_b200.pipeline import run_accounting

    g = rg.synth_powerlaw(20000, 5, 32, 8, seed=7)
    book = rg.partition_edgecut(g, 2)
    train = np.flatnonzero(g.train_mask)
    plan = rg.generate_plan(g, train, [10, 25], 512, 1, 7, prng="sfc64")
    sets = []
    for i, seeds in enumerate(plan.batch_seeds[0]):
        fr, _ = po.block(g.indptr, g.indices, seeds, [10, 25],
                         orc.batch_seed(7, 0, i), "sfc64")
        assert np.array_equal(plan.input_sets[0][i], fr[-1])
        sets.append(fr[-1])
    got = run_accounting(g, book, [10, 25], 512, 1, 7, prng="sfc64", workers=[0])
    all_ids, _ = orc.access_counts(sets, book.owner, 0)
    hot = orc.hot_set(*orc.access_counts(sets, book.owner, 0), int(len(all_ids) * 15 / 100))
    fb = sum(orc.route_counts(s, book.owner, 0, hot)[2] for s in sets)
    assert got[0]["records"][0]["nodes_pulled"] == fb


@pytest.fixture(scope="module")
def products(rg, golden):
    """Products-shape graph (hash-pinned to the reference's generator), its
    8-way LDG partition and the device store for worker 0."""
    from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore

    rec = golden["generator"]["products"]
    n, m, d, c, s = rec["args"]
    g = rg.synth_powerlaw(n, m, d, c, s)
    h = lambda a: hashlib.blake2b(np.ascontiguousarray(a).tobytes(),  # noqa: E731
                                  digest_size=16).hexdigest()
    assert h(g.indptr.astype("<i8")) == rec["hash"]["indptr"]
    assert h(g.indices.astype("<i4")) == rec["hash"]["indices"]
    book = rg.partition_edgecut(g, 8)
    dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
    store = FeatureStore(book.owner, 8, d)
    ids = [np.flatnonzero(book.owner == q) for q in range(8)]
    for q in range(8):
        store.set_shard(q, FeatureStore.pad_rows(g.features[ids[q]], store.src_stride, dg.device))
    store.build_route(ids)
    return g, dg, store


def test_products_full_size(products):
    """Products shape at full size: inputs hash-equal to the reference's
    generator, a full epoch of device sampling + gather whose remote-row and
    RPC accounting equals the survey's oracle figures (SURVEY.md §8a row 14:
    933,549,256 rows, 11,725 RPCs for worker 0), first and last batch
    bit-exact against the oracle, bundle rows equal to the feature rows."""
    from paper_2505_10806_b200.pipeline import WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule, block_from_sampler

    g, dg, store = products
    d = g.feat_dim
    feats = torch.from_numpy(g.features).cuda()
    train = np.flatnonzero(g.train_mask)
    pipe = WorkerPipeline(dg, store, 0, train, [15, 10, 5], 1024, 7, 32, nbuf=1)
    sched = SeedSchedule(7, 1, pipe.nb)
    pipe.start_epoch(sched, 0)
    perm = pipe.perm.cpu().numpy()
    smp = pipe.sampler
    for i0 in range(0, pipe.nb, pipe.G):
        ng = pipe.step(i0)
        if i0 == 0 or i0 + ng == pipe.nb:
            slot = 0 if i0 == 0 else ng - 1
            i = i0 + slot
            seeds = perm[i * 1024:(i + 1) * 1024]
            blk = block_from_sampler(smp, slot, seeds, 0, i)
            fr, ed = orc.block(g.indptr, g.indices, seeds, [15, 10, 5], orc.batch_seed(7, 0, i))
            for a, w in zip(blk.frontiers, fr):
                assert np.array_equal(a, w), i
            for (s1, d1), (s2, d2) in zip(blk.edges, ed):
                assert np.array_equal(s1, s2) and np.array_equal(d1, d2), i
            nin = len(fr[-1])
            rows = pipe.rows[slot, :nin, :d]
            want = feats[torch.from_numpy(fr[-1]).cuda()]
            assert torch.equal(rows, want), i
    t = pipe.totals()
    assert t["bad"] == 0
    assert t["hit"] + t["fallback"] == 933_549_256
    assert t["rpcs"] == 11_725


def test_products_reference_goldens(rg, products):
    """Products scale, pinned to the REFERENCE's own outputs at the metric's
    configuration (tests/golden/make_golden_products.py ran gnnpipe's
    sample_block / collect_access / top_hot / assemble_bundle over the whole
    epoch): every batch's input_nodes and the plan digest, the access table
    of all 8 workers, the hot sets at 5/10/15/20/65 % and worker 0's per-batch
    accounting (local, hit, fallback, RPCs) at 0/5/10/15/20/65 %, all
    bit-exact (plan.py:72-141, prefetch.py:41-88, train.py:165-168)."""
    import json
    from pathlib import Path

    from paper_2505_10806_b200 import _lib
    from paper_2505_10806_b200.pipeline import WorkerPipeline, resolve_n_hot
    from paper_2505_10806_b200.plan import candidates, threshold_select
    from paper_2505_10806_b200.sampler import SeedSchedule

    gold_dir = Path(__file__).resolve().parent / "golden"
    gold = json.loads((gold_dir / "products.json").read_text())
    z = np.load(gold_dir / "products_w0.npz")
    h16 = lambda *a: hashlib.blake2b(b"".join(np.ascontiguousarray(x).tobytes()  # noqa: E731
                                              for x in a), digest_size=16).hexdigest()
    g, dg, store = products
    owner = np.asarray(store.owner_np)
    train = np.flatnonzero(g.train_mask)
    pipe = WorkerPipeline(dg, store, 0, train, [15, 10, 5], 1024, 7, 32, nbuf=1)
    nb = pipe.nb
    assert nb == gold["config"]["batches"]
    sched = SeedSchedule(7, 1, nb)

    # every batch's input nodes + the reference plan digest
    pipe.start_epoch(sched, 0)
    smp = pipe.sampler
    dig = hashlib.blake2b(digest_size=8)
    total = 0
    for i0 in range(0, nb, pipe.G):
        ng = pipe.step(i0)
        nf = smp.nfront[smp.L, :ng].cpu().numpy()
        front = smp.front[smp.L][:ng].cpu().numpy()
        for b in range(ng):
            ids = front[b, : nf[b]].astype("<i8")
            i = i0 + b
            assert nf[b] == z["input_len"][i], i
            assert hashlib.blake2b(ids.tobytes(), digest_size=16).digest() == \
                z["input_hash"][i].tobytes(), i
            dig.update(np.array([0, i], dtype="<u8").tobytes())
            dig.update(ids.astype("<u8").tobytes())
            total += int(nf[b])
    assert f"{int.from_bytes(dig.digest(), 'little'):016x}" == gold["plan_digest"]
    assert total == gold["inputs_total"]

    # collect_access: dense counts (worker independent) and every worker's table
    counts = pipe.count_epoch(sched, 0)
    c_np = counts.cpu().numpy()
    allt = gold["all_nodes_table"]
    assert h16(c_np.astype("<i4")) == allt["dense_i32"]
    assert int(c_np.sum()) == allt["accesses"] and int(c_np.max()) == allt["max"]
    hot_w0 = {}
    for p in range(8):
        rec = gold["workers"][str(p)]
        ids = np.flatnonzero((c_np > 0) & (owner != p))
        assert len(ids) == rec["n_remote"], p
        assert h16(ids.astype("<i8"), c_np[ids].astype("<i8")) == rec["table"], p
        _, nout, hist, bm = candidates(counts, store.owner, p, nb)
        assert int(nout.item()) == rec["n_remote"]
        for pct, want in rec["hot"].items():
            n_hot = resolve_n_hot(float(pct), rec["n_remote"])
            assert n_hot == want["n_hot"], (p, pct)
            if p != 0 and pct != "15":
                continue
            hot = threshold_select(counts, bm, hist.cpu().numpy().astype(np.int64), n_hot)
            hot_np = hot.cpu().numpy().astype(np.int64)
            assert h16(hot_np.astype("<i8")) == want["ids"], (p, pct)
            if p == 0:
                hot_w0[int(pct)] = hot
    want15 = np.cumsum(z["hot15_delta"].astype(np.int64))
    assert np.array_equal(hot_w0[15].cpu().numpy(), want15)

    # worker 0's per-batch accounting with each steady cache (and none)
    for pct in [0, 5, 10, 15, 20, 65]:
        pipe.cache = None if pct == 0 else pipe.build_cache(hot_w0[pct])
        pipe.start_epoch(sched, 0)
        for i0 in range(0, nb, pipe.G):
            pipe.step(i0)
        c = pipe.totals()["per_batch"]
        rpcs = np.array([bin(int(m)).count("1") for m in c[:, _lib.RG_CNT_OWNER_MASK]])
        got = np.stack([c[:, 0], c[:, 1], c[:, 2], rpcs], axis=1)
        assert np.array_equal(got, z[f"acct_{pct}"]), pct
        acc = gold["w0_accounting"][str(pct)]
        assert int(c[:, 2].sum()) == acc["nodes_pulled"] and int(rpcs.sum()) == acc["rpc_calls"]
        assert int(c[:, 1].sum()) == acc["cache_hits"]
    pipe.cache = None


def test_products_epoch_properties(products):
    """Every batch of a full Products epoch (not just sampled ones), checked
    on the device through size-independent properties of sample_block
    (sampler.py:86-152) and assemble_bundle (prefetch.py:41-88):
    take = min(deg, F); each ELL row strictly ascending (without replacement)
    and a subset of the node's CSR row; F_{d+1} = unique(F_d U src) sorted;
    bundle rows = the feature rows of the input nodes."""
    from paper_2505_10806_b200.pipeline import WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule

    g, dg, store = products
    n, d = g.num_nodes, g.feat_dim
    feats = torch.from_numpy(g.features).cuda()
    indptr = dg.indptr
    deg = indptr[1:] - indptr[:-1]
    # CSR rows are ascending, so row * n + col is globally sorted
    rowkey = (torch.repeat_interleave(torch.arange(n, device="cuda"), deg) * n
              + dg.indices.long())
    train = np.flatnonzero(g.train_mask)
    pipe = WorkerPipeline(dg, store, 0, train, [15, 10, 5], 1024, 7, 32, nbuf=1)
    pipe.start_epoch(SeedSchedule(7, 1, pipe.nb), 0)
    smp = pipe.sampler
    checked = 0
    for i0 in range(0, pipe.nb, pipe.G):
        ng = pipe.step(i0)
        nf = smp.nfront[:, :ng].long()
        for lv in range(smp.L):
            F, cap = smp.step_fan[lv], smp.caps[lv]
            ar = torch.arange(cap, device="cuda")
            valid = ar[None, :] < nf[lv][:, None]                       # (ng, cap)
            v = smp.front[lv][:ng].long() * valid
            cnt = smp.cnt[lv][:ng]
            want = torch.minimum(deg[v], torch.tensor(F, device="cuda"))
            assert torch.equal(cnt[valid], want[valid].int()), (i0, lv)
            ell = smp.ell[lv][:ng].view(ng, cap, F).long()
            ev = valid[:, :, None] & (torch.arange(F, device="cuda")[None, None, :]
                                       < cnt[:, :, None])
            if F > 1:
                both = ev[:, :, 1:]
                assert bool((ell[:, :, 1:] > ell[:, :, :-1])[both].all()), (i0, lv)
            key = (v[:, :, None] * n + ell)[ev]
            pos = torch.searchsorted(rowkey, key).clamp_max(rowkey.numel() - 1)
            assert torch.equal(rowkey[pos], key), (i0, lv)
            # union: per slot offset by b * n, then one sorted unique
            off = torch.arange(ng, device="cuda")[:, None] * n
            cur = (v + off)[valid]
            src = (ell + off[:, :, None])[ev]
            uni = torch.unique(torch.cat([cur, src]))
            valid2 = torch.arange(smp.caps[lv + 1], device="cuda")[None, :] < nf[lv + 1][:, None]
            nxt = (smp.front[lv + 1][:ng].long() + off)[valid2]
            assert torch.equal(uni, nxt), (i0, lv)
        L = smp.L
        validL = torch.arange(smp.caps[L], device="cuda")[None, :] < nf[L][:, None]
        ids = smp.front[L][:ng].long()[validL]
        assert torch.equal(pipe.rows[:ng, :, :d][validL], feats[ids]), i0
        checked += ng
    assert checked == pipe.nb
    assert pipe.totals()["bad"] == 0


@pytest.mark.parametrize("mode", ["rapid", "baseline"])
def test_training_run_matches_reference_records(rg, golden, mode, tmp_path):
    """train.run on the device (data path + GraphSAGE step + SGD + eval)
    against the reference's REPLAY run: accounting columns and digest
    bit-exact, loss within rel 1e-5, train accuracy within 1e-3."""
    from paper_2505_10806_b200.train import RunConfig, read_metrics, run, worker_metrics_path

    cfg = RunConfig(**golden["replay"]["config"], mode=mode,
                    metrics_out=str(tmp_path / "m.csv"))
    res = run(cfg)
    ref = golden["replay"][mode]
    for r, w in zip(res, ref):
        assert r.plan_digest == w["digest"] == "31a0e51d3b2d9a8c"
        assert list(r.cache_fill) == w["fill"]
        for rec, we in zip(r.records, w["epochs"]):
            assert [rec.rpc_calls, rec.nodes_pulled, rec.bytes_pulled, rec.cache_hits,
                    rec.cache_misses, rec.reuse_ratio] == we[:6]
            assert rec.loss == pytest.approx(we[6], rel=1e-5)
            assert abs(rec.train_acc - we[7]) <= 1e-3
        csv_rec = read_metrics(worker_metrics_path(cfg.metrics_out, r.part))
        assert [c.nodes_pulled for c in csv_rec] == [x.nodes_pulled for x in r.records]


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_graph_trainer_matches_eager_step(rg, golden, precision):
    """The graph-captured training step (model.GraphTrainer: chunked weight
    gradients, rg_softmax_xent, rg_sgd_apply, accumulating-GEMM bias) equals
    the eager loss_and_grad + sgd_step path (model.py:107-146) up to the
    fp32 summation order: per-epoch losses within rel 1e-5 (f64: 1e-10),
    final parameters within the same tolerance."""
    from paper_2505_10806_b200.train import RunConfig, run

    base = dict(golden["replay"]["config"], epochs=2, precision=precision)
    a = run(RunConfig(**base, mode="rapid", cuda_graphs=True))
    b = run(RunConfig(**base, mode="rapid", cuda_graphs=False))
    rel = 1e-5 if precision == "f32" else 1e-10
    for ra, rb in zip(a, b):
        for xa, xb in zip(ra.records, rb.records):
            assert xa.loss == pytest.approx(xb.loss, rel=rel)
        for pa, pb in zip(ra.params, rb.params):
            for ta, tb in ((pa.w_self, pb.w_self), (pa.w_neigh, pb.w_neigh), (pa.bias, pb.bias)):
                assert torch.allclose(ta, tb, rtol=rel * 10, atol=rel)


def test_training_mode_equivalence(rg, golden):
    """Criterion 3 of the reference acceptance suite (test_acceptance.py:113-122):
    rapid and baseline consume bit-identical rows, so losses, accuracies and
    final parameters are identical."""
    from paper_2505_10806_b200.train import RunConfig, run

    base = dict(golden["replay"]["config"], epochs=2)
    a = run(RunConfig(**base, mode="rapid"))
    b = run(RunConfig(**base, mode="baseline"))
    for ra, rb in zip(a, b):
        assert [x.loss for x in ra.records] == [x.loss for x in rb.records]
        assert [x.train_acc for x in ra.records] == [x.train_acc for x in rb.records]
        for pa, pb in zip(ra.params, rb.params):
            assert torch.equal(pa.w_self, pb.w_self) and torch.equal(pa.w_neigh, pb.w_neigh)
            assert torch.equal(pa.bias, pb.bias)


@pytest.mark.parametrize("mode", ["prefetch", "nccl", "pull"])
def test_two_gpu_peer_gather_bit_exact(mode):
    """One process per GPU, peer shards over NVLink (CUDA IPC), with the
    group prefetch into local shadows (NVLink loads, or NCCL all-to-all as
    the transport) or per-batch peer pulls:
    batch 0 of every rank bit-exact (blocks and rows, including rows that
    came over NVLink) and the epoch accounting unchanged.  Needs >= 2 GPUs;
    skipped otherwise."""
    import json
    import os
    import socket
    import subprocess
    import sys
    from pathlib import Path

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = Path(__file__).resolve().parents[1]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(root / "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--no-cpu", "--no-e2e", "--check",
           "--group", "32"]  # correctness run: small groups
    if mode == "pull":
        cmd.append("--pull")
    elif mode == "nccl":
        cmd += ["--transport", "nccl"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root,
                         env=dict(os.environ))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["check"]["all_ranks_bit_exact"] is True
    # the ranks split each group's sampling and copy the shares over NVLink
    assert line["check"]["shared_sampling_bit_exact"] is True
    assert line["remote_rows_epoch"]["uncached"] == 933_549_256
    assert line["remote_rows_epoch"]["rpcs"] == 11_725
    if mode == "pull":
        assert line["nvlink"]["peer_rows_per_batch"] > 0
    else:
        assert line["nvlink"]["prefetched_rows_per_batch"] > 0


def test_prefetch_kernels_units(rg):
    """K9 building blocks on one GPU: route-kind bits, masked group union,
    row copy into shadows and the NCCL-transport scatter, against torch."""
    from paper_2505_10806_b200 import _lib
    from paper_2505_10806_b200.engine import bases_array

    gen = torch.Generator().manual_seed(3)
    n, G = 5000, 5
    nw = (n + 31) // 32
    kinds = torch.randint(0, 4, (n,), generator=gen)
    rows_of = torch.zeros(n, dtype=torch.int64)
    for q in range(4):
        m = kinds == q
        rows_of[m] = torch.arange(int(m.sum()))
    route = ((kinds << 28) | rows_of).to(torch.int64)
    route[::97] = 0xFFFFFFFF  # invalid words
    route32 = torch.from_numpy(route.numpy().astype(np.uint32).view(np.int32)).cuda()
    s = _lib.stream_handle()
    bits = torch.empty(nw, dtype=torch.int32, device="cuda")
    _lib.call("rg_route_kind_bits", route32.data_ptr(), n, 0b1010, bits.data_ptr(), s)
    want = torch.zeros(nw * 32, dtype=torch.bool)
    valid = route != 0xFFFFFFFF
    want[:n] = valid & ((kinds == 1) | (kinds == 3))
    got = ((bits.cpu().to(torch.int64)[:, None] >> torch.arange(32)) & 1).reshape(-1).bool()
    assert torch.equal(got, want)
    bm = torch.randint(-2**31, 2**31 - 1, (G, nw), generator=gen, dtype=torch.int64).to(
        torch.int32).cuda()
    out = torch.empty(nw, dtype=torch.int32, device="cuda")
    _lib.call("rg_group_union", bm.data_ptr(), nw, G, bits.data_ptr(), out.data_ptr(), s)
    ref = bm[0].clone()
    for b in range(1, G):
        ref |= bm[b]
    assert torch.equal(out, ref & bits)
    # prefetch_rows / scatter_rows: kinds 1 and 3 from "peer" shards into shadows
    stride = 12
    shards = {q: torch.randn((int((kinds == q).sum()), stride), generator=gen).cuda()
              for q in range(4)}
    ids = torch.nonzero(want[:n]).flatten().to(torch.int32).cuda()
    nid = torch.tensor([ids.numel()], dtype=torch.int32, device="cuda")
    src = [0] * 16
    dst = [0] * 16
    shadow = {}
    for q in (1, 3):
        src[q] = shards[q].data_ptr()
        shadow[q] = torch.zeros_like(shards[q])
        dst[q] = shadow[q].data_ptr()
    _lib.call("rg_prefetch_rows", ids.data_ptr(), nid.data_ptr(), ids.numel(),
              route32.data_ptr(), bases_array(src), bases_array(dst), stride, stride, s)
    for q in (1, 3):
        sel = rows_of[(kinds == q) & valid]
        assert torch.equal(shadow[q][sel.cuda()], shards[q][sel.cuda()])
    # scatter: rows listed in ids order land at their (kind, row)
    perm = torch.randperm(ids.numel(), generator=gen).cuda()
    ids_p = ids[perm].contiguous()
    k_p = kinds[ids_p.cpu().long()]
    r_p = rows_of[ids_p.cpu().long()]
    payload = torch.stack([shards[int(k)][int(r)] for k, r in zip(k_p, r_p)]).cuda()
    for q in (1, 3):
        shadow[q].zero_()
    _lib.call("rg_scatter_rows", ids_p.data_ptr(), ids_p.numel(), route32.data_ptr(),
              payload.data_ptr(), stride, bases_array(dst), stride, stride, s)
    for q in (1, 3):
        sel = rows_of[(kinds == q) & valid]
        assert torch.equal(shadow[q][sel.cuda()], shards[q][sel.cuda()])


@pytest.mark.parametrize("group", [16, 4])  # dense (window gather) / sparse (id lists)
def test_shared_sampling_two_workers_one_gpu(group):
    """Shared sampling without a second GPU: two workers'
    pipelines in one process, wired to each other's buffers and sequence
    counters by plain device addresses instead of IPC mappings, produce
    three groups alternately (slot reuse included), each sampling half of
    every group and copying the other half.  Every batch's whole block
    (frontiers, counts, ELL edges, bitmap) and bundle rows equal a pipeline
    that sampled everything itself, and so do the per-batch counters.
    Runs in a subprocess with 32 hardware work queues (both workers' streams
    share one GPU here, and with the default 8 queues a spinning cross-worker
    wait could alias onto the queue of the work it waits for); the helper
    loads every kernel before the first wait is in flight and drives each
    worker from its own host thread, as one process per GPU would (a single
    thread interleaving both timed out in the id-list mode: a host-side
    stall while one worker's wait spun kept the other's signal unqueued)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    helper = Path(__file__).with_name("shared_one_gpu.py")
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32")
    out = subprocess.run([sys.executable, str(helper), str(group)], capture_output=True,
                         text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "shared ok" in out.stdout


def test_group_prefetch_pipeline_single_gpu(rg, products):
    """The whole group-prefetch path on one GPU: shards 1..7 registered as
    'peer' addresses (set_shard(q, None, base)), so every step copies the
    group's union into shadows and gathers all-local; bundle rows equal the
    feature rows and the epoch accounting equals the plain pipeline's."""
    from paper_2505_10806_b200.engine import FeatureStore
    from paper_2505_10806_b200.pipeline import WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule

    g, dg, store = products
    d = g.feat_dim
    book_owner = store.owner_np
    st2 = FeatureStore(book_owner, 8, d)
    for q in range(8):
        if q == 0:
            st2.set_shard(q, store.shards[0])
        else:
            st2.set_shard(q, None, base=store.shards[q].data_ptr())
    st2.route = store.route
    assert st2.peer_mask == 0b11111110
    train = np.flatnonzero(g.train_mask)
    feats = torch.from_numpy(g.features).cuda()
    pipe = WorkerPipeline(dg, st2, 0, train, [15, 10, 5], 1024, 7, 16, nbuf=2)
    pipe.enable_prefetch()
    assert pipe.prefetch
    sched = SeedSchedule(7, 1, pipe.nb)
    pipe.start_epoch(sched, 0)
    pipe.enter_streams()
    for i0 in range(0, 8 * 16, 16):
        pipe.step_overlapped(i0)
    pipe.sync_streams()
    torch.cuda.synchronize()
    # the last group's rows (slot of step 7) against the features
    slot = (pipe.k - 1) % pipe.nbuf
    smp = pipe.samplers[slot]
    nf = smp.nfront[smp.L].cpu().numpy()
    rows = pipe.row_bufs[slot]
    for b in (0, 7, 15):
        ids = smp.front[smp.L][b, : nf[b]].long()
        assert torch.equal(rows[b, : nf[b], :d], feats[ids])
    assert int(pipe.pf_rows.item()) > 0
    t = pipe.totals()
    ref = WorkerPipeline(dg, store, 0, train, [15, 10, 5], 1024, 7, 16, nbuf=1)
    ref.start_epoch(sched, 0)
    for i0 in range(0, 8 * 16, 16):
        ref.step(i0)
    r = ref.totals()
    assert t["bad"] == 0 and np.array_equal(t["per_batch"][:128, :5], r["per_batch"][:128, :5])


def test_rgf1_rpb1_straight_to_device(rg, tmp_path):
    """formats.load_graph_device / load_partition_device (graph.py:219-290,
    partition.py:97-119 layouts): the file's sections land in HBM equal to
    the host loader's arrays; a sampling run on the loaded CSR equals the
    oracle; the reference's error classes for corrupt files."""
    from paper_2505_10806_b200 import formats
    from paper_2505_10806_b200.graph import GraphFormatError, GraphValidationError

    g = rg.synth_powerlaw(3000, 4, 12, 5, seed=7)
    book = rg.partition_edgecut(g, 3)
    gp, pp = tmp_path / "g.rgf1", tmp_path / "p.rpb1"
    rg.save_graph(g, gp)
    rg.save_partition(book, pp)
    dev = formats.load_graph_device(gp)
    assert torch.equal(dev.graph.indptr.cpu(), torch.from_numpy(g.indptr.astype(np.int64)))
    assert torch.equal(dev.graph.indices.cpu(), torch.from_numpy(g.indices.astype(np.int32)))
    assert torch.equal(dev.features.cpu(), torch.from_numpy(g.features))
    assert torch.equal(dev.labels.cpu(), torch.from_numpy(g.labels.astype(np.int64)))
    for m, want in ((dev.train_mask, g.train_mask), (dev.val_mask, g.val_mask),
                    (dev.test_mask, g.test_mask)):
        assert torch.equal(m.cpu(), torch.from_numpy(want))
    assert dev.graph.sorted_rows and dev.graph.max_degree == int(np.diff(g.indptr).max())
    k, owner = formats.load_partition_device(pp)
    assert k == 3 and torch.equal(owner.cpu(), torch.from_numpy(book.owner.astype(np.uint8)))
    # the device CSR drives the sampler directly
    from paper_2505_10806_b200.engine import BlockSampler

    smp = BlockSampler(dev.graph, [5, 4], 64, group=1)
    seeds = np.flatnonzero(g.train_mask)[:64]
    smp.set_seeds(0, seeds, 11)
    smp.run(1)
    fr, _ = orc.block(g.indptr, g.indices, seeds, [5, 4], 11)
    n = int(smp.nfront[2, 0].item())
    assert np.array_equal(smp.front[2][0, :n].cpu().numpy(), fr[-1])
    # corrupt files
    raw = gp.read_bytes()
    bad = tmp_path / "bad.rgf1"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(GraphFormatError):
        formats.load_graph_device(bad)
    bad.write_bytes(raw[:-10])
    with pytest.raises(OSError):
        formats.load_graph_device(bad)
    arr = bytearray(raw)
    hdr = 4 + 4 + 8 + 8 + 4 + 4
    arr[hdr + 8 * (g.num_nodes + 1): hdr + 8 * (g.num_nodes + 1) + 8] = \
        (10**9).to_bytes(8, "little")  # first neighbour id out of range
    bad.write_bytes(bytes(arr))
    with pytest.raises(GraphValidationError):
        formats.load_graph_device(bad)


def test_products_overlapped_producer_consumer_race_free(products):
    """The concurrent path end to end at Products scale: the GroupProducer
    thread samples / gathers group k+1 into the other slot while the
    consumer stream checks group k — every batch's bundle rows against the
    feature rows of its input nodes, on the device, with no host sync in the
    loop — then releases the slot for reuse.  Cross-stream slot reuse or a
    missing event would show up as mismatched rows; the per-batch accounting
    must equal a serial run's.  (compute-sanitizer is closed on this pool.)"""
    from paper_2505_10806_b200.pipeline import GroupProducer, WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule

    g, dg, store = products
    d = g.feat_dim
    feats = torch.from_numpy(g.features).cuda()
    train = np.flatnonzero(g.train_mask)
    pipe = WorkerPipeline(dg, store, 0, train, [15, 10, 5], 1024, 7, 32, nbuf=2)
    sched = SeedSchedule(7, 1, pipe.nb)
    pipe.start_epoch(sched, 0)
    bad = torch.zeros((), dtype=torch.int64, device="cuda")
    checked = torch.zeros((), dtype=torch.int64, device="cuda")
    prod = GroupProducer(pipe, range(0, pipe.nb, pipe.G))
    try:
        while (item := prod.next_group()) is not None:
            i0, ng, slot, nf = item
            smp, rows = pipe.samplers[slot], pipe.row_bufs[slot]
            L = smp.L
            valid = (torch.arange(smp.caps[L], device="cuda")[None, :]
                     < smp.nfront[L, :ng].long()[:, None])
            ids = smp.front[L][:ng].long()[valid]
            bad += (rows[:ng, :, :d][valid] != feats[ids]).any(dim=1).sum()
            checked += valid.sum()
            prod.release(slot)
    finally:
        prod.close()
    torch.cuda.synchronize()
    conc = pipe.totals()
    assert int(bad.item()) == 0
    assert int(checked.item()) == 1_126_570_328  # every input row of the epoch
    ref = WorkerPipeline(dg, store, 0, train, [15, 10, 5], 1024, 7, 32, nbuf=1)
    ref.start_epoch(sched, 0)
    for i0 in range(0, ref.nb, ref.G):
        ref.step(i0)
    assert np.array_equal(conc["per_batch"][:, :5], ref.totals()["per_batch"][:, :5])
