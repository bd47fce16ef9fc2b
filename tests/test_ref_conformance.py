"""Conformance: the reference's own hot-path test suite, restated against the
drop-in API (SURVEY.md §4 "conformance gate").

Each test names the reference test it mirrors (pkg/tests/<file>:<line>) and
checks the same property through `paper_2505_10806_b200`'s public names —
sample_block / epoch_batches / seed_for (test_sampler.py), generate_plan /
collect_access / top_hot (test_plan.py), build_steady / FeatureCache
(test_cache.py), assemble_bundle / Prefetcher incl. the rows_for_local spy
and the fault-injecting client (test_prefetch.py), and acceptance criteria
2-9 (test_acceptance.py).  The reference tree does not exist on the GPU box,
so the checks are restated here rather than imported.
"""

from __future__ import annotations

import itertools
import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
stats = pytest.importorskip("scipy.stats")


@pytest.fixture(scope="module")
def rg():
    import paper_2505_10806_b200 as rg
    from paper_2505_10806_b200 import _lib

    _lib.device()
    return rg


@pytest.fixture(scope="module")
def small(rg):
    """conftest.py:25-28: the shared 1000-node power-law graph."""
    return rg.synth_powerlaw(1000, 5, 8, 4, seed=7)


@pytest.fixture(scope="module")
def star(rg):
    """conftest.py:37-40: centre 0 with leaves 1..20."""
    return rg.from_edge_list(21, [(0, i) for i in range(1, 21)])


def _schedule(rg, s0=0, epochs=10, batches=100):
    return rg.SeedSchedule(s0=s0, epochs=epochs, batches_per_epoch=batches)


# ---------------------------------------------------------------- test_sampler.py
def test_seed_for_contract(rg):
    """test_sampler.py:15-36: deterministic, distinct across epochs, no
    collision over 100 x 1000 (e, i) pairs, IndexError outside the run."""
    s = _schedule(rg)
    assert rg.seed_for(s, 3, 7) == rg.seed_for(s, 3, 7)
    assert rg.seed_for(s, 0, 0) != rg.seed_for(s, 1, 0)
    big = _schedule(rg, epochs=100, batches=1000)
    seen = {rg.seed_for(big, e, i) for e in range(100) for i in range(1000)}
    assert len(seen) == 100_000
    tiny = _schedule(rg, epochs=2, batches=3)
    for e, i in ((2, 0), (0, 3)):
        with pytest.raises(IndexError):
            rg.seed_for(tiny, e, i)


def test_epoch_batches_contract(rg):
    """test_sampler.py:39-75: ceil batch count (153,431 / 1000 -> 154, last
    431), a single batch is a permutation, batches partition the train set,
    epochs differ, ValueError on empty train set / batch size 0."""
    out = rg.epoch_batches(np.arange(153_431), 1000, rg.SeedSchedule(1, 1, 154), 0)
    assert len(out) == 154 and len(out[-1]) == 431
    (one,) = rg.epoch_batches(np.arange(50), 100, rg.SeedSchedule(9, 1, 1), 0)
    assert sorted(one.tolist()) == list(range(50))
    train = np.arange(100, 400, 3)
    merged = np.concatenate(rg.epoch_batches(train, 16, rg.SeedSchedule(5, 2, 7), 1))
    assert len(merged) == len(train) and np.array_equal(np.sort(merged), train)
    s = rg.SeedSchedule(5, 2, 4)
    assert not np.array_equal(np.concatenate(rg.epoch_batches(np.arange(64), 16, s, 0)),
                              np.concatenate(rg.epoch_batches(np.arange(64), 16, s, 1)))
    with pytest.raises(ValueError):
        rg.epoch_batches(np.empty(0, dtype=np.int64), 10, rg.SeedSchedule(0, 1, 1), 0)
    with pytest.raises(ValueError):
        rg.epoch_batches(np.arange(5), 0, rg.SeedSchedule(0, 1, 1), 0)


def test_sample_block_properties(rg, small, star):
    """test_sampler.py:78-143: determinism; full fanout = exact 2-hop
    closure keeping every neighbour; star at fanout 2; no repeated pair;
    isolated seed kept; node-keyed draws; nested sorted frontiers; errors."""
    g = small
    a = rg.sample_block(g, np.arange(10), [3, 5], 99)
    b = rg.sample_block(g, np.arange(10), [3, 5], 99)
    assert np.array_equal(a.input_nodes, b.input_nodes)
    assert all(np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
               for x, y in zip(a.edges, b.edges))

    maxd = int(np.diff(g.indptr).max())
    seeds = np.array([0, 5, 9])
    blk = rg.sample_block(g, seeds, [maxd, maxd], 7)
    closure = set(seeds.tolist())
    for v in seeds:
        closure.update(g.neighbors(v).tolist())
    hop2 = set(closure)
    for v in closure:
        hop2.update(g.neighbors(v).tolist())
    assert set(blk.input_nodes.tolist()) == hop2
    src, dst = blk.edges[0]
    for v in seeds:
        assert np.array_equal(np.sort(src[dst == v]), np.sort(g.neighbors(v)))

    sblk = rg.sample_block(star, np.array([0]), [2], 17)
    s_src = sblk.edges[0][0]
    assert len(s_src) == 2 == len(set(s_src.tolist())) and all(1 <= x <= 20 for x in s_src)

    wr = rg.sample_block(g, np.arange(20), [4, 8], 3)
    for s_, d_ in wr.edges:
        assert len(set(zip(s_.tolist(), d_.tolist()))) == len(s_)

    iso = rg.from_edge_list(4, [(0, 1)])
    iblk = rg.sample_block(iso, np.array([2]), [3], 1)
    assert iblk.input_nodes.tolist() == [2] and len(iblk.edges[0][0]) == 0

    g2 = rg.from_edge_list(22, [(0, i) for i in range(1, 21)] + [(21, 1), (21, 2), (21, 3)])
    x = rg.sample_block(g2, np.array([0]), [2], 5).edges[0]
    y = rg.sample_block(g2, np.array([0, 21]), [2], 5).edges[0]
    assert np.array_equal(np.sort(x[0][x[1] == 0]), np.sort(y[0][y[1] == 0]))

    nb = rg.sample_block(g, np.arange(8), [3, 5], 11)
    for inner, outer in zip(nb.frontiers, nb.frontiers[1:]):
        assert np.isin(inner, outer).all()
    assert np.array_equal(nb.input_nodes, np.unique(nb.input_nodes))

    with pytest.raises(ValueError):
        rg.sample_block(g, np.array([], dtype=np.int64), [3], 0)
    with pytest.raises(ValueError):
        rg.sample_block(g, np.array([0]), [], 0)


def test_sampler_statistics(rg, star):
    """test_sampler.py:146-166 / criterion 8(a): uniform leaf marginals at
    fanout 5 (chi-square over 10^4 seeds) and independence of consecutive
    seeds (contingency over 2 x 10^4)."""
    picks = [rg.sample_block(star, np.array([0]), [5], s).edges[0][0] for s in range(20_000)]
    counts = np.bincount(np.concatenate(picks[:10_000]) - 1, minlength=20)
    assert stats.chisquare(counts)[1] > 0.01
    sel = [1 in p for p in picks]
    table = np.zeros((2, 2), dtype=np.int64)
    for u, v in zip(sel, sel[1:]):
        table[int(u), int(v)] += 1
    assert stats.chi2_contingency(table)[1] > 0.01


# ---------------------------------------------------------------- test_plan.py
@pytest.fixture(scope="module")
def plan3(rg, small):
    return rg.generate_plan(small, np.flatnonzero(small.train_mask), [3, 5], 64, 3, s0=7)


@pytest.fixture(scope="module")
def book2(rg, small):
    return rg.partition_edgecut(small, 2)


def test_generate_plan_contract(rg, small, plan3):
    """test_plan.py:20-55: stable 16-hex digest, sensitive to s0 and fanouts,
    shape, blocks re-derived equal the stored input sets, seeds inside."""
    train = np.flatnonzero(small.train_mask)
    assert rg.generate_plan(small, train, [3, 5], 64, 3, s0=7).digest == plan3.digest
    assert len(plan3.digest_hex()) == 16
    assert rg.generate_plan(small, train, [3, 5], 64, 3, s0=8).digest != plan3.digest
    assert rg.generate_plan(small, train, [3, 6], 64, 3, s0=7).digest != plan3.digest
    assert plan3.epochs == 3
    for e in range(3):
        assert plan3.num_batches(e) == -(-len(train) // 64)
        assert np.array_equal(np.sort(np.concatenate(plan3.batch_seeds[e])), train)
        for i in range(plan3.num_batches(e)):
            blk = plan3.block(e, i)
            assert np.array_equal(blk.input_nodes, plan3.input_sets[e][i])
            assert (blk.epoch, blk.batch) == (e, i)
    b0 = plan3.block(0, 0)
    assert np.isin(b0.seeds, b0.input_nodes).all()


def test_collect_access_contract(rg, small, plan3, book2):
    """test_plan.py:58-89: brute-force recount, epoch scopes sum to the
    global table, no local ids, one partition -> empty table."""
    want: dict[int, int] = {}
    for e in range(plan3.epochs):
        for ids in plan3.input_sets[e]:
            for v in ids[book2.owner[ids] != 0]:
                want[int(v)] = want.get(int(v), 0) + 1
    assert rg.collect_access(plan3, book2, 0).as_dict() == want
    merged: dict[int, int] = {}
    for e in range(3):
        for k, v in rg.collect_access(plan3, book2, 0, epoch=e).as_dict().items():
            merged[k] = merged.get(k, 0) + v
    assert merged == want
    assert (book2.owner[rg.collect_access(plan3, book2, 1).ids] != 1).all()
    one = rg.PartitionBook(k=1, owner=np.zeros(small.num_nodes, dtype=np.int64))
    f = rg.collect_access(plan3, one, 0)
    assert len(f) == 0 and f.total() == 0


def test_top_hot_contract(rg, plan3, book2):
    """test_plan.py:92-118: highest counts win, ties to the lower id,
    clamping, negative rejected, monotone in n_hot."""
    FT = rg.FrequencyTable
    assert rg.top_hot(FT(np.array([2, 5, 9, 11]), np.array([4, 1, 7, 4])), 2).tolist() == [2, 9]
    assert rg.top_hot(FT(np.array([3, 8, 12]), np.array([5, 5, 5])), 2).tolist() == [3, 8]
    small_t = FT(np.array([1, 2]), np.array([1, 2]))
    assert rg.top_hot(small_t, 10).tolist() == [1, 2] and rg.top_hot(small_t, 0).tolist() == []
    with pytest.raises(ValueError):
        rg.top_hot(FT(np.array([1]), np.array([1])), -1)
    freq = rg.collect_access(plan3, book2, 0, epoch=0)
    prev: set = set()
    for n in (5, 20, 80):
        cur = set(rg.top_hot(freq, n).tolist())
        assert prev <= cur
        prev = cur


def test_skewed_access(rg, small):
    """test_plan.py:121-132: the top 15 % of remote ids carry >= 25 % of the
    accesses on the hub-heavy generator."""
    plan = rg.generate_plan(small, np.flatnonzero(small.train_mask), [2, 3], 16, 3, s0=11)
    freq = rg.collect_access(plan, rg.partition_edgecut(small, 2), 0)
    n_hot = max(1, int(0.15 * len(freq)))
    top = np.sort(freq.counts)[::-1][:n_hot]
    assert top.sum() / freq.total() >= 0.25


# ---------------------------------------------------------------- test_cache.py
def _one_shard_client(rg, n=40, d=4, seed=3):
    feats = np.random.default_rng(seed).normal(size=(n, d)).astype(np.float32)
    shard = rg.StoreShard(0, np.arange(n, dtype=np.int64), feats)
    return feats, rg.StoreClient(np.zeros(n, dtype=np.int64), [rg.InprocTransport(shard)], d)


def test_cache_lookup_and_fill(rg):
    """test_cache.py:17-59: lookup split KAT, reassembly, empty cache,
    reuse ratio, fill charged as one bulk RPC."""
    feats, client = _one_shard_client(rg)
    c = rg.build_steady(np.array([2, 5, 9]), client)
    r = c.lookup(np.array([5, 1, 9, 30]))
    assert r.found_pos.tolist() == [0, 2] and r.missing_pos.tolist() == [1, 3]
    assert r.missing_ids.tolist() == [1, 30] and np.array_equal(r.found_rows, feats[[5, 9]])
    assert (c.hits, c.misses) == (2, 2)
    c2 = rg.build_steady(np.array([0, 7, 12]), client)
    ids = np.array([12, 3, 0, 7, 22])
    r2 = c2.lookup(ids)
    out = np.empty((len(ids), 4), np.float32)
    out[r2.found_pos] = r2.found_rows
    out[r2.missing_pos] = feats[r2.missing_ids]
    assert np.array_equal(out, feats[ids])
    c3 = rg.build_steady(np.empty(0, dtype=np.int64), client)
    r3 = c3.lookup(np.array([1, 2]))
    assert len(r3.found_pos) == 0 and r3.missing_ids.tolist() == [1, 2] and c3.misses == 2
    c4 = rg.build_steady(np.array([4]), client)
    assert c4.reuse_ratio() is None
    c4.lookup(np.array([4, 4, 6, 8]))
    assert c4.reuse_ratio() == pytest.approx(0.5)
    acct = rg.TransferAccount()
    rg.build_steady(np.array([1, 2, 3, 4, 5]), client, acct)
    assert acct.snapshot() == (1, 5, 80)


@pytest.fixture()
def two_worker(rg, small):
    g = small
    plan = rg.generate_plan(g, np.flatnonzero(g.train_mask), [3, 5], 64, 3, s0=7)
    book = rg.partition_edgecut(g, 2)
    shards = [rg.StoreShard(p, np.flatnonzero(book.owner == p), g.features[book.owner == p])
              for p in range(2)]
    client = rg.StoreClient(book.owner, [rg.InprocTransport(s) for s in shards], g.feat_dim)
    return g, plan, book, shards, client


def test_double_buffer(rg, two_worker):
    """test_cache.py:83-148: swap installs top_hot(collect_access(e+1)) with
    its real rows; swap resets counters; swap without a build is a no-op; a
    failed build keeps the steady buffer; the steady buffer serves lookups
    while a build is in flight."""
    g, plan, book, shards, client = two_worker
    c = rg.build_steady(rg.top_hot(rg.collect_access(plan, book, 0, epoch=0), 30), client)
    c.start_secondary_build(plan, 1, book, 0, 30, client)
    c.wait_secondary()
    assert c.swap() is True
    want = rg.top_hot(rg.collect_access(plan, book, 0, epoch=1), 30)
    assert np.array_equal(c.hot_ids, want)
    assert np.array_equal(c.lookup(want).found_rows, g.features[want])

    c = rg.build_steady(np.array([0, 1]), client)
    c.lookup(np.array([0, 5]))
    c.start_secondary_build(plan, 1, book, 0, 10, client)
    assert c.swap() is True and (c.hits, c.misses) == (0, 0)

    c = rg.build_steady(np.array([3, 4]), client)
    assert c.swap() is False and c.hot_ids.tolist() == [3, 4]

    class Boom:
        feat_dim = g.feat_dim

        def vector_pull(self, ids, account=None):
            raise ConnectionError("injected")

    c = rg.build_steady(np.array([3, 4]), client)
    c.start_secondary_build(plan, 1, book, 0, 10, Boom())
    c.wait_secondary()
    assert c.swap() is False and c.hot_ids.tolist() == [3, 4]

    gate = threading.Event()

    class Slow:
        feat_dim = g.feat_dim

        def vector_pull(self, ids, account=None):
            gate.wait(timeout=5)
            return client.vector_pull(ids, account)

    c = rg.build_steady(np.array([2, 6]), client)
    c.start_secondary_build(plan, 1, book, 0, 10, Slow())
    r = c.lookup(np.array([2, 6]))
    assert len(r.found_pos) == 2 and np.array_equal(r.found_rows, g.features[[2, 6]])
    gate.set()
    c.wait_secondary()
    assert c.swap() is True


# ---------------------------------------------------------------- test_prefetch.py
@pytest.fixture()
def pf_setup(rg, small):
    g = small
    plan = rg.generate_plan(g, np.flatnonzero(g.train_mask), [3, 5], 64, 2, s0=7)
    owner = rg.partition_edgecut(g, 2).owner
    shards = [rg.StoreShard(p, np.flatnonzero(owner == p), g.features[owner == p])
              for p in range(2)]
    client = rg.StoreClient(owner, [rg.InprocTransport(s) for s in shards], g.feat_dim)
    return g, plan, owner, shards[0], client


def test_assemble_bundle_contract(rg, pf_setup):
    """test_prefetch.py:31-69: rows = feature rows; a 5-row cache splits the
    remote traffic; a full cache means zero fallback and a clean account;
    local rows cost no RPC (the worker's own shard is never contacted)."""
    g, plan, owner, shard, client = pf_setup
    blk = plan.block(0, 0)
    b = rg.assemble_bundle(blk, owner, 0, shard, client, None, None)
    assert np.array_equal(b.rows, g.features[blk.input_nodes])
    assert b.n_local + b.n_fallback == len(blk.input_nodes) and b.n_cache_hit == 0
    remote = blk.input_nodes[owner[blk.input_nodes] != 0]
    acct = rg.TransferAccount()
    b = rg.assemble_bundle(blk, owner, 0, shard, client, rg.build_steady(remote[:5], client),
                           acct)
    assert np.array_equal(b.rows, g.features[blk.input_nodes])
    assert b.n_cache_hit == 5 and b.n_fallback == len(remote) - 5
    assert acct.nodes_pulled == b.n_fallback
    acct = rg.TransferAccount()
    b = rg.assemble_bundle(blk, owner, 0, shard, client, rg.build_steady(remote, client), acct)
    assert b.n_fallback == 0 and acct.snapshot() == (0, 0, 0)
    blk1 = plan.block(0, 1)
    acct = rg.TransferAccount()
    rg.assemble_bundle(blk1, owner, 0, shard, client, None, acct)
    assert acct.nodes_pulled == int((owner[blk1.input_nodes] != 0).sum())
    assert shard.rpc_calls == 0


def test_prefetcher_contract(rg, pf_setup):
    """test_prefetch.py:72-145: in order and complete, exhausted stays
    exhausted; bundles equal synchronous assembly; bounded run-ahead seen
    through a rows_for_local spy (<= depth + 1 assembled); start_batch;
    producer errors surface as PrefetchError with the batch index (a
    fault-injecting client); drain idempotent; depth < 1 rejected."""
    g, plan, owner, shard, client = pf_setup
    pf = rg.Prefetcher(plan, 0, owner, 0, shard, client, None, None, depth=3)
    seen = []
    while (b := pf.next_bundle()) is not None:
        seen.append(b.batch)
    assert seen == list(range(plan.num_batches(0))) and pf.next_bundle() is None

    pf = rg.Prefetcher(plan, 0, owner, 0, shard, client, None, None, depth=2)
    i = 0
    while (b := pf.next_bundle()) is not None:
        ref = rg.assemble_bundle(plan.block(0, i), owner, 0, shard, client, None, None)
        assert np.array_equal(b.rows, ref.rows)
        i += 1

    calls = []
    orig = shard.rows_for_local

    def spy(ids):
        calls.append(1)
        return orig(ids)

    shard.rows_for_local = spy
    try:
        pf = rg.Prefetcher(plan, 0, owner, 0, shard, client, None, None, depth=2)
        deadline = time.monotonic() + 5
        while len(calls) < 3 and time.monotonic() < deadline:
            time.sleep(0.01)
        time.sleep(0.2)
        assert 1 <= len(calls) <= 3
        pf.drain()
    finally:
        del shard.rows_for_local
    assert shard.rows_for_local == orig

    pf = rg.Prefetcher(plan, 0, owner, 0, shard, client, None, None, depth=2, start_batch=2)
    assert pf.next_bundle().batch == 2
    pf.drain()

    class Boom:
        def sync_pull(self, ids, account=None):
            raise ConnectionError("injected")

    pf = rg.Prefetcher(plan, 0, owner, 0, shard, Boom(), None, None, depth=2)
    with pytest.raises(rg.PrefetchError) as exc:
        while pf.next_bundle() is not None:
            pass
    assert exc.value.batch == 0
    pf.drain()

    pf = rg.Prefetcher(plan, 0, owner, 0, shard, client, None, None, depth=1)
    pf.next_bundle()
    pf.drain()
    pf.drain()
    assert pf.next_bundle() is None
    with pytest.raises(ValueError):
        rg.Prefetcher(plan, 0, owner, 0, shard, client, None, None, depth=0)


def test_injected_latency_is_charged_per_request(rg, small):
    """store.py:73-74: a shard with latency_ms sleeps once per request it
    serves; a bundle that pulls from one remote owner pays one latency."""
    g = small
    owner = rg.partition_edgecut(g, 2).owner
    shards = [rg.StoreShard(p, np.flatnonzero(owner == p), g.features[owner == p],
                            latency_ms=50.0 if p == 1 else 0.0) for p in range(2)]
    client = rg.StoreClient(owner, [rg.InprocTransport(s) for s in shards], g.feat_dim)
    blk = rg.sample_block(g, np.arange(32), [3, 5], 1)
    rg.assemble_bundle(blk, owner, 0, shards[0], client, None, None)  # warm
    t = time.perf_counter()
    rg.assemble_bundle(blk, owner, 0, shards[0], client, None, rg.TransferAccount())
    assert time.perf_counter() - t >= 0.05
    assert shards[1].rpc_calls == 2 and shards[0].rpc_calls == 0


# ---------------------------------------------------------------- test_acceptance.py
REPLAY = dict(gen_nodes=20_000, gen_edges_per_node=5, feat_dim=32, num_classes=8, partitions=2,
              epochs=5, batch_size=512, fanouts=[10, 25], s0=7)


@pytest.fixture(scope="module")
def replay_runs(rg, tmp_path_factory):
    out = {}
    for tag, over in (("rapid_a", {}), ("rapid_b", {}), ("baseline", {"mode": "baseline"}),
                      ("hot0", {"n_hot": 0}), ("hot1", {"n_hot_pct": 1.0}),
                      ("hot5", {"n_hot_pct": 5.0})):
        kw = dict(REPLAY, **over)
        path = tmp_path_factory.mktemp(tag) / "m.csv"
        res = rg.run(rg.RunConfig(metrics_out=str(path), **kw))
        out[tag] = (res, [str(path).replace("m.csv", f"m.w{p}.csv") for p in range(2)])
    return out


def _csv_wo_time(path):
    rows = open(path).read().splitlines()
    drop = rows[0].split(",").index("t_e_ms")
    return [[c for i, c in enumerate(r.split(",")) if i != drop] for r in rows]


def test_criteria_2_to_5(replay_runs):
    """test_acceptance.py:93-163: (2) determinism replay — digests and CSV
    columns identical; (3) rapid and baseline end with identical loss,
    accuracy and parameters; (4)/(5) the pinned REPLAY pull volumes and
    reuse (the reference log's values: criterion 4 and 5 FAIL by design,
    test_output.txt:196,215 — here we pin the numbers themselves)."""
    ra, ca = replay_runs["rapid_a"]
    rb, cb = replay_runs["rapid_b"]
    assert all(x.plan_digest == y.plan_digest for x, y in zip(ra, rb))
    assert all(_csv_wo_time(x) == _csv_wo_time(y) for x, y in zip(ca, cb))
    base, _ = replay_runs["baseline"]
    for x, y in zip(ra, base):
        assert [r.loss for r in x.records] == [r.loss for r in y.records]
        assert [r.train_acc for r in x.records] == [r.train_acc for r in y.records]
        for p, q in zip(x.params, y.params):
            assert torch.equal(p.w_self, q.w_self) and torch.equal(p.w_neigh, q.w_neigh)
            assert torch.equal(p.bias, q.bias)

    def pulls(res):
        return [sum(r.records[e].nodes_pulled for r in res) for e in range(5)]

    assert pulls(ra) == [326975, 326783, 326665, 326985, 327409]  # test_output.txt:196
    assert pulls(base) == [406701, 406553, 406308, 406717, 407090]
    totals = [sum(pulls(replay_runs[k][0])) for k in ("hot0", "hot1", "hot5")] + [sum(pulls(ra))]
    assert totals == [2033369, 2005369, 1895799, 1634817]
    assert all(a >= b for a, b in zip(totals, totals[1:]))

    def reuse(res):
        v = [r.reuse_ratio for w in res for r in w.records if r.reuse_ratio is not None]
        return float(np.mean(v))

    assert round(reuse(replay_runs["hot1"][0]), 3) == 0.014  # test_output.txt:215
    assert round(reuse(ra), 3) == 0.196


def test_criterion_6_latency_hiding(rg):
    """test_acceptance.py:172-184: at 5 ms per pull the rapid run (100 % hot
    set, prefetcher) is >= 1.5x faster per mid epoch than baseline."""
    kw = dict(gen_nodes=3000, gen_edges_per_node=3, feat_dim=16, num_classes=4, partitions=2,
              epochs=5, batch_size=32, fanouts=[5, 10], latency_ms=5.0, prefetch_depth=3,
              hidden_dim=16, s0=7, n_hot_pct=100.0)
    base = rg.run(rg.RunConfig(mode="baseline", **kw))
    rapid = rg.run(rg.RunConfig(mode="rapid", **kw))

    def mid(res):
        return float(np.mean([[w.records[e].t_e_ms for w in res] for e in range(1, 4)]))

    assert mid(rapid) <= 0.67 * mid(base), (mid(rapid), mid(base))


def test_criterion_7_gradients_fd(rg):
    """test_acceptance.py:186-253: the device model's analytic gradient vs
    central finite differences (f64) on random small graphs, max relative
    error <= 1e-6."""
    from paper_2505_10806_b200 import model
    from paper_2505_10806_b200.aggregate import edges_to_ell

    rng = np.random.default_rng(2024)
    for k in range(3):
        n = int(rng.integers(10, 51))
        edges = [(int(rng.integers(n)), int(rng.integers(n))) for _ in range(int(rng.integers(n, 3 * n)))]
        edges = [(a, b) for a, b in edges if a != b]
        g = rg.from_edge_list(n, edges, feat_dim=6, num_classes=3,
                              features=rng.normal(size=(n, 6)).astype(np.float32),
                              labels=rng.integers(0, 3, size=n))
        blk = rg.sample_block(g, np.sort(rng.choice(n, size=min(8, n), replace=False)), [3, 4],
                              int(rng.integers(1 << 30)))
        L = blk.num_layers
        ells, cnts, fans = [], [], []
        for d in range(L):
            ell, cnt, F = edges_to_ell(blk.frontiers[d], *blk.edges[d])
            ells.append(torch.from_numpy(ell).cuda())
            cnts.append(torch.from_numpy(cnt).cuda())
            fans.append(F)
        dblk = model.DeviceBlock([torch.from_numpy(f.astype(np.int32)).cuda() for f in blk.frontiers],
                                 ells, cnts, fans, n)
        rows = torch.from_numpy(g.features[blk.input_nodes].astype(np.float64)).cuda()
        labels = torch.from_numpy(np.asarray(g.labels)).cuda()
        params = model.init_params(6, 10, 3, 2, seed=k, dtype=torch.float64)
        _, grads = model.loss_and_grad(dblk, rows, labels, params)
        flat = torch.cat([torch.cat([p.w_self.ravel(), p.w_neigh.ravel(), p.bias.ravel()])
                          for p in params])
        gflat = torch.cat([torch.cat([p.w_self.ravel(), p.w_neigh.ravel(), p.bias.ravel()])
                           for p in grads])

        def loss_at(vec):
            out, i = [], 0
            for p in params:
                parts = []
                for a in (p.w_self, p.w_neigh, p.bias):
                    parts.append(vec[i:i + a.numel()].view_as(a))
                    i += a.numel()
                out.append(model.LayerParams(*parts))
            return float(model.loss_and_grad(dblk, rows, labels, out)[0])

        worst = 0.0
        for j in rng.choice(flat.numel(), size=min(40, flat.numel()), replace=False):
            tp, tm = flat.clone(), flat.clone()
            tp[j] += 1e-6
            tm[j] -= 1e-6
            num = (loss_at(tp) - loss_at(tm)) / 2e-6
            worst = max(worst, abs(float(gflat[j]) - num) / max(abs(num), 1e-3))
        assert worst <= 1e-6, worst


def test_criterion_8_exhaustive_fanout_is_unbiased(rg):
    """test_acceptance.py:256-293 (c): with exhaustive fanouts the
    batch-weighted average gradient over an epoch equals the full-batch
    gradient (f64), and small fanouts give nonzero gradient variance."""
    from paper_2505_10806_b200 import model
    from paper_2505_10806_b200.aggregate import edges_to_ell

    g = rg.synth_powerlaw(120, 3, 8, 3, seed=5)
    train = np.flatnonzero(g.train_mask)
    params = model.init_params(8, 12, 3, 2, seed=4, dtype=torch.float64)
    labels = torch.from_numpy(np.asarray(g.labels)).cuda()
    maxd = int(np.diff(g.indptr).max())

    def grad_of(blk):
        ells, cnts, fans = [], [], []
        for d in range(blk.num_layers):
            ell, cnt, F = edges_to_ell(blk.frontiers[d], *blk.edges[d])
            ells.append(torch.from_numpy(ell).cuda())
            cnts.append(torch.from_numpy(cnt).cuda())
            fans.append(F)
        dblk = model.DeviceBlock([torch.from_numpy(f.astype(np.int32)).cuda()
                                  for f in blk.frontiers], ells, cnts, fans, g.num_nodes)
        rows = torch.from_numpy(g.features[blk.input_nodes].astype(np.float64)).cuda()
        _, gr = model.loss_and_grad(dblk, rows, labels, params)
        return torch.cat([torch.cat([p.w_self.ravel(), p.w_neigh.ravel(), p.bias.ravel()])
                          for p in gr])

    full = grad_of(rg.sample_block(g, train, [maxd, maxd], 0))
    avg = torch.zeros_like(full)
    for batch in rg.epoch_batches(train, 16, rg.SeedSchedule(3, 1, 6), 0):
        avg += grad_of(rg.sample_block(g, batch, [maxd, maxd], 1)) * (len(batch) / len(train))
    assert float(torch.linalg.norm(avg - full)) <= 1e-5 * float(torch.linalg.norm(full))
    sampled = torch.stack([grad_of(rg.sample_block(g, train[:16], [2, 3], s)) for s in range(6)])
    assert float(sampled.var(dim=0).sum()) > 0


def test_criterion_9_transparency(rg):
    """test_acceptance.py:310-364: cache + fallback reassembly equals a
    plain pull, bundles equal the feature rows, and top_hot equals the
    brute-force optimum with least-id ties."""
    rng = np.random.default_rng(7)
    feats = rng.normal(size=(200, 5)).astype(np.float32)
    owner = np.arange(200) % 2
    shards = [rg.StoreShard(p, np.flatnonzero(owner == p), feats[owner == p]) for p in range(2)]
    client = rg.StoreClient(owner, [rg.InprocTransport(s) for s in shards], 5)
    cache = rg.build_steady(np.sort(rng.choice(200, size=40, replace=False)), client)
    for _ in range(100):
        ids = rng.integers(0, 200, size=int(rng.integers(1, 50)))
        r = cache.lookup(ids)
        got = np.empty((len(ids), 5), np.float32)
        got[r.found_pos] = r.found_rows
        got[r.missing_pos] = client.sync_pull(r.missing_ids)
        assert np.array_equal(got, client.sync_pull(ids))
    g = rg.synth_powerlaw(400, 3, 8, 4, seed=9)
    book = rg.partition_edgecut(g, 2)
    gsh = [rg.StoreShard(p, np.flatnonzero(book.owner == p), g.features[book.owner == p])
           for p in range(2)]
    gcl = rg.StoreClient(book.owner, [rg.InprocTransport(s) for s in gsh], g.feat_dim)
    for s in range(10):
        blk = rg.sample_block(g, np.sort(rng.choice(400, 20, replace=False)), [3, 5], s)
        b = rg.assemble_bundle(blk, book.owner, 0, gsh[0], gcl, None, None)
        assert np.array_equal(b.rows, g.features[blk.input_nodes])
    for _ in range(30):
        size = int(rng.integers(1, 13))
        ids = np.sort(rng.choice(100, size=size, replace=False)).astype(np.int64)
        counts = rng.integers(1, 6, size=size).astype(np.int64)
        table = dict(zip(ids.tolist(), counts.tolist()))
        for n_hot in range(size + 1):
            chosen = tuple(rg.top_hot(rg.FrequencyTable(ids, counts), n_hot).tolist())
            combos = list(itertools.combinations(ids.tolist(), n_hot))
            best = max(sum(table[i] for i in c) for c in combos)
            assert chosen == min(c for c in combos if sum(table[i] for i in c) == best)


def test_f64_precision_runs(rg):
    """test_train.py f64 path (RunConfig.precision = "f64"): the run
    completes with finite losses, identical accounting to f32, and the
    aggregation kernels run in float64."""
    kw = dict(gen_nodes=2000, gen_edges_per_node=3, feat_dim=6, num_classes=3, partitions=2,
              epochs=2, batch_size=64, fanouts=[3, 4], hidden_dim=8)
    r32 = rg.run(rg.RunConfig(precision="f32", **kw))
    r64 = rg.run(rg.RunConfig(precision="f64", **kw))
    for a, b in zip(r32, r64):
        assert all(np.isfinite(x.loss) for x in b.records)
        assert [x.nodes_pulled for x in a.records] == [x.nodes_pulled for x in b.records]
        assert b.params[0].w_self.dtype == torch.float64
        for x, y in zip(a.records, b.records):
            assert abs(x.loss - y.loss) <= 1e-4 * max(1.0, abs(y.loss))
