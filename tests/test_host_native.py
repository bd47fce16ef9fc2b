"""CPU tests of the native library surface: exported symbols, host entry
points (numpy-exact Philox, synth_powerlaw CSR, LDG partitioner) and the
host-side logic of the drop-in API.  No GPU needed."""

from __future__ import annotations

import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _h(a) -> str:
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=16).hexdigest()


def test_library_exports_every_declared_symbol():
    from paper_2505_10806_b200 import _lib

    lib = _lib.load()
    header = (ROOT / "include" / "rapidgnn_b200.h").read_text()
    declared = set(re.findall(r"^(?:const char\*|int|int64_t)\s+(rg_\w+)\(", header, re.M))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.exported_symbols())
    assert lib.rg_abi_version() == 2


def test_library_exports_only_the_c_abi():
    """The .so's dynamic symbol table is exactly the header's rg_* entry
    points (version script): the statically linked CUDA runtime stays
    local, so none of its cuda* entry points is re-exported."""
    import shutil
    import subprocess

    from paper_2505_10806_b200 import _lib

    if shutil.which("nm") is None:
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    names = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    header = (ROOT / "include" / "rapidgnn_b200.h").read_text()
    declared = set(re.findall(r"^(?:const char\*|int|int64_t)\s+(rg_\w+)\(", header, re.M))
    assert names == declared, sorted(names ^ declared)


def test_philox_matches_numpy():
    from paper_2505_10806_b200 import _lib

    for seed in (0, 7, 123456789):
        bg = np.random.Philox(seed)
        key = bg.state["state"]["key"]
        want = bg.random_raw(37)
        got = np.zeros(37, dtype=np.uint64)
        _lib.host_call("rg_philox_raw", int(key[0]), int(key[1]), 37, got.ctypes.data)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("name", ["small", "replay", "c1"])
def test_synth_powerlaw_matches_reference_hashes(golden, name):
    from paper_2505_10806_b200.graph import synth_powerlaw
    from paper_2505_10806_b200.partition import partition_edgecut

    rec = golden["generator"][name]
    n, m, d, c, s = rec["args"]
    g = synth_powerlaw(n, m, d, c, s)
    hh = rec["hash"]
    assert _h(g.indptr.astype("<i8")) == hh["indptr"]
    assert _h(g.indices.astype("<i4")) == hh["indices"]
    assert _h(g.features.astype("<f4")) == hh["features"]
    assert _h(g.labels.astype("<i8")) == hh["labels"]
    assert hashlib.blake2b(g.train_mask.astype("u1").tobytes() + g.val_mask.astype("u1").tobytes()
                           + g.test_mask.astype("u1").tobytes(), digest_size=16).hexdigest() \
        == hh["masks"]
    for k, want in rec["owner"].items():
        assert _h(partition_edgecut(g, int(k)).owner.astype("<i8")) == want


@pytest.mark.slow
@pytest.mark.parametrize("name", ["products"])
def test_full_size_generator_structure(golden, name):
    """Products-shape CSR + LDG owners equal the reference's at full size."""
    from paper_2505_10806_b200.graph import synth_powerlaw_csr
    from paper_2505_10806_b200 import _lib

    rec = golden["generator"][name]
    n, m, d, c, s = rec["args"]
    indptr, indices, _ = synth_powerlaw_csr(n, m, s)
    assert _h(indptr.astype("<i8")) == rec["hash"]["indptr"]
    assert _h(indices.astype("<i4")) == rec["hash"]["indices"]
    owner = np.empty(n, dtype=np.int32)
    _lib.host_call("rg_partition_edgecut", n, indptr.ctypes.data, indices.ctypes.data, 8,
                   owner.ctypes.data)
    assert _h(owner.astype("<i8")) == rec["owner"]["8"]


def test_synth_rejects_bad_args():
    from paper_2505_10806_b200.graph import synth_powerlaw

    with pytest.raises(ValueError):
        synth_powerlaw(5, 5, 2, 2, 0)


def test_seed_schedule_and_errors():
    from oracle import gnn_oracle as orc
    from paper_2505_10806_b200.sampler import SeedSchedule, seed_for

    s = SeedSchedule(s0=0, epochs=2, batches_per_epoch=3)
    assert seed_for(s, 1, 2) == orc.batch_seed(0, 1, 2)
    with pytest.raises(IndexError):
        seed_for(s, 2, 0)
    with pytest.raises(IndexError):
        seed_for(s, 0, 3)
    e, i = np.meshgrid(np.arange(50, dtype=np.uint64), np.arange(200, dtype=np.uint64),
                       indexing="ij")
    assert len(np.unique(orc.mix_v((e << np.uint64(32)) | i))) == 10_000


def test_accounting_helpers():
    from paper_2505_10806_b200.store import (LookupError_, TransferAccount, TransportError,
                                             bytes_for)

    assert bytes_for(15_000, 602) == 36_120_000
    assert bytes_for(232_965, 602) == 560_979_720
    assert bytes_for(0, 10) == 0
    a = TransferAccount()
    a.charge(2, 4, 3)
    a.charge(1, 1, 3)
    assert a.snapshot() == (3, 5, 60)
    assert issubclass(LookupError_, KeyError) and issubclass(TransportError, ConnectionError)


def test_route_table_words():
    from paper_2505_10806_b200 import _lib
    from paper_2505_10806_b200.engine import route_table

    owner = np.array([1, 0, 1, 2, 0])
    shard_ids = [np.array([1, 4]), np.array([0, 2]), np.array([3])]
    r = route_table(owner, shard_ids)
    assert (r >> _lib.RG_KIND_SHIFT).tolist() == [1, 0, 1, 2, 0]
    assert (r & _lib.RG_ROW_MASK).tolist() == [0, 0, 1, 0, 1]
    # a shard that does not hold what the owner map claims -> invalid route
    bad = route_table(np.zeros(5, dtype=np.int64), shard_ids)
    assert bad[0] == _lib.RG_ROUTE_INVALID and bad[1] != _lib.RG_ROUTE_INVALID


def test_rows_sorted_detection():
    from paper_2505_10806_b200.engine import rows_sorted

    indptr = np.array([0, 3, 5, 5, 7])
    assert rows_sorted(indptr, np.array([1, 4, 9, 0, 2, 3, 8]))
    assert not rows_sorted(indptr, np.array([1, 9, 4, 0, 2, 3, 8]))
    assert rows_sorted(np.array([0, 0]), np.array([], dtype=np.int64))


def test_partition_random_and_halo():
    from paper_2505_10806_b200.graph import from_edge_list
    from paper_2505_10806_b200.partition import (edge_cut, halo_expand, partition_edgecut,
                                                 partition_random)

    edges = [(a, b) for a in range(6) for b in range(a + 1, 6)]
    edges += [(6 + a, 6 + b) for a in range(6) for b in range(a + 1, 6)]
    g = from_edge_list(12, edges)
    book = partition_edgecut(g, 2)
    assert edge_cut(g, book.owner) == 0  # LDG puts each clique in one part
    hb = halo_expand(g, partition_random(g, 3, seed=1))
    for p, halo in enumerate(hb.halo):
        assert np.all(hb.owner[halo] != p)


def test_placement_maps():
    from paper_2505_10806_b200.multigpu import placement, workers_of

    assert placement(8, 2) == {q: q % 2 for q in range(8)}
    assert workers_of(1, 8, 4) == [1, 5]
    assert sorted(sum((workers_of(r, 8, 8) for r in range(8)), [])) == list(range(8))


def _gloo_worker(rank, world, port, out):
    import os

    import torch.distributed as dist

    from paper_2505_10806_b200 import multigpu

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class FakeStore:
        def __init__(self, k):
            self.shards = [None] * k
            self.set = {}

        def set_shard(self, q, rows, base=None):
            self.set[q] = base

    st = FakeStore(4)
    mine = {q: (bytes([q]) * 64, 16 * q) for q in range(4) if q % world == rank}
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    # resolve peer handles the way open_peer_shards does, with a fake opener
    for r, handles in enumerate(gathered):
        if r == rank:
            continue
        for q, (hb, off) in handles.items():
            st.set_shard(q, None, base=hb[0] * 1000 + off)
    out.put((rank, sorted(st.set.items())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_shard_exchange():
    """World-size-2 exchange of shard handles (the multi-GPU host protocol)."""
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # rank 0 holds shards 0, 2 and maps 1, 3 from rank 1 (and vice versa)
    assert res[0] == [(1, 1016), (3, 3048)]
    assert res[1] == [(0, 0), (2, 2032)]


def test_rgf1_rpb1_bytes_match_reference(tmp_path):
    """RGF1 / RPB1 writers produce the reference's exact bytes; loaders
    round-trip and reject corrupt containers (test_graph.py:60-111)."""
    import json

    from paper_2505_10806_b200.graph import (GraphFormatError, load_graph, save_graph,
                                             synth_powerlaw)
    from paper_2505_10806_b200.partition import load_partition, partition_edgecut, save_partition

    gold = json.loads((ROOT / "tests" / "golden" / "golden_formats.json").read_text())
    for name, rec in gold.items():
        g = synth_powerlaw(*rec["args"])
        p = tmp_path / f"{name}.rgf"
        save_graph(g, p)
        b = p.read_bytes()
        assert len(b) == rec["rgf1_len"]
        assert hashlib.blake2b(b, digest_size=16).hexdigest() == rec["rgf1_blake2b"]
        q = tmp_path / f"{name}.rpb"
        book = partition_edgecut(g, 2)
        save_partition(book, q)
        assert hashlib.blake2b(q.read_bytes(), digest_size=16).hexdigest() == rec["rpb1_blake2b"]
        g2 = load_graph(p)
        for f in ("indptr", "indices", "features", "labels", "train_mask", "val_mask",
                  "test_mask"):
            assert np.array_equal(getattr(g2, f), getattr(g, f))
        assert np.array_equal(load_partition(q).owner, book.owner)
    bad = tmp_path / "bad.rgf"
    bad.write_bytes(b"XXXX" + p.read_bytes()[4:])
    with pytest.raises(GraphFormatError):
        load_graph(bad)
    bad.write_bytes(p.read_bytes()[:100])
    with pytest.raises(OSError):
        load_graph(bad)


def _gloo_exchange_worker(rank, world, port, out):
    import os

    import torch
    import torch.distributed as dist

    from paper_2505_10806_b200.multigpu import exchange_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r owns ids with id % world == r; asks for a rank-dependent set
    ids = torch.tensor([7, 2, 9, 4, 11, 0, 5] if rank == 0 else [1, 8, 3, 6, 10],
                       dtype=torch.int32)
    dest = ids.to(torch.int64) % world

    def serve(req):
        assert bool((req.to(torch.int64) % world == rank).all())
        r = req.to(torch.float32)
        return torch.stack([r * 10, r * 10 + 1, -r], dim=1)

    send_ids, rows = exchange_rows(ids, dest, world, serve)
    ok = bool(torch.equal(rows[:, 0], send_ids.to(torch.float32) * 10)) and \
        bool(torch.equal(rows[:, 2], -send_ids.to(torch.float32)))
    out.put((rank, ok, sorted(send_ids.tolist()) == sorted(ids.tolist()),
             send_ids.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_row_exchange():
    """NCCL-transport host protocol (multigpu.exchange_rows) on 2 gloo ranks:
    every requested id comes back with its owner's row, grouped by owner."""
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (ok, same, order) for r, ok, same, order in (q.get(timeout=120) for _ in range(2))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        ok, same, order = res[r]
        assert ok and same
        owners = [i % 2 for i in order]
        assert owners == sorted(owners)  # grouped by owner rank, stable


def test_device_path_has_no_cpu_fallback(monkeypatch):
    """The product path fails loudly without a GPU or without the extension:
    no silent host or oracle fallback (the tier's parity rule)."""
    import torch

    from paper_2505_10806_b200 import _lib
    import paper_2505_10806_b200 as rg

    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    g = rg.synth_powerlaw(200, 3, 4, 3, 1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rg.sample_block(g, np.array([0, 5, 9]), [3, 2], 11)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.call("rg_mix64", None, None, 0, None)
    # a missing shared library is an import-time error, not a fallback
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", ROOT / "does_not_exist.so")
    with pytest.raises(_lib.ExtensionMissing):
        _lib.load()


def test_reference_arm_runs_without_the_product_library():
    """bench.py --impl reference: the reference's CPU path on the host cores,
    inputs from the C oracle (hash-pinned), the worker-0 hot set, and the
    same `config` keys as the B200 arm; it asserts that neither the product
    package nor librapidgnn_b200.so was loaded before printing its line."""
    import json
    import subprocess
    import sys

    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert set(line["config"]) == {"workload", "batch_size", "fanouts", "partitions", "worker",
                                   "cache_pct", "n_hot", "prng"}
    assert line["config"]["n_hot"] == 7125  # int(15 % of worker 0's C1 remote nodes)
    assert line["cpu_baseline"]["kind"] == "port"


def test_shared_sampling_spans_cover_exactly_the_share():
    """Shared sampling copies a peer's share of a group as
    byte spans of the slot-major sampler buffers: emulating the copies on
    host tensors moves exactly slots [c0, c1) of every buffer (all levels'
    frontiers, counts, ELL rows, nfront entries, bitmaps) and nothing else;
    the shares of N ranks tile the group."""
    from types import SimpleNamespace

    import torch

    from paper_2505_10806_b200.pipeline import WorkerPipeline

    G, L, nw = 7, 3, 5
    caps, fan = [4, 12, 40, 90], [2, 3, 2]

    def sampler(fill):
        g = torch.Generator().manual_seed(fill)
        r = lambda *shape: torch.randint(-9, 9, shape, generator=g, dtype=torch.int32)
        return SimpleNamespace(L=L, bm=r(G, nw), wpre=r(G, nw), nfront=r(L + 1, G),
                               front=[r(G, c) for c in caps],
                               ell=[r(G, caps[d] * fan[d]) for d in range(L)],
                               cnt=[r(G, caps[d]) for d in range(L)])

    def bufs(s):
        return [s.bm, s.wpre, s.nfront, *s.front, *s.ell, *s.cnt]

    for world in (2, 3, 4):
        me = SimpleNamespace(G=G, world=world)
        ranges = [WorkerPipeline._share_range(me, G, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == G
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        for c0, c1 in ranges:
            src, dst = sampler(1), sampler(2)
            before = [t.clone() for t in bufs(dst)]
            for i, off, nbytes in WorkerPipeline._share_spans(me, src, c0, c1):
                s8 = bufs(src)[i].view(-1).view(torch.uint8)
                d8 = bufs(dst)[i].view(-1).view(torch.uint8)
                d8[off:off + nbytes] = s8[off:off + nbytes]
            for k, (a, b, old) in enumerate(zip(bufs(src), bufs(dst), before)):
                if k == 2:  # nfront [L+1, G]: columns are slots
                    assert torch.equal(b[:, c0:c1], a[:, c0:c1])
                    rest = torch.ones(G, dtype=torch.bool)
                    rest[c0:c1] = False
                    assert torch.equal(b[:, rest], old[:, rest])
                else:
                    assert torch.equal(b[c0:c1], a[c0:c1])
                    assert torch.equal(b[:c0], old[:c0]) and torch.equal(b[c1:], old[c1:])
