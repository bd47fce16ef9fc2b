"""Products-scale goldens from the REFERENCE implementation (build container only).

Pins, at the metric's own configuration (BASELINE.json configs[2]: Products
shape, synth_powerlaw(2449029, 13, 100, 47, seed=7), partition_edgecut(k=8),
batch 1024, fanouts [15, 10, 5], s0 = 7, one epoch), the outputs the
reference itself computes for:

  * every batch's input_nodes (blake2b-128 per batch, and the reference's own
    plan digest, plan.py:84-104, over the whole epoch);
  * collect_access (plan.py:117-130): the all-node table (my_part = -1) and
    worker 0's table, hashed, with totals;
  * top_hot (plan.py:133-141) at n_hot = int(N * pct / 100.0)
    (train.py:165-168) for pct in {5, 10, 15, 20, 65}: hashes, and worker 0's
    15 % set itself (the bench's reference arm serves its cache from it);
  * per-batch assemble_bundle accounting (prefetch.py:41-88 with
    cache.lookup and StoreClient._pull): (n_local, n_hit, n_fallback, rpcs)
    for worker 0 at pct in {0 (uncached), 5, 10, 15, 20, 65}.

It imports gnnpipe from /root/reference and calls the reference functions
themselves; batches are sampled by 8 forked processes (the reference's
sample_block takes ~3 s per Products batch on one core).  Outputs:
tests/golden/products.json and tests/golden/products_w0.npz.  Nothing on the
GPU box reads /root/reference; tests read only these committed files.

  python tests/golden/make_golden_products.py   (~40 min on 8 cores)
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from gnnpipe.cache import build_steady  # noqa: E402
from gnnpipe.graph import synth_powerlaw  # noqa: E402
from gnnpipe.partition import partition_edgecut  # noqa: E402
from gnnpipe.plan import BatchPlan, FrequencyTable, collect_access, top_hot  # noqa: E402
from gnnpipe.prefetch import assemble_bundle  # noqa: E402
from gnnpipe.sampler import SeedSchedule, epoch_batches, sample_block, seed_for  # noqa: E402
from gnnpipe.store import InprocTransport, StoreClient, StoreShard, TransferAccount  # noqa: E402

OUT = Path(__file__).resolve().parent
TMP = Path(os.environ.get("PGOLD_TMP", "/tmp/pgold"))
N, M, D, C, S0 = 2_449_029, 13, 100, 47, 7
K, B, FANOUTS = 8, 1024, [15, 10, 5]
PCTS = [5, 10, 15, 20, 65]
W = 8

_G = {}


def h16(*arrays) -> str:
    m = hashlib.blake2b(digest_size=16)
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def _sample(r: int) -> int:
    g, batches, sched = _G["g"], _G["batches"], _G["sched"]
    n = 0
    for i in range(r, len(batches), W):
        f = TMP / f"in_{i:05d}.npy"
        if f.exists():
            continue
        blk = sample_block(g, batches[i], FANOUTS, seed_for(sched, 0, i), 0, i)
        np.save(TMP / f"tmp_{i:05d}.npy", blk.input_nodes.astype(np.int32))
        os.replace(TMP / f"tmp_{i:05d}.npy", f)
        n += 1
    return n


def _account(pct: int):
    """Worker 0's per-batch bundle accounting with the reference's own
    assemble_bundle / FeatureCache / StoreClient (d = 1 rows: the accounting
    does not depend on d; bytes = 4 d n is scaled afterwards)."""
    g, book, inputs, hot = _G["g"], _G["book"], _G["inputs"], _G["hot"][pct] if pct else None
    owner = book.owner
    shards = []
    for q in range(K):
        owned = np.flatnonzero(owner == q)
        shards.append(StoreShard(q, owned, g.features[owned, :1]))
    client = StoreClient(owner, [InprocTransport(s) for s in shards], 1)
    cache = build_steady(hot, client, TransferAccount()) if pct else None
    acc = TransferAccount()
    out = np.zeros((len(inputs), 4), dtype=np.int64)
    for i, ids in enumerate(inputs):
        r0 = acc.rpc_calls
        blk = SimpleNamespace(input_nodes=ids.astype(np.int64), epoch=0, batch=i)
        b = assemble_bundle(blk, owner, 0, shards[0], client, cache, acc)
        out[i] = (b.n_local, b.n_cache_hit, b.n_fallback, acc.rpc_calls - r0)
    hits = cache.hits if cache is not None else 0
    misses = cache.misses if cache is not None else 0
    return pct, out, acc.snapshot(), hits, misses


def main():
    TMP.mkdir(parents=True, exist_ok=True)
    t = time.time()
    g = synth_powerlaw(N, M, D, C, S0)
    log(f"synth_powerlaw {time.time() - t:.0f}s")
    t = time.time()
    book = partition_edgecut(g, K)
    log(f"partition_edgecut {time.time() - t:.0f}s")
    train = np.flatnonzero(g.train_mask)
    nb = -(-len(train) // B)
    sched = SeedSchedule(s0=S0, epochs=1, batches_per_epoch=nb)
    batches = epoch_batches(train, B, sched, 0)
    _G.update(g=g, book=book, batches=batches, sched=sched)

    t = time.time()
    with mp.get_context("fork").Pool(W) as pool:
        done = pool.map(_sample, range(W))
    log(f"sampled {sum(done)} new batches of {nb} in {time.time() - t:.0f}s")

    # int32 halves the ~9 GB of input sets; every use below is value-based
    inputs = [np.load(TMP / f"in_{i:05d}.npy") for i in range(nb)]
    dig = hashlib.blake2b(digest_size=8)
    for i, ids in enumerate(inputs):
        dig.update(np.array([0, i], dtype="<u8").tobytes())
        dig.update(ids.astype("<u8").tobytes())
    plan = BatchPlan(graph=g, schedule=sched, fanouts=list(FANOUTS), batch_seeds=[batches],
                     input_sets=[inputs], digest=int.from_bytes(dig.digest(), "little"))
    t = time.time()
    everyone = collect_access(plan, book, -1, epoch=0)  # owner != -1: every input node
    w0 = collect_access(plan, book, 0, epoch=0)
    log(f"collect_access {time.time() - t:.0f}s")
    # worker p's table is the all-node table restricted to owner != p (counts are per id)
    keep = book.owner[everyone.ids] != 0
    assert np.array_equal(w0.ids, everyone.ids[keep]) and np.array_equal(w0.counts,
                                                                          everyone.counts[keep])
    per_worker = {}
    hot = {}
    for p in range(K):
        sel = book.owner[everyone.ids] != p
        tab = FrequencyTable(ids=everyone.ids[sel], counts=everyone.counts[sel])
        rec = {"n_remote": len(tab), "accesses": tab.total(),
               "table": h16(tab.ids.astype("<i8"), tab.counts.astype("<i8")), "hot": {}}
        for pct in PCTS:
            n_hot = int(len(tab) * pct / 100.0)
            ids = top_hot(tab, n_hot)
            rec["hot"][str(pct)] = {"n_hot": n_hot, "ids": h16(ids.astype("<i8")),
                                    "hit_accesses": int(tab.counts[np.searchsorted(tab.ids, ids)]
                                                        .sum())}
            if p == 0:
                hot[pct] = ids
        per_worker[str(p)] = rec
    log(f"top_hot {time.time() - t:.0f}s")

    _G.update(inputs=inputs, hot=hot)
    t = time.time()
    with mp.get_context("fork").Pool(len(PCTS) + 1) as pool:
        acc = pool.map(_account, [0] + PCTS)
    log(f"assemble_bundle accounting {time.time() - t:.0f}s")
    accounting = {}
    arrays = {}
    for pct, per_batch, snap, hits, misses in acc:
        accounting[str(pct)] = {"rpc_calls": snap[0], "nodes_pulled": snap[1],
                                "bytes_pulled_d100": snap[1] * D * 4, "cache_hits": hits,
                                "cache_misses": misses,
                                "per_batch": h16(per_batch.astype("<i8"))}
        arrays[f"acct_{pct}"] = per_batch.astype(np.int32)

    counts_dense = np.zeros(N, dtype=np.int32)
    counts_dense[everyone.ids] = everyone.counts
    h15 = hot[15]
    arrays["hot15_delta"] = np.diff(h15, prepend=0).astype(np.uint32)
    arrays["input_hash"] = np.frombuffer(
        b"".join(hashlib.blake2b(ids.astype("<i8").tobytes(), digest_size=16).digest()
                 for ids in inputs), dtype=np.uint8).reshape(nb, 16)
    arrays["input_len"] = np.array([len(x) for x in inputs], dtype=np.int32)
    np.savez_compressed(OUT / "products_w0.npz", **arrays)
    out = {
        "config": {"n": N, "m": M, "d": D, "classes": C, "s0": S0, "parts": K, "batch": B,
                   "fanouts": FANOUTS, "epochs": 1, "batches": nb},
        "source": "gnnpipe (reference) sample_block / collect_access / top_hot / "
                  "assemble_bundle, run by tests/golden/make_golden_products.py",
        "plan_digest": plan.digest_hex(),
        "inputs_total": int(sum(len(x) for x in inputs)),
        "all_nodes_table": {"n": len(everyone), "accesses": everyone.total(),
                            "max": int(everyone.counts.max()),
                            "table": h16(everyone.ids.astype("<i8"),
                                         everyone.counts.astype("<i8")),
                            "dense_i32": h16(counts_dense.astype("<i4"))},
        "workers": per_worker,
        "w0_accounting": accounting,
    }
    (OUT / "products.json").write_text(json.dumps(out, indent=1) + "\n")
    log("wrote", OUT / "products.json", OUT / "products_w0.npz")


if __name__ == "__main__":
    main()
