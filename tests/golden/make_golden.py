"""Generate the golden fixtures from the REFERENCE implementation.

Runs only in the build container, where the reference package is mounted at
/root/reference (read-only).  It imports gnnpipe from there, records its
outputs on fixed inputs, and writes them under tests/golden/:

  small.npz    arrays: the 1000-node test graph (synth_powerlaw(1000,5,8,4,7)),
               sample_block cases, a 3-epoch plan, collect_access / top_hot
               tables, epoch permutations
  golden.json  scalars: plan digests, assemble_bundle provenance/accounting,
               run() metrics for the pinned REPLAY config
               (tests/test_acceptance.py:27-30) and config C1, content
               hashes of synth_powerlaw / partition_edgecut outputs at test,
               C1, Reddit and Products shapes

Nothing on the GPU box reads /root/reference; the tests only read these
committed files.  Re-run:  python tests/golden/make_golden.py [--no-large]
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from gnnpipe.cache import build_steady  # noqa: E402
from gnnpipe.graph import from_edge_list, synth_powerlaw  # noqa: E402
from gnnpipe.partition import partition_edgecut  # noqa: E402
from gnnpipe.plan import collect_access, generate_plan, top_hot  # noqa: E402
from gnnpipe.prefetch import assemble_bundle  # noqa: E402
from gnnpipe.sampler import SeedSchedule, epoch_batches, sample_block  # noqa: E402
from gnnpipe.store import InprocTransport, StoreClient, StoreShard, TransferAccount  # noqa: E402
from gnnpipe.train import RunConfig, run  # noqa: E402

OUT = Path(__file__).resolve().parent


def h(*arrays) -> str:
    m = hashlib.blake2b(digest_size=16)
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()


def graph_hash(g) -> dict:
    return {
        "indptr": h(g.indptr.astype("<i8")),
        "indices": h(g.indices.astype("<i4")),
        "features": h(g.features.astype("<f4")),
        "labels": h(g.labels.astype("<i8")),
        "masks": h(g.train_mask.astype("u1"), g.val_mask.astype("u1"), g.test_mask.astype("u1")),
    }


def records(results) -> list:
    out = []
    for r in results:
        out.append({
            "part": r.part,
            "digest": r.plan_digest,
            "fill": list(r.cache_fill.snapshot()),
            "epochs": [[x.rpc_calls, x.nodes_pulled, x.bytes_pulled, x.cache_hits,
                        x.cache_misses, x.reuse_ratio, x.loss, x.train_acc] for x in r.records],
        })
    return out


def sample_cases(g, star, path_g, iso):
    maxdeg = int(g.degrees().max())
    rng = np.random.default_rng(2024)
    train = np.flatnonzero(g.train_mask)
    cases = [
        ("small", np.arange(10), [3, 5], 99),
        ("full", np.array([0, 5, 9]), [maxdeg, maxdeg], 7),
        ("wr", np.arange(20), [4, 8], 3),
        ("nest", np.arange(8), [3, 5], 11),
        ("replay_fan", np.sort(rng.choice(train, 64, replace=False)), [10, 25], 0x1234567),
        ("products_fan", rng.choice(train, 64, replace=False), [15, 10, 5], 2**63 + 5),
        ("wide", np.arange(0, 40), [40, 48], 5),
        ("fan1", np.arange(100, 164), [1, 1, 1], 77),
        ("dups", np.array([3, 3, 7, 1, 7]), [2, 3], 13),
        ("hubs", np.arange(0, 6), [2, 33, 7], 2**64 - 1),
    ]
    out = {}
    meta = []
    for name, seeds, fan, s in cases:
        b = sample_block(g, seeds, fan, s)
        meta.append({"name": name, "graph": "small", "fanouts": fan, "seed": str(s),
                     "layers": b.num_layers})
        out[f"{name}_seeds"] = np.asarray(seeds, dtype=np.int64)
        for d, f in enumerate(b.frontiers):
            out[f"{name}_front{d}"] = f
        for d, (src, dst) in enumerate(b.edges):
            out[f"{name}_src{d}"] = src
            out[f"{name}_dst{d}"] = dst
    for gname, gg, seeds, fan, s in (("star", star, [0], [2], 17), ("star5", star, [0, 3], [5, 1], 9),
                                     ("path", path_g, [1], [1, 1], 4), ("iso", iso, [2], [3], 1)):
        b = sample_block(gg, np.array(seeds), fan, s)
        meta.append({"name": gname, "graph": gname.rstrip("5"), "fanouts": fan, "seed": str(s),
                     "layers": b.num_layers})
        out[f"{gname}_seeds"] = np.array(seeds, dtype=np.int64)
        for d, f in enumerate(b.frontiers):
            out[f"{gname}_front{d}"] = f
        for d, (src, dst) in enumerate(b.edges):
            out[f"{gname}_src{d}"] = src
            out[f"{gname}_dst{d}"] = dst
    return out, meta


def main(large: bool) -> None:
    t0 = time.time()
    arrays: dict[str, np.ndarray] = {}
    gold: dict = {"reference": "gnnpipe @ /root/reference/pkg (arxiv 2505.10806 desk re-creation)",
                  "numpy": np.__version__}

    g = synth_powerlaw(1000, 5, 8, 4, seed=7)
    book2 = partition_edgecut(g, 2)
    arrays.update(indptr=g.indptr, indices=g.indices, features=g.features, labels=g.labels,
                  train_mask=g.train_mask, owner2=book2.owner)
    star = from_edge_list(21, [(0, i) for i in range(1, 21)])
    path_g = from_edge_list(3, [(0, 1), (1, 2)])
    iso = from_edge_list(4, [(0, 1)])

    cases, meta = sample_cases(g, star, path_g, iso)
    arrays.update({f"case_{k}": v for k, v in cases.items()})
    gold["sample_cases"] = meta

    # epoch permutations (sampler.py:43-57)
    sch = SeedSchedule(s0=1, epochs=1, batches_per_epoch=154)
    big = epoch_batches(np.arange(153_431), 1000, sch, 0)
    gold["epoch_153431"] = {"n_batches": len(big), "last": len(big[-1]),
                            "hash": h(np.concatenate(big).astype("<i8")),
                            "head": np.concatenate(big)[:16].tolist()}
    train = np.flatnonzero(g.train_mask)
    sch3 = SeedSchedule(s0=7, epochs=3, batches_per_epoch=-(-len(train) // 64))
    for e in range(3):
        arrays[f"perm_e{e}"] = np.concatenate(epoch_batches(train, 64, sch3, e))

    # plan over the small graph (tests/test_plan.py fixture)
    plan = generate_plan(g, train, [3, 5], 64, 3, s0=7)
    gold["plan_small"] = {"digest": plan.digest_hex(), "batches": plan.num_batches(0),
                          "fanouts": [3, 5], "batch_size": 64, "epochs": 3, "s0": 7}
    for e in range(3):
        sets = plan.input_sets[e]
        arrays[f"plan_in_e{e}"] = np.concatenate(sets)
        arrays[f"plan_off_e{e}"] = np.cumsum([0] + [len(s) for s in sets])
    for p in range(2):
        for scope in (None, 0, 1, 2):
            f = collect_access(plan, book2, p, epoch=scope)
            tag = f"p{p}_{'all' if scope is None else 'e%d' % scope}"
            arrays[f"freq_ids_{tag}"] = f.ids
            arrays[f"freq_cnt_{tag}"] = f.counts
            for n_hot in (0, 1, 5, 20, 80, len(f) - 1, len(f), len(f) + 5):
                if n_hot < 0:
                    continue
                arrays[f"hot_{tag}_{n_hot}"] = top_hot(f, n_hot)

    # bundle provenance + accounting (prefetch.py:41-88)
    owner = book2.owner
    shards = [StoreShard(p, np.flatnonzero(owner == p).astype(np.int64), g.features[owner == p])
              for p in range(2)]
    client = StoreClient(owner, [InprocTransport(s) for s in shards], g.feat_dim)
    bundles = []
    for p in range(2):
        f0 = collect_access(plan, book2, p, epoch=0)
        for n_hot in (0, 30, len(f0)):
            cache = build_steady(top_hot(f0, n_hot), client, TransferAccount()) if n_hot else None
            for i in range(4):
                acct = TransferAccount()
                b = assemble_bundle(plan.block(0, i), owner, p, shards[p], client, cache, acct)
                bundles.append({"part": p, "n_hot": n_hot, "batch": i, "n_local": b.n_local,
                                "n_hit": b.n_cache_hit, "n_fallback": b.n_fallback,
                                "account": list(acct.snapshot()),
                                "hits": cache.hits if cache else 0,
                                "misses": cache.misses if cache else 0})
    gold["bundles_small"] = bundles

    # generator / partitioner content hashes
    gens = {"small": [1000, 5, 8, 4, 7], "replay": [20000, 5, 32, 8, 7],
            "c1": [100000, 10, 128, 8, 7]}
    if large:
        gens.update(reddit=[232965, 246, 602, 41, 7], products=[2449029, 13, 100, 47, 7])
    gold["generator"] = {}
    for name, (n, m, d, c, s) in gens.items():
        ts = time.time()
        gg = synth_powerlaw(n, m, d, c, s)
        rec = {"args": [n, m, d, c, s], "hash": graph_hash(gg), "num_edges": int(gg.num_edges)}
        ks = (2, 8) if name in ("small", "replay", "c1") else (8,)
        rec["owner"] = {str(k): h(partition_edgecut(gg, k).owner.astype("<i8")) for k in ks}
        rec["seconds"] = round(time.time() - ts, 1)
        gold["generator"][name] = rec
        print(f"generator {name}: {rec['seconds']} s", flush=True)
        del gg

    # pinned REPLAY runs (tests/test_acceptance.py:27-30, 60-68)
    replay = dict(gen_nodes=20_000, gen_edges_per_node=5, feat_dim=32, num_classes=8,
                  partitions=2, epochs=5, batch_size=512, fanouts=[10, 25], s0=7)
    gold["replay"] = {"config": replay}
    for label, over in (("rapid", dict(mode="rapid")), ("baseline", dict(mode="baseline")),
                        ("hot0", dict(mode="rapid", n_hot=0)),
                        ("hot1", dict(mode="rapid", n_hot_pct=1.0)),
                        ("hot5", dict(mode="rapid", n_hot_pct=5.0)),
                        ("global", dict(mode="rapid", hot_scope="global"))):
        ts = time.time()
        gold["replay"][label] = records(run(RunConfig(**replay, **over)))
        print(f"replay {label}: {time.time() - ts:.1f} s", flush=True)

    c1 = dict(gen_nodes=100_000, gen_edges_per_node=10, feat_dim=128, num_classes=8,
              partitions=2, epochs=2, batch_size=1024, fanouts=[10, 5], s0=7)
    gold["c1"] = {"config": c1}
    for label, over in (("rapid", dict(mode="rapid")), ("baseline", dict(mode="baseline"))):
        ts = time.time()
        gold["c1"][label] = records(run(RunConfig(**c1, **over)))
        print(f"c1 {label}: {time.time() - ts:.1f} s", flush=True)

    np.savez_compressed(OUT / "small.npz", **arrays)
    (OUT / "golden.json").write_text(json.dumps(gold, indent=1))
    print(f"done in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main(large="--no-large" not in sys.argv)
