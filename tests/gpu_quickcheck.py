"""Quick device-vs-oracle check (run on a GPU box): python tests/gpu_quickcheck.py"""

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from oracle import gnn_oracle as orc  # noqa: E402
import paper_2505_10806_b200 as rg  # noqa: E402


def check_block(g, seeds, fanouts, s, tag):
    t = time.time()
    b = rg.sample_block(g, seeds, fanouts, s)
    t1 = time.time() - t
    fr, ed = orc.block(g.indptr, g.indices, seeds, fanouts, s)
    ok = all(np.array_equal(a, c) for a, c in zip(b.frontiers, fr))
    ok = ok and all(np.array_equal(a[0], c[0]) and np.array_equal(a[1], c[1])
                    for a, c in zip(b.edges, ed))
    print(f"{tag}: {'OK' if ok else 'MISMATCH'}  |in|={len(b.input_nodes)} t={t1:.3f}s", flush=True)
    if not ok:
        for d, (a, c) in enumerate(zip(b.frontiers, fr)):
            print("  front", d, len(a), len(c), np.array_equal(a, c))
        for d, (a, c) in enumerate(zip(b.edges, ed)):
            print("  edges", d, len(a[0]), len(c[0]), np.array_equal(a[0], c[0]),
                  np.array_equal(a[1], c[1]))
    return ok


def main():
    ok = True
    g = rg.synth_powerlaw(1000, 5, 8, 4, 7)
    ok &= check_block(g, np.arange(10), [3, 5], 99, "small")
    ok &= check_block(g, np.array([0, 5, 9]), [200, 200], 7, "full")
    ok &= check_block(g, np.arange(40), [40, 48], 5, "wide")
    ok &= check_block(g, np.array([3, 3, 7, 1, 7]), [2, 3], 13, "dups")
    g2 = rg.synth_powerlaw(20000, 5, 32, 8, 7)
    rng = np.random.default_rng(1)
    for k in range(3):
        ok &= check_block(g2, rng.choice(20000, 512, replace=False), [10, 25], int(rng.integers(2**63)),
                          f"replay{k}")
    g3 = rg.synth_powerlaw(200000, 13, 16, 4, 7)
    for k in range(2):
        ok &= check_block(g3, rng.choice(200000, 1024, replace=False), [15, 10, 5],
                          int(rng.integers(2**63)), f"p-like{k}")
    # bundle
    book = rg.partition_edgecut(g2, 2)
    shards = [rg.StoreShard(p, np.flatnonzero(book.owner == p), g2.features[book.owner == p])
              for p in range(2)]
    client = rg.StoreClient(book.owner, [rg.InprocTransport(s) for s in shards], g2.feat_dim)
    blk = rg.sample_block(g2, np.arange(512), [10, 25], 3)
    acct = rg.TransferAccount()
    remote = blk.input_nodes[book.owner[blk.input_nodes] != 0]
    cache = rg.build_steady(remote[::3], client)
    bun = rg.assemble_bundle(blk, book.owner, 0, shards[0], client, cache, acct)
    exp = orc.route_counts(blk.input_nodes, book.owner, 0, remote[::3])
    got = (bun.n_local, bun.n_cache_hit, bun.n_fallback, acct.rpc_calls)
    rows_ok = np.array_equal(bun.rows, g2.features[blk.input_nodes])
    print("bundle", got, exp, rows_ok, flush=True)
    ok &= rows_ok and got == exp
    print("ALL OK" if ok else "FAILURES")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
