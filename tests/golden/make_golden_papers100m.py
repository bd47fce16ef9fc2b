"""Pin the papers100M-shaped input structure (BASELINE.json configs[4]).

Test infrastructure.  The reference's own synth_powerlaw takes hours at
111 M nodes, so the pin goes through the C oracle (oracle/oracle_graph.c),
which tests/test_oracle_golden.py holds to the reference's content hashes at
five smaller shapes (tests/golden/golden.json "generator").  This script
runs the oracle and the product generator / partitioner at the papers100M
shape in this container, asserts they agree, and records the content hashes
(indptr, indices, train mask, LDG owner) in tests/golden/papers100m.json;
bench.py --check compares the box's inputs against them.

    python tests/golden/make_golden_papers100m.py     # ~10 min, ~30 GB RAM
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

N, M, D, C, SEED, K = 111_059_956, 7, 128, 172, 7, 8


def h(a) -> str:
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=16).hexdigest()


def hashes(indptr, indices, train_mask, owner) -> dict:
    return {"indptr": h(np.asarray(indptr, dtype="<i8")),
            "indices": h(np.asarray(indices, dtype="<i4")),
            "train_mask": h(np.asarray(train_mask, dtype="u1")),
            "owner": h(np.asarray(owner, dtype="u1"))}


def main() -> None:
    from oracle import graph_oracle as go

    t = time.time()
    og = go.synth_powerlaw(N, M, D, SEED, with_features=False)
    oown = go.partition_edgecut(og, K)
    ref = hashes(og.indptr, og.indices, og.train_mask, oown)
    t_oracle = time.time() - t
    print(f"oracle: {t_oracle:.0f} s {ref}", flush=True)
    del og, oown

    from paper_2505_10806_b200.graph import synth_powerlaw
    from paper_2505_10806_b200.partition import partition_edgecut

    t = time.time()
    g = synth_powerlaw(N, M, D, C, SEED, with_features=False, with_labels=False)
    book = partition_edgecut(g, K)
    got = hashes(g.indptr, g.indices, g.train_mask, book.owner)
    t_prod = time.time() - t
    print(f"product: {t_prod:.0f} s {got}", flush=True)
    assert got == ref, "product generator / partitioner differ from the C oracle"
    out = {"args": {"n": N, "m": M, "seed": SEED, "k": K},
           "num_edges": int(len(g.indices)), "hash": ref,
           "note": "C oracle (pinned to the reference at 5 shapes) == product, "
                   f"oracle {t_oracle:.0f} s, product {t_prod:.0f} s on the build container"}
    (Path(__file__).parent / "papers100m.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
