"""Per-batch GPU cost of the graph-captured training step (model.GraphTrainer)
at Products shape: replays of one slot's 32 batch graphs, CUDA-event timed;
run under ncu for the per-kernel split.

  python tools/train_probe.py [--reps 3]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import paper_2505_10806_b200 as rg
    from paper_2505_10806_b200 import model
    from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore
    from paper_2505_10806_b200.pipeline import WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule

    torch.backends.cuda.matmul.allow_tf32 = False
    g = rg.synth_powerlaw(2_449_029, 13, 100, 47, 7)
    book = rg.partition_edgecut(g, 8)
    dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
    st = FeatureStore(book.owner, 8, 100)
    ids = [np.flatnonzero(book.owner == q) for q in range(8)]
    for q in range(8):
        st.set_shard(q, FeatureStore.pad_rows(g.features[ids[q]], st.src_stride, dg.device))
    st.build_route(ids)
    pipe = WorkerPipeline(dg, st, 0, np.flatnonzero(g.train_mask), [15, 10, 5], 1024, 7, 32,
                          nbuf=1)
    pipe.start_epoch(SeedSchedule(7, 1, pipe.nb), 0)
    ng = pipe.step(0)
    labels = torch.from_numpy(np.asarray(g.labels)).cuda()
    tr = model.GraphTrainer(model.init_params(100, 32, 47, 3, 1234), labels, 100, g.num_nodes,
                            0.05)
    for b in range(ng):
        tr.step(pipe.sampler, pipe.rows, b)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        for b in range(ng):
            tr.step(pipe.sampler, pipe.rows, b)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / (a.reps * ng)
    print(json.dumps({"ms_per_batch_gpu": ms, "batches_per_s": 1e3 / ms, "captures": tr.captures,
                      "loss_sum": float(tr.loss_sum.item())}))


if __name__ == "__main__":
    main()
