"""A small workload that touches every product kernel once, for
compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):

  compute-sanitizer --tool memcheck python tools/sanitize_step.py

The smoke (sample_block + assemble_bundle with a hot cache), two
overlapped pipeline steps with the group prefetch (a "peer" shard read
through the prefetch path) and slot reuse across streams, the plan pass
(counts, histogram, threshold select, cache fill), the PRNG-variant and
fanout > 32 sampler paths, and one trained group through the GroupProducer
(positions, aggregation forward / backward, radix transpose).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import __graft_entry__
    import paper_2505_10806_b200 as rg
    from paper_2505_10806_b200 import model
    from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore
    from paper_2505_10806_b200.pipeline import GroupProducer, WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule

    __graft_entry__.smoke()
    g = rg.synth_powerlaw(20000, 5, 12, 4, seed=7)
    book = rg.partition_edgecut(g, 2)
    dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
    st = FeatureStore(book.owner, 2, g.feat_dim)
    ids = [np.flatnonzero(book.owner == q) for q in range(2)]
    shards = [FeatureStore.pad_rows(g.features[i], st.src_stride, dg.device) for i in ids]
    st.set_shard(0, shards[0])
    st.set_shard(1, None, base=shards[1].data_ptr())
    st.build_route(ids)
    train = np.flatnonzero(g.train_mask)
    pipe = WorkerPipeline(dg, st, 0, train, [10, 25], 256, 7, 4, nbuf=2)
    pipe.enable_prefetch()
    sched = SeedSchedule(7, 2, pipe.nb)
    counts = pipe.count_epoch(sched, 0)
    hot = pipe.select_hot(counts, 500, pipe.nb)
    pipe.build_cache(hot)
    pipe.start_epoch(sched, 0)
    pipe.enter_streams()
    for i0 in (0, 4, 8):
        pipe.step_overlapped(i0)
    pipe.sync_streams()
    torch.cuda.synchronize()
    for prng in ("pcg32", "sfc64", "xoshiro256pp", "splitmix"):
        rg.sample_block(g, train[:64], [40, 5], 3, prng=prng)  # fanout > 32: CTA path
    # one trained group through the producer (aggregation kernels, transpose)
    pipe2 = WorkerPipeline(dg, st, 0, train, [10, 25], 256, 7, 4, nbuf=2)
    pipe2.build_cache(hot)
    pipe2.start_epoch(sched, 1)
    labels = torch.from_numpy(np.asarray(g.labels)).cuda()
    params = model.init_params(g.feat_dim, 16, 4, 2, 5)
    prod = GroupProducer(pipe2, [0, 4])
    while (item := prod.next_group()) is not None:
        i0, ng, slot, nf = item
        smp = pipe2.samplers[slot]
        for b in range(ng):
            blk = model.block_from_slot(smp, b, nf[:, b])
            rows = pipe2.row_bufs[slot][b, : int(nf[smp.L, b]), : g.feat_dim]
            loss, grads = model.loss_and_grad(blk, rows, labels, params)
            params = model.sgd_step(params, grads, 0.05)
        prod.release(slot)
    prod.close()
    torch.cuda.synchronize()
    print("sanitize workload ok", float(loss))


if __name__ == "__main__":
    main()
