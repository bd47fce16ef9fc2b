"""K8 probe: GraphSAGE mean aggregation at Products layer 0 (the bundle's
consumer, model.py:72-81 / 126-135), timed with CUDA events; run under ncu
with -k regex:sage for the DRAM counters.

  python tools/sage_probe.py [--reps 20]

Prints one JSON line: per kernel the event-timed duration and the
algorithmic bytes (every ELL edge's source row read, self rows read, mean /
self rows written; backward: every edge's dmean row read, dself rows read,
dh rows written) as GB/s and as a fraction of the measured HBM peak.
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
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import paper_2505_10806_b200 as rg
    from paper_2505_10806_b200 import model
    from paper_2505_10806_b200.aggregate import sage_mean, sage_mean_backward, sage_positions
    from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore
    from paper_2505_10806_b200.pipeline import WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule

    g = rg.synth_powerlaw(2_449_029, 13, 100, 47, 7)
    book = rg.partition_edgecut(g, 8)
    dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
    st = FeatureStore(book.owner, 8, 100)
    ids = [np.flatnonzero(book.owner == q) for q in range(8)]
    for q in range(8):
        st.set_shard(q, FeatureStore.pad_rows(g.features[ids[q]], st.src_stride, dg.device))
    st.build_route(ids)
    pipe = WorkerPipeline(dg, st, 0, np.flatnonzero(g.train_mask), [15, 10, 5], 1024, 7, 1,
                          nbuf=1)
    pipe.start_epoch(SeedSchedule(7, 1, pipe.nb), 0)
    pipe.step(0)
    smp = pipe.sampler
    nf = smp.nfront[:, 0].cpu().numpy()
    blk = model.block_from_slot(smp, 0, nf)
    d = smp.L - 1  # model layer 0 aggregates level L-1 -> L
    src_front, dst_front = blk.frontiers[d + 1], blk.frontiers[d]
    h = pipe.rows[0, : int(nf[smp.L]), :100]
    n_src, n_dst = int(nf[d + 1]), int(nf[d])
    F = blk.step_fan[d]
    rank = torch.empty(dg.n, dtype=torch.int32, device="cuda")
    pos = sage_positions(src_front, dst_front, blk.ell[d], blk.cnt[d], F, dg.n, rank)
    edges = int(blk.cnt[d].sum().item())
    dself = torch.randn(n_dst, 100, device="cuda")
    dmean = torch.randn(n_dst, 100, device="cuda")

    def timed(fn):
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(args.reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.reps

    ms_pos = timed(lambda: sage_positions(src_front, dst_front, blk.ell[d], blk.cnt[d], F,
                                          dg.n, rank))
    ms_fwd = timed(lambda: sage_mean(h, pos, blk.cnt[d]))
    ms_bwd = timed(lambda: sage_mean_backward(dself, dmean, blk.cnt[d], pos))
    from paper_2505_10806_b200 import _lib
    nbytes = int(_lib.device().rg_sage_transpose_scratch(n_src, n_dst, F))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    toff = torch.empty(n_src + 1, dtype=torch.int32, device="cuda")
    tdst = torch.empty(n_dst * F, dtype=torch.int32, device="cuda")
    ms_tr = timed(lambda: _lib.call("rg_sage_transpose", pos.epos.data_ptr(), blk.cnt[d].data_ptr(),
                                    n_dst, F, n_src, toff.data_ptr(), tdst.data_ptr(),
                                    scratch.data_ptr(), nbytes, _lib.stream_handle()))
    seg = (toff[1:] - toff[:-1])
    longest = int(seg.max().item())
    row = 400
    fwd_bytes = edges * (row + 4) + n_dst * (row + 4 + 4) + 2 * n_dst * row
    bwd_bytes = edges * (row + 8) + n_dst * row + n_src * row
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    out = {"shape": {"n_src": n_src, "n_dst": n_dst, "edges": edges, "H": 100, "fanout": F},
           "positions_ms": ms_pos,
           "fwd": {"ms": ms_fwd, "bytes": fwd_bytes, "gbs": fwd_bytes / ms_fwd / 1e6,
                   "frac": fwd_bytes / ms_fwd / 1e6 / peak},
           "bwd_total": {"ms": ms_bwd, "bytes": bwd_bytes, "gbs": bwd_bytes / ms_bwd / 1e6,
                         "frac": bwd_bytes / ms_bwd / 1e6 / peak,
                         "note": "includes the radix-sort transpose and self_of"},
           "transpose_ms": ms_tr, "bwd_kernel_ms_est": ms_bwd - ms_tr,
           "longest_src_segment": longest,
           "peak_gbs": peak}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
