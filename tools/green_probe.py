"""Spatial split probe: the gather (HBM-write-bound) and the next group's
sampler (instruction-issue-bound) on disjoint SM sets through green contexts
(cuGreenCtxCreate / cuGreenCtxStreamCreate), Products G = 128 as bench.py
builds it.  Prints one JSON line: for each gather SM count X the gather alone
on X SMs, the sampler alone on the remaining SMs, and the overlapped step
(sample k+1 on one partition while gather k runs on the other).

  python tools/green_probe.py [--steps 10] [--splits 64,80,96,112]
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


def _chk(ret):
    """cuda.bindings returns (err, *values)."""
    if int(ret[0]) != 0:
        raise RuntimeError(f"driver error {ret[0]}")
    return ret[1] if len(ret) == 2 else ret[1:]


def green_streams(n_sm_a: int):
    """Two green contexts on device 0: >= n_sm_a SMs, and the rest; one
    non-blocking stream in each."""
    from cuda.bindings import driver as drv

    dev = _chk(drv.cuDeviceGet(0))
    res = _chk(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    groups, _, rem = _chk(drv.cuDevSmResourceSplitByCount(1, res, 0, n_sm_a))
    out = []
    for r in (groups[0], rem):
        desc = _chk(drv.cuDevResourceGenerateDesc([r], 1))
        g = _chk(drv.cuGreenCtxCreate(desc, dev,
                                      drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
        s = _chk(drv.cuGreenCtxStreamCreate(g, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
        out.append((int(r.sm.smCount), g, s))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--splits", default="64,80,96,112")
    a = ap.parse_args()
    import bench
    from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore
    from paper_2505_10806_b200.pipeline import WorkerPipeline, resolve_n_hot
    from paper_2505_10806_b200.plan import candidates, threshold_select
    from paper_2505_10806_b200.sampler import SeedSchedule

    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")
    cfg = bench.CONFIGS["products"]
    g, book = bench.build_inputs(cfg)
    k, d = cfg["parts"], cfg["d"]
    owner = book.owner
    dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
    store = FeatureStore(owner, k, d)
    shard_ids = [np.flatnonzero(owner == q) for q in range(k)]
    for q in range(k):
        store.set_shard(q, FeatureStore.pad_rows(g.features[shard_ids[q]], store.src_stride, dg.device))
    store.build_route(shard_ids)
    train = np.flatnonzero(g.train_mask)
    G = cfg.get("group", 128)
    pipe = WorkerPipeline(dg, store, 0, train, cfg["fanouts"], cfg["batch"], bench.S0, G, nbuf=2)
    sched = SeedSchedule(bench.S0, 1, pipe.nb)
    counts = pipe.count_epoch(sched, 0)
    _, nout, hist, bm = candidates(counts, store.owner, 0, pipe.nb)
    hot = threshold_select(counts, bm, hist.cpu().numpy().astype(np.int64),
                           resolve_n_hot(15.0, int(nout.item())))
    pipe.build_cache(hot)
    pipe.start_epoch(sched, 0)
    n_full = pipe.nb // G
    smp = pipe.samplers[0]

    def timed(fn, reps):
        fn(0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r in range(reps):
            fn(1 + r)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {"full_chip": {}}
    # reference: everything on the whole chip
    pipe.plan.fill(pipe.perm, 0, 0, G, smp)
    smp.run(G)

    def gather_only(r):
        pipe.gather(G, 0, smp, pipe.row_bufs[0], slot=0, prefetched=True)

    def sample_only(r):
        pipe.plan.fill(pipe.perm, 0, (r % n_full) * G, G, smp)
        smp.run(G)

    out["full_chip"]["gather_ms"] = timed(gather_only, a.steps)
    out["full_chip"]["sample_ms"] = timed(sample_only, a.steps)

    def overlapped(r):
        pipe.step_overlapped((r % n_full) * G)

    s_sample0, s_gather0 = pipe.s_sample, pipe.s_gather

    def overlapped_step(r):
        pipe.enter_streams()
        overlapped(r)
        pipe.sync_streams()

    def run_overlapped(reps):
        torch.cuda.synchronize()
        pipe.enter_streams()
        for r in range(3):
            overlapped(r)
        pipe.sync_streams()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.enter_streams()
        for r in range(reps):
            overlapped(3 + r)
        pipe.sync_streams()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out["full_chip"]["overlapped_step_ms"] = run_overlapped(a.steps)
    for x in [int(v) for v in a.splits.split(",")]:
        (na, ga, sa), (nb_, gb, sb) = green_streams(x)
        A = torch.cuda.ExternalStream(int(sa))
        B = torch.cuda.ExternalStream(int(sb))
        rec = {"gather_sms": na, "sample_sms": nb_}
        pipe.plan.fill(pipe.perm, 0, 0, G, smp)
        smp.run(G)
        torch.cuda.synchronize()
        with torch.cuda.stream(A):
            rec["gather_ms"] = timed(gather_only, a.steps)
        with torch.cuda.stream(B):
            rec["sample_ms"] = timed(sample_only, a.steps)
        pipe.s_sample, pipe.s_gather = B, A
        rec["overlapped_step_ms"] = run_overlapped(a.steps)
        pipe.s_sample, pipe.s_gather = s_sample0, s_gather0
        out[f"split_{x}"] = rec
        print(json.dumps(rec), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
