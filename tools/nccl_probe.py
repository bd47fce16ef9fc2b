"""Phase breakdown of the NCCL group-prefetch exchange (Products, G=64, no hot cache):
torchrun --nproc-per-node 2 tools/nccl_probe.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
from paper_2505_10806_b200 import multigpu
from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore
from paper_2505_10806_b200.graph import synth_powerlaw
from paper_2505_10806_b200.partition import partition_edgecut
from paper_2505_10806_b200.pipeline import WorkerPipeline
from paper_2505_10806_b200.sampler import SeedSchedule

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
g = synth_powerlaw(2449029, 13, 100, 47, 7)
book = partition_edgecut(g, 8)
dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
st = FeatureStore(book.owner, 8, 100)
ids = [np.flatnonzero(book.owner == q) for q in range(8)]
for q in range(8):
    if q % world == rank:
        st.set_shard(q, FeatureStore.pad_rows(g.features[ids[q]], st.src_stride, dg.device))
st.build_route(ids)
pipe = WorkerPipeline(dg, st, rank, np.flatnonzero(g.train_mask), [15, 10, 5], 1024, 7, 64, nbuf=1)
pipe.enable_prefetch("nccl", rank, world)
pipe.start_epoch(SeedSchedule(7, 1, pipe.nb), 0)
smp = pipe.sampler
orig = multigpu.exchange_rows
T = {}
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(); return e
def timed_exchange(ids_, dest, world_, serve, counts=None):
    e0 = ev()
    if counts is None:
        dest = dest.to(torch.int64)
        order = torch.argsort(dest, stable=True)
        send_ids = ids_[order].contiguous()
        counts = torch.bincount(dest, minlength=world_).to(torch.int64)
    else:  # already grouped by owner (pipeline: masked union per peer rank)
        send_ids = ids_.contiguous()
        counts = torch.tensor(counts, dtype=torch.int64, device=ids_.device)
    e1 = ev()
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts)
    sc = [int(x) for x in counts.tolist()]; rc = [int(x) for x in recv_counts.tolist()]
    e2 = ev()
    req = torch.empty(sum(rc), dtype=ids_.dtype, device=ids_.device)
    dist.all_to_all_single(req, send_ids, rc, sc)
    e3 = ev()
    rows = serve(req)
    e4 = ev()
    got = torch.empty((sum(sc),) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    dist.all_to_all_single(got, rows.contiguous(), sc, rc)
    e5 = ev()
    T.setdefault("list", []).append((e0, e1, e2, e3, e4, e5, sum(sc)))
    return send_ids, got
multigpu.exchange_rows = timed_exchange
for k in range(4):
    i0 = k * 64
    pipe.plan.fill(pipe.perm, 0, i0, 64)
    smp.run(64)
    torch.cuda.synchronize(); dist.barrier()
    a = ev(); pipe.prefetch_group(64, smp, 0); b = ev()
    torch.cuda.synchronize()
    e0, e1, e2, e3, e4, e5, n = T["list"][-1]
    if rank == 0:
        print(f"group {k}: total {a.elapsed_time(b):.3f} ms | sort+count {e0.elapsed_time(e1):.3f} "
              f"counts a2a+sync {e1.elapsed_time(e2):.3f} ids a2a {e2.elapsed_time(e3):.3f} "
              f"serve {e3.elapsed_time(e4):.3f} rows a2a {e4.elapsed_time(e5):.3f} "
              f"({n} rows, {n*400/ e4.elapsed_time(e5)/1e6:.0f} GB/s) pre {a.elapsed_time(e0):.3f} post {e5.elapsed_time(b):.3f}", flush=True)
dist.destroy_process_group()
