"""Overlap probe: Products-shape, G=32: time sampling alone, gather alone, and
sampling of group k+1 concurrently with the gather of group k (two streams)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore
from paper_2505_10806_b200.graph import synth_powerlaw
from paper_2505_10806_b200.partition import partition_edgecut
from paper_2505_10806_b200.pipeline import WorkerPipeline
from paper_2505_10806_b200.sampler import SeedSchedule

g = synth_powerlaw(2449029, 13, 100, 47, 7)
book = partition_edgecut(g, 8)
dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
st = FeatureStore(book.owner, 8, 100)
ids = [np.flatnonzero(book.owner == q) for q in range(8)]
for q in range(8):
    st.set_shard(q, FeatureStore.pad_rows(g.features[ids[q]], st.src_stride, dg.device))
st.build_route(ids)
pipe = WorkerPipeline(dg, st, 0, np.flatnonzero(g.train_mask), [15, 10, 5], 1024, 7, 32, nbuf=2)
sched = SeedSchedule(7, 1, pipe.nb)
pipe.start_epoch(sched, 0)
A, B = pipe.samplers
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


def sample(smp, i0):
    pipe.plan.fill(pipe.perm, 0, i0, 32, smp)
    smp.run(32)


def gather(smp, i0, rows):
    pipe.gather(32, i0, smp, rows)


for _ in range(2):
    sample(A, 0); gather(A, 0, pipe.row_bufs[0]); sample(B, 32)
torch.cuda.synchronize()
e = [ev() for _ in range(8)]
e[0].record(); sample(A, 64); e[1].record()
e[2].record(); gather(A, 64, pipe.row_bufs[0]); e[3].record()
torch.cuda.synchronize()
print(f"sample alone {e[0].elapsed_time(e[1]):.3f} ms, gather alone {e[2].elapsed_time(e[3]):.3f} ms")
# concurrent: gather A (group 64) on sA, sample B (group 96) on sB
cur = torch.cuda.current_stream()
sA.wait_stream(cur); sB.wait_stream(cur)
e[4].record()
sA.wait_event(e[4]); sB.wait_event(e[4])
with torch.cuda.stream(sA):
    gather(A, 64, pipe.row_bufs[0]); ea = ev(); ea.record(sA)
with torch.cuda.stream(sB):
    sample(B, 96); eb = ev(); eb.record(sB)
cur.wait_stream(sA); cur.wait_stream(sB)
e[5].record()
torch.cuda.synchronize()
print(f"concurrent: gather ends {e[4].elapsed_time(ea):.3f} ms, sample ends {e[4].elapsed_time(eb):.3f} ms, both {e[4].elapsed_time(e[5]):.3f} ms")

# sampling next to a register-free HBM copy (cudaMemcpyAsync D2D of ~2 GB;
# no SM registers held): does the sampler keep its speed when HBM is busy?
big_a = torch.empty(2 * 1024**3 // 4, dtype=torch.float32, device="cuda")
big_b = torch.empty_like(big_a)
for _ in range(2):
    big_b.copy_(big_a)
torch.cuda.synchronize()
e0, e1 = ev(), ev()
e0.record(); big_b.copy_(big_a); e1.record(); torch.cuda.synchronize()
tc = e0.elapsed_time(e1)
print(f"copy alone {tc:.3f} ms = {2 * big_a.numel() * 4 / tc / 1e6:.0f} GB/s")
e4 = ev(); e4.record()
sA.wait_event(e4); sB.wait_event(e4)
with torch.cuda.stream(sA):
    big_b.copy_(big_a); ea = ev(); ea.record(sA)
with torch.cuda.stream(sB):
    sample(B, 96); eb = ev(); eb.record(sB)
torch.cuda.synchronize()
print(f"concurrent with copy: copy ends {e4.elapsed_time(ea):.3f} ms, sample ends {e4.elapsed_time(eb):.3f} ms")
with torch.cuda.stream(sB):
    sample(B, 96)
e4 = ev(); e4.record()
sA.wait_event(e4); sB.wait_event(e4)
with torch.cuda.stream(sB):
    sample(B, 96); eb = ev(); eb.record(sB)
with torch.cuda.stream(sA):
    big_b.copy_(big_a); ea = ev(); ea.record(sA)
torch.cuda.synchronize()
print(f"sampler first: copy ends {e4.elapsed_time(ea):.3f} ms, sample ends {e4.elapsed_time(eb):.3f} ms")
