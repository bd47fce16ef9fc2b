"""Test helper (tests/test_gpu_parity.py::test_shared_sampling_two_workers_one_gpu):
two workers' pipelines on one GPU share each group's sampling through plain
device addresses; every shared block and bundle equals a locally sampled
run.  Run as `python tests/shared_one_gpu.py GROUP` (needs a GPU)."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2505_10806_b200 as rg  # noqa: E402

group = int(sys.argv[1])
from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore
from paper_2505_10806_b200.pipeline import WorkerPipeline
from paper_2505_10806_b200.sampler import SeedSchedule

g = rg.synth_powerlaw(20000, 5, 16, 4, seed=3)
book = rg.partition_edgecut(g, 2)
dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
store = FeatureStore(book.owner, 2, g.feat_dim)
ids = [np.flatnonzero(book.owner == q) for q in range(2)]
for q in range(2):
    store.set_shard(q, FeatureStore.pad_rows(g.features[ids[q]], store.src_stride, dg.device))
store.build_route(ids)
train = np.flatnonzero(g.train_mask)
mk = lambda p, nbuf: WorkerPipeline(dg, store, p, train, [5, 3], 256, 7, group, nbuf=nbuf)
pipes = [mk(0, 2), mk(1, 2)]
assert pipes[0]._window_gather(group) == (group == 16)
tens = [p.shared_tensors(r, 2, timeout_ms=5000) for r, p in enumerate(pipes)]
ptrs = [[tens[r][i].data_ptr() for r in range(2)] for i in range(len(tens[0]))]
sched = SeedSchedule(7, 1, pipes[0].nb)
# load every kernel before any cross-worker wait is in flight: with lazy
# module loading a first launch can stall the (single) host thread while a
# wait kernel spins for work this thread has not enqueued yet
from paper_2505_10806_b200 import _lib  # noqa: E402

for p in pipes:
    p.start_epoch(sched, 0)
    p.step(0)
    _lib.call("rg_flag_signal", ptr0 := p.sh_flags.data_ptr(), 0, _lib.stream_handle())
    _lib.call("rg_flag_wait", ptr0, 0, 1000, p.sh_status.data_ptr(), _lib.stream_handle())
torch.cuda.synchronize()
for p in pipes:
    p.wire_shared(ptrs)
    p.start_epoch(sched, 0)
    p.enter_streams()
starts = [0, group, 2 * group]


def worker(p):  # one host thread per worker, as one process per GPU would be
    for i0 in starts:
        p.step_overlapped(i0)
    p.sync_streams()


import threading  # noqa: E402

ths = [threading.Thread(target=worker, args=(p,)) for p in pipes]
for t in ths:
    t.start()
for t in ths:
    t.join()
torch.cuda.synchronize()
assert all(p.shared_status() == 0 for p in pipes)
i0, ng = starts[-1], group
for r, p in enumerate(pipes):
    ref = mk(r, 1)
    ref.start_epoch(sched, 0)
    for j in starts:
        ref.step(j)
    torch.cuda.synchronize()
    sh, loc = p.samplers[p.last_slot], ref.sampler
    L = sh.L
    assert torch.equal(sh.nfront[:, :ng], loc.nfront[:, :ng])
    for b in range(ng):
        assert torch.equal(sh.bm[b], loc.bm[b])
        for d in range(L + 1):
            m = int(loc.nfront[d, b])
            assert torch.equal(sh.front[d][b, :m], loc.front[d][b, :m])
        for d in range(L):
            m, F = int(loc.nfront[d, b]), sh.step_fan[d]
            assert torch.equal(sh.cnt[d][b, :m], loc.cnt[d][b, :m])
            live = torch.arange(F, device="cuda")[None, :] < loc.cnt[d][b, :m, None].long()
            assert torch.equal(sh.ell[d][b, :m * F].view(m, F)[live],
                               loc.ell[d][b, :m * F].view(m, F)[live])
        n = int(loc.nfront[L, b])
        assert torch.equal(p.row_bufs[p.last_slot][b, :n], ref.rows[b, :n])
    assert torch.equal(p.counters[: i0 + ng], ref.counters[: i0 + ng])
print("shared ok", group)
