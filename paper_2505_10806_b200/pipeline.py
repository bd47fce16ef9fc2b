"""Worker pipeline: the per-batch hot path for one worker, G batches per step.

One step = for G consecutive batches of the plan: fill seeds from the epoch
permutation, sample L levels, gather every input row (local shard / steady
cache / owning shard) into G bundle slots, accumulate the provenance
counters.  This is exactly the Prefetcher producer body (prefetch.py:
120-125 = plan.block + assemble_bundle) for G batches at a time, issued on
one CUDA stream with no host synchronisation; the reference's run-ahead of
Q batches becomes "the next G batches are in flight together".

The per-epoch part (plan pass counts -> remote candidates -> top_hot ->
cache fill -> cache route) follows train.py:190-204 / cache.py:80-148.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ptr
from .engine import BlockSampler, DeviceGraph, FeatureStore, bases_array
from .plan import PlanPass, candidates, threshold_select
from .sampler import SeedSchedule

I32 = torch.int32

# kernels launched per C-ABI call (for the gpu_launches count)
KERNELS_PER_CALL = {"rg_fill_seeds": 1, "rg_mark_seeds": 1, "rg_bitmap_compact": 2,
                    "rg_sample_level": 1, "rg_gather_bundle": 1}


@dataclass
class HotCache:
    hot_ids: torch.Tensor  # int32 ascending
    rows: torch.Tensor  # n_hot x stride
    route: torch.Tensor  # int32 bits of uint32 route words
    fill: tuple  # (rpcs, nodes, bytes)


def resolve_n_hot(pct: float, num_remote: int) -> int:
    """train.py:165-168 (float expression, truncation)."""
    return int(num_remote * pct / 100.0)


class WorkerPipeline:
    def __init__(self, dg: DeviceGraph, store: FeatureStore, my_part: int, train_nodes: np.ndarray,
                 fanouts, batch_size: int, s0: int, group: int):
        self.dg, self.store, self.my_part = dg, store, int(my_part)
        self.plan = PlanPass(dg, train_nodes, fanouts, batch_size, s0, group=group)
        self.sampler: BlockSampler = self.plan.sampler
        self.G = self.plan.G
        self.nb = self.plan.nb
        smp = self.sampler
        self.cap_in = smp.caps[smp.L]
        self.rows = torch.empty((self.G, self.cap_in, store.stride), dtype=torch.float32,
                                device=dg.device)
        # per-batch provenance counters of the current epoch (nb x 8)
        self.counters = torch.zeros((self.nb, _lib.RG_NCOUNTERS), dtype=I32, device=dg.device)
        self.cache: HotCache | None = None
        self.perm: torch.Tensor | None = None
        self.epoch = 0
        self.launches = 0

    # -- per epoch ---------------------------------------------------------
    def count_epoch(self, schedule: SeedSchedule, e: int) -> torch.Tensor:
        counts = torch.zeros(self.dg.n, dtype=I32, device=self.dg.device)
        self.plan.run_epoch(schedule, e, counts)
        return counts

    def select_hot(self, counts: torch.Tensor, n_hot: int, max_count: int) -> torch.Tensor:
        ids, nout, hist, bm = candidates(counts, self.store.owner, self.my_part, max_count)
        return threshold_select(counts, bm, hist.cpu().numpy().astype(np.int64), n_hot)

    def build_cache(self, hot_ids: torch.Tensor) -> HotCache:
        """VectorPull of the hot rows + cache route (cache.py:139-148)."""
        st = self.store
        n_hot = int(hot_ids.numel())
        rows = torch.empty((max(n_hot, 1), st.stride), dtype=torch.float32, device=self.dg.device)
        route = torch.empty_like(st.route)
        cnt = torch.zeros((1, _lib.RG_NCOUNTERS), dtype=I32, device=self.dg.device)
        s = _lib.stream_handle()
        if n_hot:
            nids = torch.tensor([n_hot], dtype=I32, device=self.dg.device)
            _lib.call("rg_gather_bundle", ptr(hot_ids), ptr(nids), n_hot, 1, ptr(st.route),
                      bases_array(st.bases).ctypes.data, st.stride, -1, ptr(rows), ptr(cnt), s)
        _lib.call("rg_route_with_cache", ptr(st.route), st.n, ptr(hot_ids), n_hot, ptr(route), s)
        c = cnt.cpu().numpy()[0].view(np.uint32)
        rpcs = bin(int(c[_lib.RG_CNT_OWNER_MASK])).count("1")
        self.cache = HotCache(hot_ids, rows, route, (rpcs, n_hot, 4 * st.d * n_hot))
        return self.cache

    def start_epoch(self, schedule: SeedSchedule, e: int) -> None:
        self.epoch = e
        self.perm = self.plan.permutation(schedule, e)
        self.counters.zero_()

    # -- per step (G batches) ----------------------------------------------
    def step(self, i0: int) -> int:
        """Sample + gather batches i0 .. i0+ng-1 of the current epoch."""
        ng = min(self.G, self.nb - i0)
        smp, st = self.sampler, self.store
        self.plan.fill(self.perm, self.epoch, i0, ng)
        smp.run(ng)
        self.gather(ng, i0)
        self.launches += 1 + 1 + 2 + smp.L * 3 + 1
        return ng

    def gather(self, ng: int, i0: int) -> None:
        smp, st = self.sampler, self.store
        bases = list(st.bases)
        route = st.route
        if self.cache is not None and self.cache.hot_ids.numel():
            bases[_lib.RG_KIND_CACHE] = self.cache.rows.data_ptr()
            route = self.cache.route
        _lib.call("rg_gather_bundle", ptr(smp.front[smp.L]), ptr(smp.nfront[smp.L]), self.cap_in,
                  ng, ptr(route), bases_array(bases).ctypes.data, st.stride, self.my_part,
                  ptr(self.rows), ptr(self.counters) + i0 * _lib.RG_NCOUNTERS * 4,
                  _lib.stream_handle())

    def totals(self) -> dict:
        """Epoch accounting so far (syncs): provenance sums and fallback
        RPCs = sum over batches of #owners that served a fallback row."""
        c = self.counters.cpu().numpy().view(np.uint32).astype(np.int64)
        masks = c[:, _lib.RG_CNT_OWNER_MASK]
        rpcs = int(sum(bin(int(m)).count("1") for m in masks))
        return {"local": int(c[:, 0].sum()), "hit": int(c[:, 1].sum()),
                "fallback": int(c[:, 2].sum()), "bad": int(c[:, 4].sum()), "rpcs": rpcs,
                "per_batch": c}
