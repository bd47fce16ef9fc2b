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

import os
import queue
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, multigpu
from ._lib import ptr
from .engine import BlockSampler, DeviceGraph, FeatureStore, bases_array
from .plan import PlanPass, candidates, threshold_select
from .sampler import SeedSchedule

I32 = torch.int32

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
    """nbuf = 2 double-buffers the sampler state and the bundle slots so
    that sampling of group k+1 (latency/ALU-bound) runs on one stream while
    the gather of group k (HBM-bound) runs on another — the device form of
    the reference's one-batch-ahead prefetch (prefetch.py:91-164)."""

    def __init__(self, dg: DeviceGraph, store: FeatureStore, my_part: int, train_nodes: np.ndarray,
                 fanouts, batch_size: int, s0: int, group: int, nbuf: int = 2,
                 prng: str = "splitmix"):
        self.dg, self.store, self.my_part = dg, store, int(my_part)
        self.plan = PlanPass(dg, train_nodes, fanouts, batch_size, s0, group=group, prng=prng)
        self.sampler: BlockSampler = self.plan.sampler
        self.G = self.plan.G
        self.nb = self.plan.nb
        smp = self.sampler
        self.cap_in = smp.caps[smp.L]
        self.nbuf = int(nbuf)
        self.samplers = [smp] + [BlockSampler(dg, fanouts, batch_size, group=self.G, prng=prng)
                                 for _ in range(self.nbuf - 1)]
        self.row_bufs = [torch.empty((self.G, self.cap_in, store.stride), dtype=torch.float32,
                                     device=dg.device) for _ in range(self.nbuf)]
        self.rows = self.row_bufs[0]
        self.s_sample = torch.cuda.Stream()
        self.s_gather = torch.cuda.Stream()
        # the group prefetch (N > 1) gets its own stream: sample(k+1) no longer
        # queues behind prefetch(k) (papers100M-shaped N = 2: 1,536 vs 1,425
        # batches/s; Products unchanged).  Stream priorities and a deferred
        # schedule (sample k + gather k-1 on one stream, the copy beside them)
        # measured no better: co-running kernels slow each other
        self.s_prefetch = torch.cuda.Stream()
        self.prefetch_stream = os.environ.get("RG_PREFETCH_STREAM", "1") != "0"
        self.ev_prefetched = [torch.cuda.Event() for _ in range(self.nbuf)]
        self.ev_sampled = [torch.cuda.Event() for _ in range(self.nbuf)]
        self.ev_gathered = [torch.cuda.Event() for _ in range(self.nbuf)]
        self.k = 0
        # per-batch provenance counters of the current epoch (nb x 8)
        self.counters = torch.zeros((self.nb, _lib.RG_NCOUNTERS), dtype=I32, device=dg.device)
        self.cache: HotCache | None = None
        self.perm: torch.Tensor | None = None
        self.epoch = 0
        self.launches = 0
        self._cl = int(_lib.load().rg_bitmap_compact_launches(dg.nwords))  # per compaction
        self.prefetch = False
        self.pf_transport = "p2p"
        self.timeline: list | None = None  # [(name, slot, start ev, end ev)] when set
        # "window": id-window-major gather from the input bitmaps (default);
        # "ids": the rank-major chunk queue over the sorted id lists
        self.gather_mode = os.environ.get("RG_GATHER_MODE", "window")

    # -- group prefetch of peer rows (multi-GPU, rg_prefetch.cu) -------------
    def enable_prefetch(self, transport: str = "p2p", rank: int = 0, world: int = 1) -> None:
        """Serve peer-owned rows from local shadows: once a group is sampled,
        the union of its batches' input nodes that live on peer shards is
        copied over NVLink once (rg_group_union + compaction +
        rg_prefetch_rows) into a local shadow of each peer shard, one shadow
        set per buffer slot; the gather then reads only local HBM through
        the unchanged route words (accounting identical).

        transport "p2p": the copy reads the peer shard through its CUDA IPC
        address (NVLink loads).  "nccl": the owners serve the requested rows
        through two torch.distributed all-to-alls (ids out, rows back) and
        they are scattered into the shadows — no peer mapping needed, so it
        also spans nodes."""
        if transport not in ("p2p", "nccl"):
            raise ValueError(f"unknown transport {transport!r}")
        st, dev = self.store, self.dg.device
        self.pf_transport, self.rank, self.world = transport, int(rank), int(world)
        if (transport == "p2p" and self.G * self.cap_in < 4 * self.dg.n
                and os.environ.get("RG_PREFETCH_SPARSE", "pull") == "pull"):
            # sparse groups (papers100M-shaped, G = 8: the union is ~2.3 % of
            # the nodes and the batches barely share rows): no shadows — the
            # gather reads peer rows over NVLink itself, so the transfer runs
            # inside the HBM-bound gather instead of as a serial copy before it
            # (N = 2: 2,137 vs 1,625 batches/s with the row prefetch)
            self.pf_peers, self.shadow, self.prefetch = [], [], False
            self.pf_mode = "pull"
            return
        if transport == "nccl":
            # owner rank per node; peers = shards other ranks hold
            self.owner_rank = (st.owner.to(torch.int64) % self.world).to(torch.uint8)
            self.nccl_peers = [q for q in range(st.k) if q % self.world != self.rank]
            st.peer_mask = sum(1 << q for q in self.nccl_peers)
            # kinds (partitions) held by each rank: the per-owner request lists
            # come out of one masked union + compaction per peer rank, already
            # grouped by owner and sorted (no argsort)
            self.rank_kinds = [sum(1 << q for q in range(st.k) if q % self.world == r)
                               for r in range(self.world)]
            self.pf_req = torch.empty((self.world, st.n), dtype=I32, device=dev)
            self.pf_req_n = torch.zeros(self.world, dtype=I32, device=dev)
        peers = [q for q in range(st.k) if (st.peer_mask >> q) & 1]
        self.pf_peers = peers
        self.shadow = []
        for _ in range(self.nbuf):
            bufs = {q: torch.empty((int((st.owner_np == q).sum()), st.src_stride),
                                   dtype=torch.float32, device=dev) for q in peers}
            self.shadow.append(bufs)
        nw = self.dg.nwords
        lib = _lib.device()
        self.pf_mask = torch.empty(nw, dtype=I32, device=dev)
        self.pf_union = torch.empty(nw, dtype=I32, device=dev)
        self.pf_chunk = torch.empty(int(lib.rg_bitmap_chunks(nw)), dtype=I32, device=dev)
        self.pf_ids = torch.empty(st.n, dtype=I32, device=dev)
        self.pf_n = torch.zeros(self.nbuf, dtype=I32, device=dev)
        self.pf_rows = torch.zeros(1, dtype=torch.int64, device=dev)  # rows copied (stats)
        self.pf_whole_shards = os.environ.get("RG_PREFETCH_WHOLE", "1") != "0"
        self.prefetch = bool(peers)

    # -- shared sampling (multi-GPU) ------------------------------------------
    def enable_shared_sampling(self, rank: int, world: int, timeout_ms: int = 20000) -> None:
        """Split each group's sampling across the ranks.  Every worker
        processes every batch (train.py:291-311), so the N ranks sample the
        same blocks; here rank r samples only slots [r*ng/N, (r+1)*ng/N) of
        a group and copies the other slots' sampled blocks from the peers'
        sampler buffers over NVLink (copy engine): first what the gather
        reads (the level-L bitmaps + ranks, or the id lists), which gates the
        gather, then the rest of every level (frontiers, counts, ELL edges),
        so each rank ends up holding every batch's whole block, as if it had
        sampled them all.  Cross-process order by 64-bit group sequence
        counters in each rank's memory polled through the IPC mapping
        (rg_flag_signal / rg_flag_wait): "slot s holds my share of group k"
        and "I copied the peers' shares of group k".  Bundles, blocks and
        accounting are unchanged (bench --check compares a shared group with
        a locally sampled one)."""
        if int(world) < 2:
            return
        tensors = self.shared_tensors(rank, world, timeout_ms)
        self.wire_shared(multigpu.exchange_buffers(tensors, self.rank, self.world))

    def shared_tensors(self, rank: int, world: int, timeout_ms: int = 20000) -> list:
        """Allocate the shared-sampling counters; returns the buffers every
        peer maps: [flags] + per slot [bm, wpre, nfront, front 0..L,
        ell 0..L-1, cnt 0..L-1]."""
        self.rank, self.world = int(rank), int(world)
        dev = self.dg.device
        self.sh_flags = torch.zeros((2, self.nbuf), dtype=torch.int64, device=dev)
        self.sh_status = torch.zeros(1, dtype=I32, device=dev)
        self.sh_timeout = int(timeout_ms)
        self.ev_inputs = [torch.cuda.Event() for _ in range(self.nbuf)]
        self.s_block = torch.cuda.Stream()
        tensors = [self.sh_flags]
        for smp in self.samplers:
            tensors += [smp.bm, smp.wpre, smp.nfront, *smp.front, *smp.ell, *smp.cnt]
        return tensors

    def wire_shared(self, ptrs: list) -> None:
        """ptrs[i][r] = address of rank r's shared_tensors()[i] in this
        process (multigpu.exchange_buffers; the peers' through CUDA IPC)."""
        L = self.sampler.L
        per = 3 + (L + 1) + 2 * L
        self.sh_peer_flags = ptrs[0]
        self.sh_peer_bufs = [ptrs[1 + per * i: 1 + per * (i + 1)] for i in range(self.nbuf)]
        self.shared = True
        self.sh_seq = 0
        self.sh_last = [0] * self.nbuf  # sequence number last sampled into each slot

    def _share_range(self, ng: int, r: int) -> tuple[int, int]:
        return r * ng // self.world, (r + 1) * ng // self.world

    def _share_spans(self, smp, c0: int, c1: int) -> list:
        """(buffer index, byte offset, bytes) of slots [c0, c1) in every
        shared sampler buffer, in the enable_shared_sampling order."""
        L, G = smp.L, self.G
        rows = [smp.bm, smp.wpre]
        out = [(i, c0 * t.stride(0) * 4, (c1 - c0) * t.stride(0) * 4) for i, t in enumerate(rows)]
        out += [(2, 4 * (d * G + c0), 4 * (c1 - c0)) for d in range(L + 1)]  # nfront[d]
        for i, t in enumerate([*smp.front, *smp.ell, *smp.cnt]):
            out.append((3 + i, c0 * t.stride(0) * 4, (c1 - c0) * t.stride(0) * 4))
        return out

    def _sample_shared(self, ng: int, smp, slot: int, seq: int) -> None:
        """Current stream: sample my share of the group into `slot`, publish
        it, copy the peers' shares — what the gather reads first (then
        ev_inputs[slot]), the rest of the blocks after — and publish that."""
        s = _lib.stream_handle()
        fl = ptr(self.sh_flags)
        # the peers finished copying the previous group held in this slot
        prev = self.sh_last[slot]
        self.sh_last[slot] = seq
        if prev > 0:
            for r in range(self.world):
                if r != self.rank:
                    _lib.call("rg_flag_wait", self.sh_peer_flags[r] + 8 * (self.nbuf + slot),
                              prev, self.sh_timeout, ptr(self.sh_status), s)
        b0, b1 = self._share_range(ng, self.rank)
        smp.run(b1, b0=b0)
        _lib.call("rg_flag_signal", fl + 8 * slot, seq, s)
        # what the group's gather reads: the window gather the bitmaps +
        # ranks, the id-list gather front[L] / nfront[L], a row-wise or NCCL
        # group prefetch the bitmaps (the group union)
        L = smp.L
        window = self._window_gather(ng)
        whole = (self.pf_transport == "p2p" and getattr(self, "pf_whole_shards", True)
                 and ng * self.cap_in >= 4 * self.dg.n)
        first = set()
        if window or (self.prefetch and not whole):
            first.add((0, 0))  # bm
        if window:
            first.add((1, 0))  # wpre
        else:
            first.add((2, L))  # nfront[L]
            first.add((3 + L, 0))  # front[L]
        local = self.sh_peer_bufs[slot]
        spans = {}
        for r in range(self.world):
            c0, c1 = self._share_range(ng, r)
            if r == self.rank or c1 <= c0:
                continue
            _lib.call("rg_flag_wait", self.sh_peer_flags[r] + 8 * slot, seq, self.sh_timeout,
                      ptr(self.sh_status), s)
            spans[r] = self._share_spans(smp, c0, c1)
        # with the bitmaps copied, the input id lists (front[L], 62 % of a
        # Products block) are re-derived by a local compaction instead
        derive = {(2, L), (3 + L, 0)} if window else set()

        def copies(phase, stream):
            for r, sp in spans.items():
                nfront_d = 0
                for i, off, nbytes in sp:
                    key = (i, nfront_d if i == 2 else 0)
                    if i == 2:
                        nfront_d += 1
                    if (key in first) == (phase == 0) and (i != 1 or window) and key not in derive:
                        _lib.call("rg_copy_bytes", local[i][self.rank] + off,
                                  local[i][r] + off, nbytes, stream)
                if phase == 1 and derive:
                    c0, c1 = self._share_range(ng, r)
                    nw, capL = self.dg.nwords, smp.caps[L]
                    _lib.call("rg_bitmap_compact", ptr(smp.bm) + 4 * c0 * nw, nw, c1 - c0,
                              ptr(smp.chunk), ptr(smp.front[L]) + 4 * c0 * capL, capL,
                              ptr(smp.nfront) + 4 * (L * self.G + c0), None, stream)
                    self.launches += self._cl

        copies(0, s)  # the gather's inputs, on the sampling stream
        self.ev_inputs[slot].record()
        # the rest of the blocks on their own stream: the next group's
        # sampling does not queue behind them
        with torch.cuda.stream(self.s_block):
            self.s_block.wait_event(self.ev_inputs[slot])
            sb = _lib.stream_handle()
            copies(1, sb)
            _lib.call("rg_flag_signal", fl + 8 * (self.nbuf + slot), seq, sb)
            self.ev_sampled[slot].record(self.s_block)
        self.launches += 2 + (self.world - 1) + (1 if prev > 0 else 0) * (self.world - 1)

    def shared_status(self) -> int:
        """1 if any cross-GPU wait timed out (results then invalid)."""
        return int(self.sh_status.item()) if getattr(self, "shared", False) else 0

    def _dense(self, ng: int) -> bool:
        st = self.store
        return ng * self.cap_in >= 4 * self.dg.n and st.stride * 4 * 32 <= 200 * 1024

    def _window_gather(self, ng: int) -> bool:
        """True if gather() reads the group's bitmaps + ranks (the staged
        window gather), False if it reads the id lists."""
        peer_mask = 0 if self.prefetch else self.store.peer_mask
        return (self.gather_mode == "window" and self._dense(ng) and ng <= 128
                and peer_mask == 0)

    def _route(self):
        if self.cache is not None and self.cache.hot_ids.numel():
            return self.cache.route
        return self.store.route

    def prefetch_group(self, ng: int, smp, slot: int) -> None:
        """Copy the group's peer rows into shadow[slot] (current stream)."""
        st, s = self.store, _lib.stream_handle()
        route = self._route()
        nw = self.dg.nwords
        dst = [0] * 16
        for q, t in self.shadow[slot].items():
            dst[q] = t.data_ptr()
        nid = ptr(self.pf_n) + 4 * slot
        if self.pf_transport == "nccl":
            self._exchange_nccl(ng, smp, slot, route, dst)
            self.pf_rows += self.pf_n[slot]
            self.launches += 6
            return
        if self.pf_whole_shards and ng * self.cap_in >= 4 * self.dg.n:
            # dense group: its union of peer rows is nearly every row of the
            # peer shards (Products G = 128: 1.03 M of 1.22 M at N = 2), so the
            # shards are copied whole on the copy engines (contiguous, ~820 GB/s
            # measured, no SMs) instead of gathered row by row (~540 GB/s)
            for q, t in self.shadow[slot].items():
                _lib.call("rg_copy_bytes", t.data_ptr(), st.bases[q], t.numel() * 4, s)
                self.pf_rows += t.shape[0]
            self.pf_mode = "whole shards"
            return
        self.pf_mode = "rows"
        _lib.call("rg_route_kind_bits", ptr(route), st.n, st.peer_mask, ptr(self.pf_mask), s)
        _lib.call("rg_group_union", ptr(smp.bm), nw, ng, ptr(self.pf_mask), ptr(self.pf_union), s)
        _lib.call("rg_bitmap_compact", ptr(self.pf_union), nw, 1, ptr(self.pf_chunk),
                  ptr(self.pf_ids), st.n, nid, None, s)
        _lib.call("rg_prefetch_rows", ptr(self.pf_ids), nid, st.n, ptr(route),
                  bases_array(st.bases), bases_array(dst), st.src_stride, st.stride, s)
        self.pf_rows += self.pf_n[slot]
        self.launches += 3 + self._cl

    def _exchange_nccl(self, ng: int, smp, slot: int, route, dst) -> None:
        """NCCL transport: requested ids to their owners, rows back, scatter
        into shadow[slot] (current stream; one host sync for the sizes).
        The request list for owner rank r = compaction of the group union
        masked with r's kinds, so the lists arrive grouped and sorted."""
        st, s = self.store, _lib.stream_handle()
        nw = self.dg.nwords
        for r in range(self.world):
            if r == self.rank:
                continue
            _lib.call("rg_route_kind_bits", ptr(route), st.n, self.rank_kinds[r],
                      ptr(self.pf_mask), s)
            _lib.call("rg_group_union", ptr(smp.bm), nw, ng, ptr(self.pf_mask),
                      ptr(self.pf_union), s)
            _lib.call("rg_bitmap_compact", ptr(self.pf_union), nw, 1, ptr(self.pf_chunk),
                      ptr(self.pf_req[r]), st.n, ptr(self.pf_req_n) + 4 * r, None, s)
        counts = self.pf_req_n.cpu().tolist()  # one host sync for every split size
        counts[self.rank] = 0
        self.pf_n[slot] = sum(counts)
        ids = torch.cat([self.pf_req[r, :counts[r]] for r in range(self.world)])
        send_ids, rows = multigpu.exchange_rows(ids, None, self.world, self._serve,
                                                counts=counts)
        _lib.call("rg_scatter_rows", ptr(send_ids), send_ids.numel(), ptr(route), ptr(rows),
                  st.src_stride, bases_array(dst), st.src_stride, st.src_stride,
                  _lib.stream_handle())

    def _serve(self, req):
        """Owner side of the NCCL transport: rows (src_stride floats) of the
        requested ids, all held by this rank's shards (base route)."""
        st = self.store
        out = torch.empty((max(1, req.numel()), st.src_stride), dtype=torch.float32,
                          device=req.device)
        if req.numel():
            nreq = torch.tensor([req.numel()], dtype=I32, device=req.device)
            cnt = torch.zeros((1, _lib.RG_NCOUNTERS), dtype=I32, device=req.device)
            _lib.call("rg_gather_bundle", ptr(req), ptr(nreq), req.numel(), 1, ptr(st.route),
                      bases_array(st.bases), st.src_stride, st.src_stride, -1, 0, ptr(out),
                      ptr(cnt), _lib.stream_handle())
        return out[: req.numel()]

    # -- per epoch ---------------------------------------------------------
    def count_epoch(self, schedule: SeedSchedule, e: int, shared: bool = False) -> torch.Tensor:
        """Access counts of every node over epoch e (collect_access,
        plan.py:108-130; worker-independent, the remote mask is applied at
        extraction).  shared (N > 1, torch.distributed up): each rank samples
        every N-th group and one NCCL all-reduce sums the integer counts —
        the same table on every rank, 1/N of the sampling."""
        counts = torch.zeros(self.dg.n, dtype=I32, device=self.dg.device)
        world = getattr(self, "world", 1) if shared else 1
        if world > 1:
            import torch.distributed as dist

            self.plan.run_epoch(schedule, e, counts, share=(self.rank, world))
            dist.all_reduce(counts)
        else:
            self.plan.run_epoch(schedule, e, counts)
        return counts

    def select_hot(self, counts: torch.Tensor, n_hot: int, max_count: int) -> torch.Tensor:
        ids, nout, hist, bm = candidates(counts, self.store.owner, self.my_part, max_count)
        return threshold_select(counts, bm, hist.cpu().numpy().astype(np.int64), n_hot)

    def build_cache(self, hot_ids: torch.Tensor) -> HotCache:
        """VectorPull of the hot rows + cache route (cache.py:139-148),
        installed as the steady cache."""
        self.cache = self.make_cache(hot_ids)
        return self.cache

    def make_cache(self, hot_ids: torch.Tensor) -> HotCache:
        """A cache buffer for hot_ids on the current stream, not installed
        (the secondary of the double buffer, cache.py:80-104)."""
        st = self.store
        n_hot = int(hot_ids.numel())
        rows = torch.empty((max(n_hot, 1), st.src_stride), dtype=torch.float32,
                           device=self.dg.device)
        route = torch.empty_like(st.route)
        cnt = torch.zeros((1, _lib.RG_NCOUNTERS), dtype=I32, device=self.dg.device)
        s = _lib.stream_handle()
        _lib.call("rg_route_with_cache", ptr(st.route), st.n, ptr(hot_ids), n_hot, ptr(route), s)
        if self.pf_transport == "nccl":
            # owners serve the hot rows over the all-to-all; scatter into the
            # cache slots through the cache route (kind 15 | slot)
            dst = [0] * 16
            dst[_lib.RG_KIND_CACHE] = rows.data_ptr()
            send_ids, got = multigpu.exchange_rows(hot_ids, self.owner_rank[hot_ids.long()],
                                                   self.world, self._serve)
            _lib.call("rg_scatter_rows", ptr(send_ids), send_ids.numel(), ptr(route), ptr(got),
                      st.src_stride, bases_array(dst), st.src_stride, st.src_stride, s)
            rpcs = int(torch.unique(st.owner[hot_ids.long()]).numel()) if n_hot else 0
        else:
            if n_hot:
                nids = torch.tensor([n_hot], dtype=I32, device=self.dg.device)
                _lib.call("rg_gather_bundle", ptr(hot_ids), ptr(nids), n_hot, 1, ptr(st.route),
                          bases_array(st.bases), st.src_stride, st.src_stride, -1,
                          st.peer_mask, ptr(rows), ptr(cnt), s)
            c = cnt.cpu().numpy()[0].view(np.uint32)
            rpcs = bin(int(c[_lib.RG_CNT_OWNER_MASK])).count("1")
        return HotCache(hot_ids, rows, route, (rpcs, n_hot, 4 * st.d * n_hot))

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
        self.launches += 3 + self._cl + smp.L * (2 + self._cl)
        return ng

    def step_graph(self, i0: int) -> int:
        """step(i0) replayed from a CUDA graph captured on first use (one
        graph per group start: i0 is a kernel argument).  Removes the
        per-launch host cost, which dominates small graphs (C1: ~41 MB per
        batch, 6 us at HBM speed)."""
        ng = min(self.G, self.nb - i0)
        key = (self.epoch, i0, ng)
        graphs = self.__dict__.setdefault("_graphs", {})
        gr = graphs.get(key)
        if gr is None:
            if len(graphs) > 4096:
                graphs.clear()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):  # warm the allocator outside capture
                self.step(i0)
            torch.cuda.current_stream().wait_stream(side)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                self.step(i0)
            graphs[key] = gr
        gr.replay()
        return ng

    def step_overlapped(self, i0: int, host_seeds=None) -> int:
        """Like step(), but sampling and gather of consecutive groups overlap
        on two streams (buffer k % nbuf).  Call sync_streams() before reading
        results on the current stream.  host_seeds = (seeds [G, cap0] int32,
        nseeds [G] int32, batch seeds [G] int64) pinned host tensors: the
        group's seeds are copied H2D on the sampling stream instead of being
        filled from the device plan."""
        ng = min(self.G, self.nb - i0)
        slot = self.k % self.nbuf
        self.k += 1
        self.last_slot = slot
        smp = self.samplers[slot]
        tl = self.timeline

        def mark(name, stream, ev=None):
            if tl is None:
                return None
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            if ev is not None:
                tl.append((name, slot, ev, e))
            return e

        with torch.cuda.stream(self.s_sample):
            self.s_sample.wait_event(self.ev_gathered[slot])  # slot free again
            if getattr(self, "shared", False):  # and the last block copies into it done
                self.s_sample.wait_event(self.ev_sampled[slot])
            e0 = mark("sample", self.s_sample)
            if host_seeds is None:
                self.plan.fill(self.perm, self.epoch, i0, ng, smp)
            else:
                smp.seeds.copy_(host_seeds[0], non_blocking=True)
                smp.nseeds.copy_(host_seeds[1], non_blocking=True)
                smp.rng.copy_(host_seeds[2], non_blocking=True)
            if getattr(self, "shared", False):
                self.sh_seq += 1
                self._sample_shared(ng, smp, slot, self.sh_seq)
            else:
                smp.run(ng)
            e1 = mark("sample", self.s_sample, e0)
            if self.prefetch and not self.prefetch_stream:
                self.prefetch_group(ng, smp, slot)
                mark("prefetch", self.s_sample, e1)
            if not getattr(self, "shared", False):  # shared: recorded after the block copies
                self.ev_sampled[slot].record(self.s_sample)
        # shared sampling: the gather needs only the input sets (the rest of
        # the peers' blocks is still being copied on its own stream)
        gate = self.ev_inputs[slot] if getattr(self, "shared", False) else self.ev_sampled[slot]
        if self.prefetch and self.prefetch_stream:
            with torch.cuda.stream(self.s_prefetch):
                self.s_prefetch.wait_event(gate)
                e3 = mark("prefetch", self.s_prefetch)
                self.prefetch_group(ng, smp, slot)
                mark("prefetch", self.s_prefetch, e3)
                self.ev_prefetched[slot].record(self.s_prefetch)
            gate = self.ev_prefetched[slot]
        with torch.cuda.stream(self.s_gather):
            self.s_gather.wait_event(gate)
            e2 = mark("gather", self.s_gather)
            self.gather(ng, i0, smp, self.row_bufs[slot], slot=slot, prefetched=True)
            mark("gather", self.s_gather, e2)
            self.ev_gathered[slot].record(self.s_gather)
        self.launches += 3 + self._cl + smp.L * (2 + self._cl)
        return ng

    def acquire(self, slot: int) -> None:
        """Current stream waits until group `slot` is sampled and gathered."""
        torch.cuda.current_stream().wait_event(self.ev_sampled[slot])
        torch.cuda.current_stream().wait_event(self.ev_gathered[slot])

    def release(self, slot: int) -> None:
        """The current stream's queued work is the last reader of `slot`:
        the next step_overlapped into it waits for that work."""
        self.ev_gathered[slot].record(torch.cuda.current_stream())

    def enter_streams(self) -> None:
        """Order both side streams after the current stream's work."""
        cur = torch.cuda.current_stream()
        if getattr(self, "shared", False):
            self.s_block.wait_stream(cur)
        self.s_sample.wait_stream(cur)
        self.s_prefetch.wait_stream(cur)
        self.s_gather.wait_stream(cur)

    def sync_streams(self) -> None:
        cur = torch.cuda.current_stream()
        if getattr(self, "shared", False):
            cur.wait_stream(self.s_block)
        cur.wait_stream(self.s_sample)
        cur.wait_stream(self.s_prefetch)
        cur.wait_stream(self.s_gather)

    def gather(self, ng: int, i0: int, smp=None, rows=None, slot: int = 0,
               prefetched: bool = False) -> None:
        """Bundle rows of the group sampled in smp.  With prefetch enabled,
        peer rows come from shadow[slot] (filled here first unless the
        caller already ran prefetch_group for this group and slot)."""
        smp = smp or self.sampler
        rows = self.rows if rows is None else rows
        st = self.store
        bases = list(st.bases)
        route = st.route
        if self.cache is not None and self.cache.hot_ids.numel():
            bases[_lib.RG_KIND_CACHE] = self.cache.rows.data_ptr()
            route = self.cache.route
        peer_mask = st.peer_mask
        if self.prefetch:
            if not prefetched:
                self.prefetch_group(ng, smp, slot)
            for q, t in self.shadow[slot].items():
                bases[q] = t.data_ptr()
            peer_mask = 0  # every row is local now
        cnt = ptr(self.counters) + i0 * _lib.RG_NCOUNTERS * 4
        # the bitmap-driven (staged union) gather pays off when the group's
        # batches share rows: G * cap_in / n bounds the mean reuse of a union
        # row (Products G = 128: 56, measured ~35 -> 5.97 vs 6.70 ms); for
        # sparse groups (papers100M-shaped, G = 8: 0.31) the id-list queue
        # gather is faster (15.8 vs ~3.5 ms per launch)
        if self._window_gather(ng):
            # staged union gather straight from the group's input bitmaps
            self.gather_kernel = "gather_staged_kernel (rg_gather_window)"
            _lib.call("rg_gather_window", ptr(smp.bm), ptr(smp.wpre), self.dg.nwords, ng,
                      self.cap_in, ptr(route), bases_array(bases), st.src_stride, st.stride,
                      self.my_part, st.peer_mask, ptr(rows), cnt, _lib.stream_handle())
            return
        self.gather_kernel = ("gather_queue_kernel (rg_gather_bundle)" if peer_mask == 0 else
                              "gather_bundle_kernel<row-aligned> (rg_gather_bundle)")
        _lib.call("rg_gather_bundle", ptr(smp.front[smp.L]), ptr(smp.nfront[smp.L]), self.cap_in,
                  ng, ptr(route), bases_array(bases), st.src_stride, st.stride,
                  self.my_part, peer_mask, ptr(rows), cnt, _lib.stream_handle())

    def totals(self) -> dict:
        """Epoch accounting so far (syncs): provenance sums and fallback
        RPCs = sum over batches of #owners that served a fallback row."""
        c = self.counters.cpu().numpy().view(np.uint32).astype(np.int64)
        masks = c[:, _lib.RG_CNT_OWNER_MASK]
        rpcs = int(sum(bin(int(m)).count("1") for m in masks))
        return {"local": int(c[:, 0].sum()), "hit": int(c[:, 1].sum()),
                "fallback": int(c[:, 2].sum()), "bad": int(c[:, 4].sum()), "rpcs": rpcs,
                "peer": int(c[:, _lib.RG_CNT_PEER].sum()), "per_batch": c}


class GroupProducer:
    """Producer thread of the device pipeline (prefetch.py:91-164 at group
    granularity): samples and gathers groups i0 = starts[0], starts[1], ...
    on the pipeline's side streams (step_overlapped) while the consumer
    trains the previous group on its own stream.  At most nbuf groups are
    live: a slot is produced into again only after the consumer released it
    (token per slot), and its device reuse is ordered by the consumer's
    release event.  The host wait for a group's sizes (nfront) happens on
    this thread, never on the consumer's.  latency_ms > 0 sleeps the
    injected per-request latency (store.py:73-74) here, once per fallback
    RPC of the group, so the producer hides it like the reference's
    Prefetcher thread does."""

    def __init__(self, pipe: WorkerPipeline, starts, latency_ms: float = 0.0):
        if pipe.nbuf < 2:
            raise ValueError("GroupProducer needs a double-buffered pipeline (nbuf >= 2)")
        self.pipe = pipe
        self.latency_ms = float(latency_ms)
        self._q: queue.Queue = queue.Queue()
        self._tokens = threading.Semaphore(pipe.nbuf)
        self._stop = threading.Event()
        self.capture_lock = threading.Lock()
        self._done = False
        pin = torch.cuda.is_available()
        self._nf = [torch.zeros((pipe.sampler.L + 1, pipe.G), dtype=I32).pin_memory()
                    if pin else None for _ in range(pipe.nbuf)]
        self._cnt = [torch.zeros((pipe.G, _lib.RG_NCOUNTERS), dtype=I32).pin_memory()
                     if pin else None for _ in range(pipe.nbuf)]
        self._ev = [torch.cuda.Event() for _ in range(pipe.nbuf)]
        self._dev = torch.cuda.current_device()
        pipe.enter_streams()
        self._t = threading.Thread(target=self._run, args=(list(starts),), daemon=True)
        self._t.start()

    def _run(self, starts) -> None:
        pipe = self.pipe
        try:
            torch.cuda.set_device(self._dev)
            for i0 in starts:
                while not self._tokens.acquire(timeout=0.05):
                    if self._stop.is_set():
                        return
                if self._stop.is_set():
                    return
                # CUDA API work of this thread is excluded while the consumer
                # captures a CUDA graph (capture_lock): a concurrent launch or
                # sync from another thread can invalidate a capture
                with self.capture_lock:
                    ng = pipe.step_overlapped(i0)
                    slot = pipe.last_slot
                    with torch.cuda.stream(pipe.s_gather):
                        self._nf[slot].copy_(pipe.samplers[slot].nfront, non_blocking=True)
                        if self.latency_ms > 0:
                            self._cnt[slot][:ng].copy_(pipe.counters[i0:i0 + ng],
                                                       non_blocking=True)
                        self._ev[slot].record(pipe.s_gather)
                while True:
                    with self.capture_lock:
                        if self._ev[slot].query():
                            break
                    time.sleep(50e-6)
                if self.latency_ms > 0:
                    masks = self._cnt[slot][:ng, _lib.RG_CNT_OWNER_MASK].numpy().view(np.uint32)
                    rpcs = sum(bin(int(m)).count("1") for m in masks)
                    time.sleep(self.latency_ms * rpcs / 1000.0)
                self._q.put((i0, ng, slot, self._nf[slot][:, :ng].numpy().copy()))
            self._q.put(None)
        except BaseException as exc:  # surfaced on the consumer side
            self._q.put(exc)

    def next_group(self):
        """(i0, ng, slot, nfront [L+1, ng]) of the next group, its rows usable
        on the current stream; None at the end."""
        if self._done:
            return None
        item = self._q.get()
        if item is None:
            self._done = True
            return None
        if isinstance(item, BaseException):
            self._done = True
            raise item
        self.pipe.acquire(item[2])
        return item

    def release(self, slot: int) -> None:
        self.pipe.release(slot)
        self._tokens.release()

    def close(self) -> None:
        self._stop.set()
        self._t.join()
        self.pipe.sync_streams()


def run_accounting(g, book, fanouts, batch_size: int, epochs: int, s0: int, mode: str = "rapid",
                   n_hot: int | None = None, n_hot_pct: float = 15.0, hot_scope: str = "epoch",
                   workers=None, group: int = 16, features: bool = True,
                   prng: str = "splitmix") -> dict:
    """Per-worker, per-epoch data-path accounting of the reference's worker
    loop (train.py:171-264 without the SGD step): rpc_calls, nodes_pulled,
    bytes_pulled, cache_hits, cache_misses, reuse_ratio, plus the cache
    fill account.  Every batch really is sampled and gathered on the
    device; only the training consumer is absent.

    Semantics reproduced: n_hot = int(#remote(all epochs) * pct / 100)
    (train.py:165-168); epoch scope installs top_hot(collect_access(e)) for
    each epoch via the double buffer, resetting hit/miss counters on each
    successful swap; global scope builds one set and never swaps, so its
    counters accumulate (cache.py:116-129); baseline mode has no cache,
    misses = nodes pulled and reuse 0.0 or None (train.py:238-240)."""
    if mode not in ("baseline", "rapid") or hot_scope not in ("epoch", "global"):
        raise ValueError("bad mode / hot scope")
    owner = np.asarray(book.owner)
    k = int(book.k)
    dg = DeviceGraph.of(g)
    d = int(g.feat_dim) if features else 4
    store = FeatureStore(owner, k, d)
    shard_ids = [np.flatnonzero(owner == q) for q in range(k)]
    for q in range(k):
        rows = (g.features[shard_ids[q]] if features
                else np.zeros((len(shard_ids[q]), d), dtype=np.float32))
        store.set_shard(q, FeatureStore.pad_rows(rows, store.src_stride, dg.device))
    store.build_route(shard_ids)
    train = np.flatnonzero(g.train_mask)
    workers = list(range(k)) if workers is None else list(workers)
    pipe0 = WorkerPipeline(dg, store, workers[0], train, fanouts, batch_size, s0, group, nbuf=1,
                           prng=prng)
    nb = pipe0.nb
    sched = SeedSchedule(s0, epochs, nb)
    counts = [pipe0.count_epoch(sched, e) for e in range(epochs)]
    counts_all = counts[0].clone()
    for c in counts[1:]:
        counts_all += c
    max_count = max(1, nb * epochs)
    out = {}
    for p in workers:
        pipe = pipe0 if p == workers[0] else WorkerPipeline(dg, store, p, train, fanouts,
                                                            batch_size, s0, group, nbuf=1,
                                                            prng=prng)
        pipe.my_part = p
        fill = [0, 0, 0]
        nh = 0
        if mode == "rapid":
            _, nout, _, _ = candidates(counts_all, store.owner, p, max_count)
            nh = n_hot if n_hot is not None else resolve_n_hot(n_hot_pct, int(nout.item()))
        hits_acc = misses_acc = 0
        recs = []
        for e in range(epochs):
            if mode == "rapid" and (hot_scope == "epoch" or e == 0):
                scope_counts = counts[e] if hot_scope == "epoch" else counts_all
                hot = pipe.select_hot(scope_counts, nh, max_count)
                cache = pipe.build_cache(hot)
                if cache.fill[1]:  # an empty pull is free (store.py:181-182)
                    fill = [fill[0] + cache.fill[0], fill[1] + cache.fill[1],
                            fill[2] + 4 * int(g.feat_dim) * cache.fill[1]]
            pipe.start_epoch(sched, e)
            for i0 in range(0, nb, pipe.G):
                pipe.step(i0)
            t = pipe.totals()
            nodes = t["fallback"]
            if mode == "rapid":
                if hot_scope == "epoch":
                    hits, misses = t["hit"], t["fallback"]
                else:
                    hits_acc += t["hit"]
                    misses_acc += t["fallback"]
                    hits, misses = hits_acc, misses_acc
                reuse = hits / (hits + misses) if hits + misses else None
            else:
                hits, misses = 0, nodes
                reuse = 0.0 if misses else None
            recs.append({"rpc_calls": t["rpcs"], "nodes_pulled": nodes,
                         "bytes_pulled": 4 * int(g.feat_dim) * nodes, "cache_hits": hits,
                         "cache_misses": misses, "reuse_ratio": reuse, "n_hot": nh,
                         "local": t["local"]})
        out[p] = {"records": recs, "fill": fill}
    return out
