"""Drop-in for gnnpipe.plan (plan.py:1-141): precomputed schedule, access
counts, hot-set selection — on the device.

generate_plan samples every batch of every epoch in groups of G on the GPU
(the same kernels as the per-batch path) and accumulates, per epoch, the
number of batches whose input set holds each node (rg_count_inputs on the
level-L bitmaps).  collect_access then only masks that dense count array
to the worker's remote nodes; top_hot is the count-threshold select of
SURVEY.md Appendix A.4 (histogram -> c* -> ordered tie quota), which equals
the reference's lexsort((ids, -counts))[:n_hot] (plan.py:133-141).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import ptr
from .engine import BlockSampler, DeviceGraph
from .sampler import (ComputationBlock, SeedSchedule, epoch_master, epoch_order_device,
                      sample_block, seed_for)

I32 = torch.int32


@dataclass
class FrequencyTable:
    """Access counts for remote node ids, one per batch appearance (plan.py:16-30)."""

    ids: np.ndarray  # sorted ascending
    counts: np.ndarray

    def as_dict(self) -> dict[int, int]:
        return {int(i): int(c) for i, c in zip(self.ids, self.counts)}

    def total(self) -> int:
        return int(self.counts.sum())

    def __len__(self) -> int:
        return len(self.ids)


@dataclass
class BatchPlan:
    """The precomputed schedule (plan.py:33-69) plus, per epoch, the device
    count array counts[e][v] = #batches of epoch e whose input set holds v."""

    graph: object
    schedule: SeedSchedule
    fanouts: list[int]
    batch_seeds: list[list[np.ndarray]]
    input_sets: list[list[np.ndarray]] | None
    digest: int = 0
    counts: list[torch.Tensor] = field(default_factory=list, repr=False)
    prng: str = "splitmix"
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def epochs(self) -> int:
        return self.schedule.epochs

    def num_batches(self, e: int) -> int:
        return len(self.batch_seeds[e])

    def block(self, e: int, i: int) -> ComputationBlock:
        """Re-derive the full block, bit-identical to the original (plan.py:57-66)."""
        return sample_block(self.graph, self.batch_seeds[e][i], self.fanouts,
                            seed_for(self.schedule, e, i), epoch=e, batch=i, prng=self.prng)

    def digest_hex(self) -> str:
        return f"{self.digest:016x}"

    def counts_all(self) -> torch.Tensor:
        if "all" not in self._cache:
            tot = self.counts[0].clone()
            for c in self.counts[1:]:
                tot += c
            self._cache["all"] = tot
        return self._cache["all"]


class PlanPass:
    """Device plan pass for one graph/fanout/batch configuration: epoch
    permutation, grouped sampling of every batch, access counting."""

    def __init__(self, dg: DeviceGraph, train_nodes: np.ndarray, fanouts, batch_size: int,
                 s0: int, group: int = 16, prng: str = "splitmix"):
        self.dg = dg
        self.train = torch.from_numpy(np.ascontiguousarray(train_nodes, dtype=np.int32)).to(
            dg.device)
        self.n_train = int(self.train.numel())
        self.batch_size = int(batch_size)
        self.nb = -(-self.n_train // self.batch_size)
        self.s0 = int(s0)
        self.G = max(1, min(int(group), self.nb))
        self.prng = prng
        self.sampler = BlockSampler(dg, fanouts, self.batch_size, group=self.G, prng=prng)

    def permutation(self, schedule: SeedSchedule, e: int) -> torch.Tensor:
        return epoch_order_device(self.train, epoch_master(schedule, e))

    def fill(self, perm: torch.Tensor, e: int, i0: int, G: int, smp=None) -> None:
        smp = smp or self.sampler
        _lib.call("rg_fill_seeds", ptr(perm), self.n_train, self.batch_size, i0, G, ptr(smp.seeds),
                  ptr(smp.nseeds), smp.caps[0], self.s0 & (2**64 - 1), e, ptr(smp.rng),
                  _lib.stream_handle())

    def run_epoch(self, schedule: SeedSchedule, e: int, counts: torch.Tensor,
                  on_group=None, share: tuple[int, int] = (0, 1)) -> torch.Tensor:
        """Sample every batch of epoch e, add its input sets to counts.
        on_group(i0, ng) is called after each group (for host consumers).
        share = (rank, world): only every world-th group from `rank` (the
        caller sums the ranks' counts, e.g. one all-reduce)."""
        perm = self.permutation(schedule, e)
        smp, dg = self.sampler, self.dg
        rank, world = share
        for i0 in range(rank * self.G, self.nb, world * self.G):
            ng = min(self.G, self.nb - i0)
            self.fill(perm, e, i0, ng)
            smp.run(ng)
            _lib.call("rg_count_inputs", ptr(smp.bm), dg.nwords, ng, dg.n, ptr(counts),
                      _lib.stream_handle())
            if on_group is not None:
                on_group(i0, ng)
        return perm


def generate_plan(g, train_nodes: np.ndarray, fanouts: list[int], batch_size: int, epochs: int,
                  s0: int, keep_inputs: bool = True, group: int = 16,
                  prng: str = "splitmix") -> BatchPlan:
    """Precompute every epoch's batches and input sets (plan.py:72-105).

    keep_inputs=False skips the host copies of the input sets and the
    digest (which hashes them) — the device counts are always kept."""
    train_nodes = np.asarray(train_nodes, dtype=np.int64)
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    if len(train_nodes) == 0:
        raise ValueError("empty train set")
    batches_per_epoch = -(-len(train_nodes) // batch_size)
    schedule = SeedSchedule(s0=s0, epochs=epochs, batches_per_epoch=batches_per_epoch)
    dg = DeviceGraph.of(g)
    pp = PlanPass(dg, train_nodes, fanouts, batch_size, s0, group=group, prng=prng)
    h = hashlib.blake2b(digest_size=8)
    batch_seeds, input_sets, counts = [], [] if keep_inputs else None, []
    smp = pp.sampler
    L = smp.L
    for e in range(epochs):
        cnt = torch.zeros(dg.n, dtype=I32, device=dg.device)
        sets_e: list[np.ndarray] = []

        def grab(i0, ng, e=e, sets_e=sets_e):
            nf = smp.nfront[L, :ng].cpu().numpy()
            if int(nf.max()) > smp.caps[L]:
                raise RuntimeError("input set overflow")
            fr = smp.front[L][:ng].cpu().numpy()
            for b in range(ng):
                ids = fr[b, : nf[b]].astype(np.int64)
                sets_e.append(ids)
                h.update(np.array([e, i0 + b], dtype="<u8").tobytes())
                h.update(ids.astype("<u8").tobytes())

        perm = pp.run_epoch(schedule, e, cnt, on_group=grab if keep_inputs else None)
        perm_np = perm.cpu().numpy().astype(np.int64)
        batch_seeds.append([perm_np[i: i + batch_size] for i in range(0, len(perm_np), batch_size)])
        counts.append(cnt)
        if keep_inputs:
            input_sets.append(sets_e)
    digest = int.from_bytes(h.digest(), "little") if keep_inputs else 0
    return BatchPlan(graph=g, schedule=schedule, fanouts=list(fanouts), batch_seeds=batch_seeds,
                     input_sets=input_sets, digest=digest, counts=counts, prng=prng)


def _owner_u8(book, device) -> torch.Tensor:
    cache = book.__dict__.setdefault("_rg_owner", {})
    t = cache.get("u8")
    if t is None:
        t = torch.from_numpy(np.asarray(book.owner).astype(np.uint8)).to(device)
        cache["u8"] = t
    return t


def candidates(counts: torch.Tensor, owner_u8: torch.Tensor, my_part: int, max_count: int):
    """Remote nodes with count > 0: (ids device int32, n, count histogram)."""
    n = int(counts.numel())
    dev = counts.device
    nwords = (n + 31) // 32
    hist = torch.zeros(max_count + 1, dtype=I32, device=dev)
    bm = torch.empty(nwords, dtype=I32, device=dev)
    s = _lib.stream_handle()
    _lib.call("rg_count_histogram", ptr(counts), ptr(owner_u8), my_part, n, ptr(hist), max_count,
              ptr(bm), s)
    ids = torch.empty(max(n, 1), dtype=I32, device=dev)
    nout = torch.zeros(1, dtype=I32, device=dev)
    chunk = torch.empty(int(_lib.device().rg_bitmap_chunks(nwords)), dtype=I32, device=dev)
    _lib.call("rg_bitmap_compact", ptr(bm), nwords, 1, ptr(chunk), ptr(ids), n, ptr(nout), None, s)
    return ids, nout, hist, bm


def threshold_select(counts: torch.Tensor, bm_cand: torch.Tensor, hist: np.ndarray,
                     n_hot: int) -> torch.Tensor:
    """Device top_hot over a count array (index space = node or table index):
    returns the selected indices ascending (int32 device)."""
    n = int(counts.numel())
    dev = counts.device
    nwords = (n + 31) // 32
    n_cand = int(hist.sum())
    if n_hot <= 0:
        return torch.empty(0, dtype=I32, device=dev)
    if n_hot >= n_cand:
        n_hot = n_cand
    # c* = largest c with #{count >= c} >= n_hot
    suffix = np.cumsum(hist[::-1])[::-1]
    c_star = int(np.flatnonzero(suffix >= n_hot).max())
    n_above = int(suffix[c_star + 1]) if c_star + 1 < len(hist) else 0
    quota = n_hot - n_above
    s = _lib.stream_handle()
    bm_gt = torch.empty(nwords, dtype=I32, device=dev)
    bm_eq = torch.empty(nwords, dtype=I32, device=dev)
    _lib.call("rg_threshold_split", ptr(counts), ptr(bm_cand), n, c_star, ptr(bm_gt), ptr(bm_eq), s)
    lib = _lib.device()
    chunk = torch.empty(int(lib.rg_bitmap_chunks(nwords)), dtype=I32, device=dev)
    eq_ids = torch.empty(max(n, 1), dtype=I32, device=dev)
    n_eq = torch.zeros(1, dtype=I32, device=dev)
    _lib.call("rg_bitmap_compact", ptr(bm_eq), nwords, 1, ptr(chunk), ptr(eq_ids), n, ptr(n_eq),
              None, s)
    q = torch.tensor([quota], dtype=I32, device=dev)
    _lib.call("rg_bitmap_set", ptr(eq_ids), ptr(q), ptr(bm_gt), s)
    out = torch.empty(max(n_hot, 1), dtype=I32, device=dev)
    n_out = torch.zeros(1, dtype=I32, device=dev)
    _lib.call("rg_bitmap_compact", ptr(bm_gt), nwords, 1, ptr(chunk), ptr(out), n_hot, ptr(n_out),
              None, s)
    return out[:n_hot]


def collect_access(plan: BatchPlan, book, my_part: int, epoch: int | None = None
                   ) -> FrequencyTable:
    """Remote input-node appearances, one per batch (plan.py:117-130)."""
    if not isinstance(plan, BatchPlan) or not plan.counts:
        raise TypeError("collect_access needs a plan from paper_2505_10806_b200.generate_plan")
    counts = plan.counts_all() if epoch is None else plan.counts[epoch]
    owner = _owner_u8(book, counts.device)
    max_count = sum(plan.num_batches(e) for e in range(plan.epochs))
    ids, nout, _, _ = candidates(counts, owner, my_part, max(1, max_count))
    k = int(nout.item())
    ids = ids[:k]
    cnt = torch.empty(max(k, 1), dtype=I32, device=counts.device)
    _lib.call("rg_gather_counts", ptr(counts), ptr(ids), ptr(nout), k, ptr(cnt),
              _lib.stream_handle())
    return FrequencyTable(ids=ids.cpu().numpy().astype(np.int64),
                          counts=cnt[:k].cpu().numpy().astype(np.int64))


def top_hot(freq: FrequencyTable, n_hot: int) -> np.ndarray:
    """The n_hot most-accessed remote nodes, ties to the lower id, sorted
    ascending (plan.py:133-141)."""
    if n_hot < 0:
        raise ValueError("n_hot must be >= 0")
    if n_hot >= len(freq.ids):
        return np.asarray(freq.ids).copy()
    if n_hot == 0:
        return np.empty(0, dtype=np.int64)
    counts_np = np.asarray(freq.counts, dtype=np.int64)
    if counts_np.min() < 1 or counts_np.max() >= 2**31:
        raise ValueError("frequency counts must be in [1, 2^31)")
    _lib.device()
    dev = torch.device("cuda")
    counts = torch.from_numpy(counts_np.astype(np.int32)).to(dev)
    m = len(counts_np)
    everyone = torch.zeros(m, dtype=torch.uint8, device=dev)  # owner 0, my_part -1
    max_count = int(counts_np.max())
    hist = torch.zeros(max_count + 1, dtype=I32, device=dev)
    bm = torch.empty((m + 31) // 32, dtype=I32, device=dev)
    _lib.call("rg_count_histogram", ptr(counts), ptr(everyone), -1, m, ptr(hist), max_count,
              ptr(bm), _lib.stream_handle())
    sel = threshold_select(counts, bm, hist.cpu().numpy().astype(np.int64), n_hot)
    return np.asarray(freq.ids)[sel.cpu().numpy().astype(np.int64)]
