"""Device engine: HBM-resident graph, group sampler, feature store, gather.

Everything here is plumbing around the C ABI (include/rapidgnn_b200.h):
torch provides device memory and the current CUDA stream, every compute
step is one of the library's sm_100a kernels.  All work of one call is
enqueued on torch's current stream without host synchronisation, so a
whole group (sample L levels + gather) can be captured in a CUDA graph.

Data layout:
  indptr   int64[n+1]        indices int32[E]
  owner    uint8[n]          route   uint32[n] = owner<<28 | row in shard
  shard q  float32[n_q, stride]  (stride = feat_dim rounded up to 4)
  cache    float32[n_hot, stride]; cache route = route with hot ids
           rewritten to (15<<28 | slot)
  group buffers: G slots per level; slot b of level d at b*cap_d.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import ptr

I32 = torch.int32


def stride_for(d: int) -> int:
    """Dense row stride (floats) of bundles: d rounded up to 16 bytes."""
    return max(4, (d + 3) // 4 * 4)


# Shard/cache row alignment.  Measured (tools/nvlink_probe.py, round 1):
# 128-byte-aligned 400-B rows gained only +1-2 % on local and peer gathers and
# lost 1 % in the full bench, so rows stay dense (16-byte aligned); the
# separate source stride remains available.
SRC_ALIGN_FLOATS = 4


def src_stride_for(d: int) -> int:
    """Row stride (floats) of shards and cache rows."""
    a = SRC_ALIGN_FLOATS
    return max(4, (d + a - 1) // a * a)


def _cur() -> int:
    return _lib.stream_handle()


def rows_sorted(indptr: np.ndarray, indices: np.ndarray) -> bool:
    """True if every CSR row is nondecreasing (lets the sampler skip its sort)."""
    indices = np.asarray(indices)
    if len(indices) < 2:
        return True
    desc = np.flatnonzero(np.diff(indices.astype(np.int64)) < 0) + 1
    if len(desc) == 0:
        return True
    # a decrease is allowed only where a new row starts
    starts = np.asarray(indptr, dtype=np.int64)
    return bool(np.isin(desc, starts).all())


class DeviceGraph:
    """CSR graph in HBM: indptr int64, indices int32 (ids < 2^31)."""

    def __init__(self, indptr: np.ndarray, indices: np.ndarray, num_nodes: int, device=None):
        _lib.device()
        if num_nodes >= 2**31 - 1:
            raise NotImplementedError("node ids must fit in int32")
        self.device = torch.device(device or "cuda")
        self.n = int(num_nodes)
        self.nwords = (self.n + 31) // 32
        self.indptr = torch.from_numpy(np.ascontiguousarray(indptr, dtype=np.int64)).to(self.device)
        self.indices = torch.from_numpy(np.ascontiguousarray(indices, dtype=np.int32)).to(self.device)
        self.num_edges = int(self.indices.numel())
        self.sorted_rows = rows_sorted(indptr, indices)
        self.max_degree = int(np.diff(np.asarray(indptr)).max()) if self.n else 0

    @classmethod
    def from_device(cls, indptr: torch.Tensor, indices: torch.Tensor,
                    num_nodes: int) -> "DeviceGraph":
        """Adopt a CSR already in HBM (formats.load_graph_device): int64
        indptr, int32 indices; row order and max degree found on the device."""
        _lib.device()
        dg = cls.__new__(cls)
        dg.device = indptr.device
        dg.n = int(num_nodes)
        dg.nwords = (dg.n + 31) // 32
        dg.indptr = indptr.contiguous()
        dg.indices = indices.contiguous()
        dg.num_edges = int(indices.numel())
        deg = indptr[1:] - indptr[:-1]
        dg.max_degree = int(deg.max().item()) if dg.n else 0
        if dg.num_edges > 1:
            dec = torch.nonzero(indices[1:] < indices[:-1]).flatten() + 1
            start = torch.zeros(dg.num_edges + 1, dtype=torch.bool, device=dg.device)
            start[indptr[1:-1]] = True
            dg.sorted_rows = bool(start[dec].all().item()) if dec.numel() else True
        else:
            dg.sorted_rows = True
        return dg

    @classmethod
    def of(cls, g) -> "DeviceGraph":
        """Device copy of a Graph (ours or the reference's), cached on it."""
        cached = getattr(g, "_rg_device", None)
        if cached is not None and cached[0] is g.indptr and cached[1] is g.indices:
            return cached[2]
        dg = cls(g.indptr, g.indices, g.num_nodes)
        try:
            object.__setattr__(g, "_rg_device", (g.indptr, g.indices, dg))
        except AttributeError:
            pass
        return dg


class BlockSampler:
    """Samples up to G mini-batches per run() (sampler.py:116-152).

    Level d of slot b lives at front[d][b, :nfront[d, b]] (sorted unique
    ids), its sampled edges as ELL rows ell[d][b, j*F_d : j*F_d+cnt[d][b,j]]
    (ascending src, dst = front[d][b, j]).  front[L] is the input node set.
    """

    def __init__(self, dg: DeviceGraph, fanouts, seed_cap: int, group: int = 1,
                 prng: str = "splitmix"):
        if len(fanouts) == 0:
            raise ValueError("fanouts must be nonempty")
        if any(int(f) < 1 for f in fanouts):
            raise ValueError("fanouts must be >= 1")
        if prng not in _lib.PRNG_KINDS:
            raise ValueError(f"unknown prng {prng!r} (one of {sorted(_lib.PRNG_KINDS)})")
        self.prng = prng
        self.prng_code = _lib.PRNG_KINDS[prng]
        self.dg = dg
        self.G = int(group)
        self.L = len(fanouts)
        self.fanouts = [int(f) for f in fanouts]
        self.step_fan = [self.fanouts[self.L - 1 - d] for d in range(self.L)]
        caps = [int(seed_cap)]
        for f in self.step_fan:
            caps.append(min(dg.n, caps[-1] * (1 + f)))
        self.caps = caps
        dev, G = dg.device, self.G
        self.seeds = torch.zeros((G, caps[0]), dtype=I32, device=dev)
        self.nseeds = torch.zeros(G, dtype=I32, device=dev)
        self.rng = torch.zeros(G, dtype=torch.int64, device=dev)  # uint64 bits
        self.front = [torch.empty((G, c), dtype=I32, device=dev) for c in caps]
        self.nfront = torch.zeros((self.L + 1, G), dtype=I32, device=dev)
        self.ell = [torch.empty((G, caps[d] * self.step_fan[d]), dtype=I32, device=dev)
                    for d in range(self.L)]
        self.cnt = [torch.empty((G, caps[d]), dtype=I32, device=dev) for d in range(self.L)]
        self.bm = torch.empty((G, dg.nwords), dtype=I32, device=dev)
        # rank of node 32w in each batch's input set (level L): drives the
        # id-window-major bundle gather (rg_gather_window)
        self.wpre = torch.empty((G, dg.nwords), dtype=I32, device=dev)
        lib = _lib.device()
        self.chunk = torch.empty((G, int(lib.rg_bitmap_chunks(dg.nwords))), dtype=I32, device=dev)
        self.slow = (torch.empty(1 + G * max(caps[:-1]), dtype=I32, device=dev)
                     if max(self.step_fan) > 32 else None)
        # per-slot (row start, degree, id) records for the sampler (16 B each)
        # (+1 record: the sampler's launch-wide work-queue counter)
        self.meta = torch.empty((G * max(caps[:-1]) + 1, 4), dtype=I32, device=dev)

    def set_seeds(self, b: int, seeds: np.ndarray, rng_seed: int) -> None:
        """Host seeds for slot b (API path; the plan path fills on device):
        one H2D copy of [seeds | count | rng seed], then device-side scatter."""
        seeds = np.asarray(seeds)
        n = len(seeds)
        if n > self.caps[0]:
            raise ValueError(f"{n} seeds exceed the sampler capacity {self.caps[0]}")
        host = np.empty(n + 3, dtype=np.int32)  # [rng seed (2 words) | count | seeds]
        host[0:2] = np.array([rng_seed & (2**64 - 1)], dtype=np.uint64).view(np.int32)
        host[2] = n
        host[3:] = seeds
        dev = torch.from_numpy(host).to(self.dg.device)
        self.rng[b: b + 1].copy_(dev[0:2].view(torch.int64))
        self.nseeds[b: b + 1].copy_(dev[2:3])
        self.seeds[b, :n].copy_(dev[3:])

    def run(self, ngroup: int | None = None, b0: int = 0) -> None:
        """Sample all L levels for slots [b0, ngroup) on the current stream
        (b0 > 0: one rank's share of a group under shared sampling; every
        per-slot array is slot-major, so the share is a pointer offset)."""
        G = (self.G if ngroup is None else int(ngroup)) - int(b0)
        if G <= 0:
            return
        dg, s = self.dg, _cur()

        def o(t):  # slot b0 of a slot-major tensor
            return ptr(t) + int(b0) * t.stride(0) * t.element_size()

        nf = [ptr(self.nfront) + 4 * (d * self.G + int(b0)) for d in range(self.L + 1)]
        self.bm[b0:b0 + G].zero_()
        _lib.call("rg_mark_seeds", o(self.seeds), o(self.nseeds), G, self.caps[0],
                  o(self.bm), dg.nwords, s)
        _lib.call("rg_bitmap_compact", o(self.bm), dg.nwords, G, ptr(self.chunk),
                  o(self.front[0]), self.caps[0], nf[0], None, s)
        for d in range(self.L):
            _lib.call("rg_sample_level", ptr(dg.indptr), ptr(dg.indices), dg.n, G,
                      o(self.front[d]), self.caps[d], nf[d], self.step_fan[d], d,
                      o(self.rng), o(self.ell[d]), o(self.cnt[d]), o(self.bm), dg.nwords,
                      ptr(self.slow), ptr(self.meta), int(dg.sorted_rows), self.prng_code, s)
            _lib.call("rg_bitmap_compact", o(self.bm), dg.nwords, G, ptr(self.chunk),
                      o(self.front[d + 1]), self.caps[d + 1], nf[d + 1],
                      o(self.wpre) if d == self.L - 1 else None, s)

    def edges(self, d: int, ngroup: int | None = None):
        """Flat (src, dst) of level d for every slot: (src, dst, nedge) device."""
        G = self.G if ngroup is None else int(ngroup)
        F, cap = self.step_fan[d], self.caps[d]
        dev = self.dg.device
        cap_e = cap * F
        src = torch.empty((G, cap_e), dtype=I32, device=dev)
        dst = torch.empty((G, cap_e), dtype=I32, device=dev)
        eoff = torch.empty((G, cap + 1), dtype=I32, device=dev)
        nedge = torch.empty(G, dtype=I32, device=dev)
        lib = _lib.device()
        chunk = torch.empty((G, int(lib.rg_scan_chunks(cap))), dtype=I32, device=dev)
        _lib.call("rg_ell_to_edges", ptr(self.front[d]), ptr(self.nfront[d]), cap,
                  ptr(self.ell[d]), ptr(self.cnt[d]), F, G, ptr(chunk), ptr(eoff), ptr(src),
                  ptr(dst), cap_e, ptr(nedge), _cur())
        return src, dst, nedge


def route_table(owner: np.ndarray, shard_ids: list[np.ndarray | None]) -> np.ndarray:
    """uint32 route words: owner<<28 | row of v inside its owner's shard.
    Nodes whose owner shard does not hold them get RG_ROUTE_INVALID
    (a pull for them is NOT_OWNED, store.py:186-187)."""
    owner = np.asarray(owner).astype(np.int64)
    n = len(owner)
    route = np.full(n, _lib.RG_ROUTE_INVALID, dtype=np.uint32)
    for q, ids in enumerate(shard_ids):
        if ids is None or len(ids) == 0:
            continue
        ids = np.asarray(ids, dtype=np.int64)
        if len(ids) > _lib.RG_ROW_MASK:
            raise NotImplementedError("shard larger than 2^28 rows")
        mine = ids[(ids >= 0) & (ids < n)]
        ok = owner[mine] == q
        rows = np.flatnonzero((ids >= 0) & (ids < n))[ok]
        route[ids[rows]] = (np.uint32(q) << np.uint32(_lib.RG_KIND_SHIFT)) | rows.astype(np.uint32)
    return route


def as_i32_bits(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32))


class FeatureStore:
    """All partition shards this GPU can address (local HBM or peer).

    shards[q] is a float32 (n_q, stride) tensor or None; bases[q] its device
    address (may be an NVLink peer address opened over CUDA IPC)."""

    def __init__(self, owner: np.ndarray, num_parts: int, feat_dim: int, device=None):
        _lib.device()
        if num_parts > _lib.RG_MAX_PARTS:
            raise NotImplementedError(f"at most {_lib.RG_MAX_PARTS} partitions")
        self.device = torch.device(device or "cuda")
        self.k = int(num_parts)
        self.d = int(feat_dim)
        self.stride = stride_for(self.d)  # bundle rows
        self.src_stride = src_stride_for(self.d)  # shard / cache rows
        self.owner_np = np.asarray(owner)
        self.n = len(self.owner_np)
        self.owner = torch.from_numpy(self.owner_np.astype(np.uint8)).to(self.device)
        self.shards: list[torch.Tensor | None] = [None] * self.k
        self.bases = [0] * 16
        self.route = None
        self.peer_mask = 0  # bit q: shard q is another GPU's memory (NVLink)

    def set_shard(self, q: int, rows: torch.Tensor | None, base: int | None = None) -> None:
        self.shards[q] = rows
        self.bases[q] = int(base if base is not None else (rows.data_ptr() if rows is not None else 0))
        if rows is None and base:
            self.peer_mask |= 1 << q
        else:
            self.peer_mask &= ~(1 << q)

    def build_route(self, shard_ids: list[np.ndarray | None]) -> None:
        self.route = as_i32_bits(route_table(self.owner_np, shard_ids)).to(self.device)

    @staticmethod
    def pad_rows(rows: np.ndarray, stride: int, device) -> torch.Tensor:
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        t = torch.zeros((rows.shape[0], stride), dtype=torch.float32, device=device)
        if rows.size:
            t[:, : rows.shape[1]].copy_(torch.from_numpy(rows))
        return t


def bases_array(bases) -> np.ndarray:
    a = np.zeros(16, dtype=np.uint64)
    a[: len(bases)] = [int(b) for b in bases]
    return a


def gather_bundle(ids: torch.Tensor, nids: torch.Tensor, cap: int, G: int, route: torch.Tensor,
                  bases: np.ndarray, src_stride: int, stride: int, my_part: int,
                  out: torch.Tensor, counters: torch.Tensor, peer_mask: int = 0) -> None:
    """rg_gather_bundle on the current stream (bases: host uint64[16])."""
    _lib.call("rg_gather_bundle", ptr(ids), ptr(nids), cap, G, ptr(route), bases.ctypes.data,
              src_stride, stride, my_part, peer_mask, ptr(out), ptr(counters), _cur())


def gather_rows(base: torch.Tensor, row_idx: np.ndarray | torch.Tensor, stride: int,
                out_stride: int | None = None) -> torch.Tensor:
    """out[i] = base[row_idx[i]] (base rows of `stride` floats) via the bundle
    kernel with an identity route; out rows have out_stride <= stride floats."""
    out_stride = stride if out_stride is None else out_stride
    dev = base.device
    idx = (torch.from_numpy(np.ascontiguousarray(row_idx, dtype=np.int32)).to(dev)
           if isinstance(row_idx, np.ndarray) else row_idx.to(torch.int32))
    n = int(idx.numel())
    out = torch.empty((max(n, 1), out_stride), dtype=torch.float32, device=dev)
    if n == 0:
        return out[:0]
    # route: kind 0 | row index, ids 0..n-1 index the route directly
    route = idx  # row index < 2^28, kind bits zero => shard 0
    ids = torch.arange(n, dtype=I32, device=dev)
    nids = torch.tensor([n], dtype=I32, device=dev)
    bases = bases_array([base.data_ptr()])
    counters = torch.zeros((1, _lib.RG_NCOUNTERS), dtype=I32, device=dev)
    gather_bundle(ids, nids, n, 1, route, bases, stride, out_stride, 0, out, counters)
    return out
