"""Drop-in for gnnpipe.sampler (sampler.py:23-152) on the B200.

Same names, signatures, return types and exceptions as the reference; the
work runs in the sm_100a kernels of librapidgnn_b200 (rg_stream_keys for the
epoch shuffle keys, rg_sample_level / rg_bitmap_compact for the L-hop
expansion).  Results are bit-identical to the reference.
"""

from __future__ import annotations

import threading
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .engine import BlockSampler, DeviceGraph
from .rng import MASK64, mix64

_SHUFFLE_TAG = 0x73687566  # sampler.py:20


@dataclass(frozen=True)
class SeedSchedule:
    """Injective (epoch, batch) -> 64-bit seed map (sampler.py:23-29)."""

    s0: int
    epochs: int
    batches_per_epoch: int


def seed_for(s: SeedSchedule, e: int, i: int) -> int:
    """mix64(s0 ^ (e<<32 | i)); IndexError outside the schedule (sampler.py:32-40)."""
    if not (0 <= e < s.epochs and 0 <= i < s.batches_per_epoch):
        raise IndexError(f"(e={e}, i={i}) outside schedule")
    return mix64(s.s0 ^ ((e << 32) | i))


def epoch_order_device(train_nodes: torch.Tensor, master: int) -> torch.Tensor:
    """Keyed permutation on device (rng.py:53-62): per-position counter keys
    from rg_stream_keys, then a stable ascending sort of the keys.  The keys
    are uint64; flipping the top bit maps unsigned order to int64 order."""
    n = int(train_nodes.numel())
    keys = torch.empty(n, dtype=torch.int64, device=train_nodes.device)
    _lib.call("rg_stream_keys", master & MASK64, n, keys.data_ptr(), _lib.stream_handle())
    keys ^= torch.tensor(-(2**63), dtype=torch.int64, device=keys.device)
    order = torch.sort(keys, stable=True).indices
    return train_nodes[order]


def epoch_master(s: SeedSchedule, e: int) -> int:
    return mix64(seed_for(s, e, 0) ^ _SHUFFLE_TAG)


def epoch_batches(train_nodes: np.ndarray, batch_size: int, s: SeedSchedule,
                  e: int) -> list[np.ndarray]:
    """Shuffle the train set with this epoch's seed and chunk it (sampler.py:43-57)."""
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    if len(train_nodes) == 0:
        raise ValueError("empty train set")
    tn = torch.from_numpy(np.ascontiguousarray(train_nodes, dtype=np.int64)).cuda()
    perm = epoch_order_device(tn, epoch_master(s, e)).cpu().numpy()
    return [perm[i: i + batch_size] for i in range(0, len(perm), batch_size)]


class DeviceEdges(Sequence):
    """edges[d] = (src, dst) int64 arrays, copied from the device on first
    access: the flat (dst, src)-sorted edge lists are built on the device when
    the block is made (rg_ell_to_edges, fresh buffers) and stay there until a
    host consumer reads them — the reference's Prefetcher consumer reads only
    the bundle rows, the device model reads the ELL form."""

    def __init__(self, parts: list, L: int):
        self._parts = parts  # [(src view, dst view)] device int32, per level
        self._L = L
        self._host = None

    def _get(self):
        if self._host is None:
            flat = torch.cat([t for pair in self._parts for t in pair])
            host = torch.empty(flat.shape, dtype=flat.dtype, pin_memory=True)
            host.copy_(flat)
            out = host.numpy().astype(np.int64)
            cuts = np.cumsum([int(t.numel()) for pair in self._parts for t in pair])[:-1]
            pieces = np.split(out, cuts)
            self._host = [(pieces[2 * d], pieces[2 * d + 1]) for d in range(self._L)]
            self._parts = None
        return self._host

    def __len__(self) -> int:
        return self._L

    def __getitem__(self, i):
        return self._get()[i]


@dataclass
class ComputationBlock:
    """Layered subgraph of one mini-batch (sampler.py:60-83).

    frontiers[0] is the sorted unique seed set, frontiers[d+1] extends
    frontiers[d] with step d's neighbours; edges[d] = (src, dst) sorted by
    (dst, src).  ``device`` holds the device-resident form (the sampler
    slot) when the block came from the GPU, so consumers can skip the
    host round trip."""

    epoch: int
    batch: int
    seeds: np.ndarray
    frontiers: list[np.ndarray]
    edges: list[tuple[np.ndarray, np.ndarray]]
    device: dict | None = field(default=None, repr=False, compare=False)

    @property
    def input_nodes(self) -> np.ndarray:
        return self.frontiers[-1]

    @property
    def num_layers(self) -> int:
        return len(self.edges)


def _sampler_for(dg: DeviceGraph, fanouts, n_seeds: int, prng: str = "splitmix") -> BlockSampler:
    """Per-thread cached sampler (its device buffers are per-call scratch,
    so concurrent callers — e.g. the Prefetcher's producer thread and the
    consumer — must not share one)."""
    cap = 1
    while cap < n_seeds:
        cap <<= 1
    key = (tuple(int(f) for f in fanouts), cap, prng, threading.get_ident())
    cache = dg.__dict__.setdefault("_samplers", {})
    smp = cache.get(key)
    if smp is None:
        if len(cache) > 16:
            cache.clear()
        smp = BlockSampler(dg, fanouts, cap, group=1, prng=prng)
        cache[key] = smp
    return smp


def block_from_sampler(smp: BlockSampler, slot: int, seeds: np.ndarray, epoch: int,
                       batch: int) -> ComputationBlock:
    """Materialise slot `slot` of a sampler run as a numpy ComputationBlock:
    flat edges per level built on the device (kept there until read, see
    DeviceEdges), one D2H of the sizes, one packed D2H of the frontiers."""
    L = smp.L
    lv = [smp.edges(d, slot + 1) for d in range(L)]
    sizes = torch.cat([smp.nfront[:, slot]] + [e[2][slot:slot + 1] for e in lv]).cpu().numpy()
    nf, ne = sizes[:L + 1], sizes[L + 1:]
    for d in range(L + 1):
        if nf[d] > smp.caps[d]:
            raise RuntimeError(f"frontier {d} overflow ({nf[d]} > {smp.caps[d]})")
    parts = [smp.front[d][slot, : nf[d]] for d in range(L + 1)]
    flat = torch.cat(parts)
    host = torch.empty(flat.shape, dtype=flat.dtype, pin_memory=True)
    host.copy_(flat)
    out = host.numpy().astype(np.int64)
    frontiers = np.split(out, np.cumsum([int(p.numel()) for p in parts])[:-1])
    edges = DeviceEdges([(lv[d][0][slot, : ne[d]], lv[d][1][slot, : ne[d]]) for d in range(L)],
                        L)
    input_dev = parts[L].clone()
    return ComputationBlock(epoch=epoch, batch=batch, seeds=seeds, frontiers=frontiers,
                            edges=edges, device={"input_nodes": input_dev})


def sample_block(g, seeds: np.ndarray, fanouts: list[int], rng_seed: int, epoch: int = 0,
                 batch: int = 0, prng: str = "splitmix") -> ComputationBlock:
    """Build the computation block for one batch of seed nodes (sampler.py:116-152).

    fanouts are listed input layer first: expansion step d uses
    fanouts[len(fanouts)-1-d].  prng selects the neighbour-selection
    generator: "splitmix" (the reference's SplitMix64 keys, default) or the
    variants "pcg32" / "sfc64" / "xoshiro256pp"."""
    if len(fanouts) == 0:
        raise ValueError("fanouts must be nonempty")
    seeds = np.asarray(seeds, dtype=np.int64)
    if len(seeds) == 0:
        raise ValueError("seeds must be nonempty")
    if seeds.min() < 0 or seeds.max() >= g.num_nodes:
        raise ValueError("seed id out of range")
    dg = DeviceGraph.of(g)
    smp = _sampler_for(dg, fanouts, len(seeds), prng)
    smp.set_seeds(0, seeds, rng_seed)
    smp.run(1)
    return block_from_sampler(smp, 0, seeds, epoch, batch)
