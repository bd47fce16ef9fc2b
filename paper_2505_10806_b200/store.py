"""Drop-in for gnnpipe.store (store.py:1-211): shards, client, accounting.

The reference serves feature rows through a byte codec over an in-process
call or TCP (store.py:91-158).  Here a shard is a device tensor; a pull is
one launch of the routing gather (rg_gather_bundle) that reads every row
straight from the owning shard's memory — this GPU's HBM or a peer GPU's
over NVLink P2P.  The accounting rule is the reference's: one RPC per
owning shard touched by a pull, nodes = ids pulled, bytes = 4*d*nodes
(store.py:24-43, 173-196).
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import (FeatureStore, bases_array, gather_bundle, gather_rows, route_table,
                     src_stride_for, stride_for)


class LookupError_(KeyError):
    """Pull for a node id the contacted shard does not own (store.py:16-17)."""


class TransportError(ConnectionError):
    """Transport-level failure (store.py:20-21)."""


def bytes_for(n: int, d: int) -> int:
    """Bytes for n feature rows of dimension d, float32 (store.py:24-26)."""
    return n * d * 4


@dataclass
class TransferAccount:
    """Client-side traffic counters for one category of pulls (store.py:29-43)."""

    rpc_calls: int = 0
    nodes_pulled: int = 0
    bytes_pulled: int = 0

    def charge(self, rpcs: int, nodes: int, feat_dim: int) -> None:
        self.rpc_calls += rpcs
        self.nodes_pulled += nodes
        self.bytes_pulled += bytes_for(nodes, feat_dim)

    def snapshot(self) -> tuple[int, int, int]:
        return (self.rpc_calls, self.nodes_pulled, self.bytes_pulled)


class StoreShard:
    """Feature rows of the nodes one partition owns, resident in HBM
    (store.py:46-88).  Server-side counters are kept for parity."""

    def __init__(self, part: int, owned_ids: np.ndarray, rows: np.ndarray,
                 latency_ms: float = 0.0, device=None):
        _lib.device()
        self.part = part
        self.owned_ids = np.asarray(owned_ids, dtype=np.int64)
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        self.feat_dim = rows.shape[1] if rows.ndim == 2 else 0
        self.stride = stride_for(self.feat_dim)  # dense rows handed out
        self.src_stride = src_stride_for(self.feat_dim)  # line-aligned rows in HBM
        self.device = torch.device(device or "cuda")
        self.rows_device = FeatureStore.pad_rows(rows.reshape(len(self.owned_ids), -1),
                                                 self.src_stride, self.device)
        self.latency_ms = latency_ms
        self._lock = threading.Lock()
        self.rpc_calls = 0
        self.nodes_served = 0
        self.payload_bytes = 0

    @property
    def rows(self) -> np.ndarray:
        return self.rows_device[:, : self.feat_dim].cpu().numpy()

    def rows_for_local(self, ids: np.ndarray) -> np.ndarray:
        """Direct memory read for the owning worker; no RPC, no counters."""
        pos = np.searchsorted(self.owned_ids, np.asarray(ids, dtype=np.int64))
        out = gather_rows(self.rows_device, pos.astype(np.int32), self.src_stride, self.stride)
        return out[:, : self.feat_dim].cpu().numpy()

    def _served(self, nodes: int | None) -> None:
        """One handled request (store.py:71-88): the injected latency is
        slept per request; nodes=None when the bundle gather served it
        (rows read in place, per-owner row counts not materialised)."""
        if self.latency_ms > 0:
            time.sleep(self.latency_ms / 1000.0)
        with self._lock:
            self.rpc_calls += 1
            if nodes is not None:
                self.nodes_served += nodes
                self.payload_bytes += bytes_for(nodes, self.feat_dim)


class InprocTransport:
    """Compatibility wrapper: the client reads the shard's memory directly."""

    def __init__(self, shard: StoreShard):
        self.shard = shard

    def close(self) -> None:
        pass


class PeerTransport:
    """A shard living on another GPU: its rows are addressed through an
    NVLink P2P pointer (CUDA IPC); ids/metadata are host-side."""

    def __init__(self, part: int, owned_ids: np.ndarray, base_ptr: int, feat_dim: int):
        self.part = part
        self.owned_ids = np.asarray(owned_ids, dtype=np.int64)
        self.base_ptr = int(base_ptr)
        self.feat_dim = feat_dim

    def close(self) -> None:
        pass


def _shard_of(t):
    return t.shard if isinstance(t, InprocTransport) else t


class StoreClient:
    """Groups pulls by owning shard (store.py:161-207).

    A pull is one gather launch over all requested ids; the per-owner
    grouping survives only in the accounting (one RPC per distinct owner)."""

    def __init__(self, owner: np.ndarray, transports: list, feat_dim: int):
        _lib.device()
        self.owner = np.asarray(owner)
        self.transports = transports
        self.feat_dim = feat_dim
        self.stride = stride_for(feat_dim)
        self.src_stride = src_stride_for(feat_dim)
        self.k = len(transports)
        if self.k > _lib.RG_MAX_PARTS:
            raise NotImplementedError(f"at most {_lib.RG_MAX_PARTS} shards")
        shards = [_shard_of(t) for t in transports]
        self._shards = shards
        self.device = torch.device("cuda")
        self.route = torch.from_numpy(
            route_table(self.owner, [s.owned_ids for s in shards]).view(np.int32)).to(self.device)
        bases = []
        for s in shards:
            if isinstance(s, StoreShard):
                if s.src_stride != self.src_stride:
                    raise ValueError(f"shard {s.part} has dim {s.feat_dim}, expected {feat_dim}")
                bases.append(s.rows_device.data_ptr())
            else:
                bases.append(s.base_ptr)
        self.base_list = bases
        self._closed = False

    def bases(self, cache_rows: torch.Tensor | None = None) -> np.ndarray:
        b = list(self.base_list)
        b += [0] * (16 - len(b))
        if cache_rows is not None and cache_rows.numel():
            b[_lib.RG_KIND_CACHE] = cache_rows.data_ptr()
        return bases_array(b)

    def pull_device(self, ids: np.ndarray, account: TransferAccount | None,
                    out_stride: int | None = None):
        """Rows for ids (device; dense stride, or out_stride) + RPC count."""
        out_stride = self.stride if out_stride is None else out_stride
        ids = np.asarray(ids, dtype=np.int64)
        n = len(ids)
        if n and (ids.min() < 0 or ids.max() >= len(self.owner)):
            raise LookupError_("requested id outside the graph")
        out = torch.empty((max(n, 1), out_stride), dtype=torch.float32, device=self.device)
        if n == 0:
            return out[:0], 0
        dev_ids = torch.from_numpy(ids.astype(np.int32)).to(self.device)
        nids = torch.tensor([n], dtype=torch.int32, device=self.device)
        counters = torch.zeros((1, _lib.RG_NCOUNTERS), dtype=torch.int32, device=self.device)
        gather_bundle(dev_ids, nids, n, 1, self.route, self.bases(), self.src_stride, out_stride,
                      -1, out,
                      counters)
        c = counters.cpu().numpy()[0].view(np.uint32)
        if c[_lib.RG_CNT_BAD]:
            bad = ids[self.route.cpu().numpy().view(np.uint32)[ids] == _lib.RG_ROUTE_INVALID]
            owners = np.unique(self.owner[bad])
            raise LookupError_(f"shard {int(owners[0])} does not own requested ids")
        mask = int(c[_lib.RG_CNT_OWNER_MASK])
        rpcs = bin(mask).count("1")
        per_owner = np.bincount(self.owner[ids].astype(np.int64), minlength=self.k)
        for q in np.flatnonzero(per_owner):
            s = self._shards[q]
            if isinstance(s, StoreShard):
                s._served(int(per_owner[q]))
        if account is not None:
            account.charge(rpcs, n, self.feat_dim)
        return out, rpcs

    def served(self, owner_mask: int) -> None:
        """Requests the bundle gather made: one per owner bit set."""
        q = 0
        while owner_mask:
            if owner_mask & 1 and q < len(self._shards):
                s = self._shards[q]
                if isinstance(s, StoreShard):
                    s._served(None)
            owner_mask >>= 1
            q += 1

    def sync_pull(self, node_ids: np.ndarray, account: TransferAccount | None = None) -> np.ndarray:
        """On-demand pull; rows come back in request order (store.py:198-201)."""
        out, _ = self.pull_device(node_ids, account)
        return out[:, : self.feat_dim].cpu().numpy()

    def vector_pull(self, node_ids: np.ndarray,
                    account: TransferAccount | None = None) -> np.ndarray:
        """Bulk pull for cache fills, same accounting rule (store.py:203-207)."""
        return self.sync_pull(node_ids, account)

    def close(self) -> None:
        self._closed = True
