"""One process per GPU: shard placement and NVLink peer mapping.

Worker p runs on GPU p mod N and partition shard q lives on GPU q mod N
(SURVEY.md §8e).  No collective sits on the data path: every process maps
the other GPUs' shards into its address space once (CUDA IPC handles,
exchanged with torch.distributed.all_gather_object), and the bundle gather
then reads remote rows with plain loads that travel over NVLink 5 /
NVSwitch — the one-sided equivalent of the reference's per-owner pull RPC
(store.py:173-196), still charged one RPC per owner touched.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_opened: dict = {}  # (rank, handle bytes) -> base address (one mapping per allocation)


def _open(rank: int, hb: bytes) -> int:
    key = (rank, hb)
    if key not in _opened:
        p = ctypes.c_void_p()
        buf = np.frombuffer(hb, dtype=np.uint8).copy()
        _lib.call("rg_ipc_open", buf.ctypes.data, ctypes.byref(p))
        _opened[key] = int(p.value)
    return _opened[key]


def placement(k: int, world: int) -> dict[int, int]:
    """partition q -> rank holding its shard."""
    return {q: q % world for q in range(k)}


def workers_of(rank: int, k: int, world: int) -> list[int]:
    """Workers (partitions) a rank runs: p with p mod world == rank."""
    return [p for p in range(k) if p % world == rank]


def shard_handles(store) -> dict[int, tuple[bytes, int]]:
    """IPC handle + offset of every shard this process holds."""
    out = {}
    for q, t in enumerate(store.shards):
        if t is None:
            continue
        h = np.zeros(64, dtype=np.uint8)
        off = np.zeros(1, dtype=np.int64)
        _lib.call("rg_ipc_handle", t.data_ptr(), h.ctypes.data, off.ctypes.data)
        out[q] = (h.tobytes(), int(off[0]))
    return out


def open_peer_shards(store, gathered: list[dict], rank: int) -> list[int]:
    """Map every other rank's shards; returns the opened base pointers."""
    opened = []
    for r, handles in enumerate(gathered):
        if r == rank:
            continue
        for q, (hb, off) in handles.items():
            if store.shards[q] is not None:
                continue
            base = _open(r, hb)
            opened.append(base)
            store.set_shard(q, None, base=base + off)
    return opened


def exchange_buffers(tensors: list, rank: int, world: int) -> list[list[int]]:
    """Map every rank's buffers: returns ptrs[i][r] = address of rank r's
    tensors[i] in this process (own entries are the local addresses)."""
    import torch.distributed as dist

    mine = []
    for t in tensors:
        h = np.zeros(64, dtype=np.uint8)
        off = np.zeros(1, dtype=np.int64)
        _lib.call("rg_ipc_handle", t.data_ptr(), h.ctypes.data, off.ctypes.data)
        mine.append((h.tobytes(), int(off[0])))
    gathered: list = [None] * world
    dist.all_gather_object(gathered, mine)
    out = [[0] * world for _ in tensors]
    for i, t in enumerate(tensors):
        for r in range(world):
            if r == rank:
                out[i][r] = t.data_ptr()
                continue
            hb, off = gathered[r][i]
            out[i][r] = _open(r, hb) + off
    return out


def exchange_shards(store, rank: int, world: int) -> list[int]:
    import torch.distributed as dist

    mine = shard_handles(store)
    gathered: list = [None] * world
    dist.all_gather_object(gathered, mine)
    return open_peer_shards(store, gathered, rank)


def exchange_rows(ids, dest, world: int, serve, counts=None):
    """Request/serve row exchange over torch.distributed (the NCCL transport of
    the group prefetch; any backend with all_to_all_single works, gloo on CPU
    in the tests).  The reference pulls rows per owner over TCP
    (store.py:173-196 -> wire.py); here every rank sends each owner the ids it
    needs in one all-to-all, owners answer with the rows in request order in a
    second one.

    ids  : 1-D int32 tensor of requested node ids (any order)
    dest : owner rank of each id (same length), or None when the caller
           passes ids already grouped by owner rank with their `counts`
    serve: req_ids -> rows tensor [len(req_ids), stride] for ids this rank owns
    Returns (send_ids, rows): rows[i] is the row of send_ids[i] (ids regrouped
    by owner rank, stable)."""
    import torch
    import torch.distributed as dist

    if counts is None:
        dest = dest.to(torch.int64)
        order = torch.argsort(dest, stable=True)
        send_ids = ids[order].contiguous()
        counts_t = torch.bincount(dest, minlength=world).to(torch.int64)
    else:
        send_ids = ids.contiguous()
        counts_t = torch.tensor(counts, dtype=torch.int64, device=ids.device)
    recv_counts = torch.empty_like(counts_t)
    dist.all_to_all_single(recv_counts, counts_t)
    sc = [int(x) for x in counts_t.tolist()]
    rc = [int(x) for x in recv_counts.tolist()]
    req = torch.empty(sum(rc), dtype=ids.dtype, device=ids.device)
    dist.all_to_all_single(req, send_ids, rc, sc)
    rows = serve(req)
    got = torch.empty((sum(sc),) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    dist.all_to_all_single(got, rows.contiguous(), sc, rc)
    return send_ids, got
