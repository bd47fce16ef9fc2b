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
            p = ctypes.c_void_p()
            buf = np.frombuffer(hb, dtype=np.uint8).copy()
            _lib.call("rg_ipc_open", buf.ctypes.data, ctypes.byref(p))
            opened.append(int(p.value))
            store.set_shard(q, None, base=int(p.value) + off)
    return opened


def exchange_shards(store, rank: int, world: int) -> list[int]:
    import torch.distributed as dist

    mine = shard_handles(store)
    gathered: list = [None] * world
    dist.all_gather_object(gathered, mine)
    return open_peer_shards(store, gathered, rank)
