"""GraphSAGE mean aggregation over a sampled block (model.py:72-81, 126-135).

The consumer of the feature bundle.  Forward: mean[t] = in-order sum of
h[pos(src)] over t's sampled edges / max(cnt_t, 1), plus the self rows
h[pos(dst_front[t])].  Backward: dh = 0; dh[self_pos] += dself; then for every
edge in (dst, src) order dh[pos(src)] += (dmean / denom)[t].  Both orders are
the reference's, so results are bit-identical for identical inputs, in fp32
and in fp64 (RunConfig.precision, train.py:117); the dense GEMMs around them
stay in torch/cuBLAS (north_star item 5).

Edges are given in the sampler's ELL form (ell[t*F + r], r < cnt[t],
ascending src), i.e. BlockSampler.ell[d] / .cnt[d] directly.  The positions
(model.py:53-55, the searchsorted calls) are resolved once per level by
``sage_positions`` and shared by the forward and the backward.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ptr

I32 = torch.int32
_DTYPES = {torch.float32: 0, torch.float64: 1}  # RG_DTYPE_F32 / RG_DTYPE_F64


def edges_to_ell(dst_front: np.ndarray, src: np.ndarray, dst: np.ndarray):
    """Host helper: flat (dst, src)-sorted edges -> (ell [n_dst*F], cnt [n_dst], F)."""
    dst_front = np.asarray(dst_front)
    pos = np.searchsorted(dst_front, dst)
    cnt = np.bincount(pos, minlength=len(dst_front)).astype(np.int32)
    F = max(1, int(cnt.max()) if len(cnt) else 1)
    ell = np.zeros(len(dst_front) * F, dtype=np.int32)
    start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    r = np.arange(len(src)) - start[pos]
    ell[pos * F + r] = src
    return ell, cnt, F


@dataclass
class LevelPositions:
    """One level's resolved positions: epos [n_dst*F] (src position of every
    ELL edge, -1 past a row's count), self_pos [n_dst].  With device counts
    (d_n_src / d_n_dst: addresses of int32 words, e.g. a sampler slot's
    nfront entries) n_src / n_dst are capacities and rows past the live
    counts are zero padding — nothing here then syncs with the host, so a
    whole training step can be captured in a CUDA graph."""

    epos: torch.Tensor
    self_pos: torch.Tensor
    n_src: int
    fanout: int
    d_n_src: int | None = None
    d_n_dst: int | None = None


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype not in _DTYPES:
        raise TypeError(f"aggregation supports float32 / float64, got {t.dtype}")
    return _DTYPES[t.dtype]


def sage_positions(src_front: torch.Tensor, dst_front: torch.Tensor, ell: torch.Tensor,
                   cnt: torch.Tensor, fanout: int, n_nodes: int,
                   rank: torch.Tensor | None = None, d_n_src: int | None = None,
                   d_n_dst: int | None = None) -> LevelPositions:
    """Ranks of every sampled edge's src and of every dst in src_front
    (rank: optional int32 [n_nodes] scratch, reusable across levels).
    d_n_src / d_n_dst: optional device counts (the tensors are then
    capacity-sized)."""
    n_src, n_dst = int(src_front.numel()), int(dst_front.numel())
    dev = src_front.device
    if rank is None:
        rank = torch.empty(n_nodes, dtype=I32, device=dev)
    epos = torch.empty(max(1, n_dst * fanout), dtype=I32, device=dev)
    self_pos = torch.empty(max(n_dst, 1), dtype=I32, device=dev)
    _lib.call("rg_sage_positions", ptr(src_front), n_src, ptr(dst_front), n_dst, ptr(ell),
              ptr(cnt), fanout, n_nodes, d_n_src, d_n_dst, ptr(rank), ptr(epos), ptr(self_pos),
              _lib.stream_handle())
    return LevelPositions(epos, self_pos[:n_dst], n_src, fanout, d_n_src, d_n_dst)


def sage_mean(h: torch.Tensor, pos: LevelPositions, cnt: torch.Tensor, H: int | None = None):
    """(mean [n_dst, H], h_self [n_dst, H]) on the current stream.  h may be a
    row-strided view (e.g. the bundle rows of a slot with their padded pitch):
    the kernel reads row p at p * h.stride(0)."""
    if h.dim() != 2 or h.stride(1) != 1:
        raise ValueError("h must be a 2-D tensor with unit column stride")
    code = _dtype_code(h)
    H = h.shape[1] if H is None else H
    if H > h.shape[1]:
        raise ValueError(f"H={H} exceeds the row width {h.shape[1]}")
    n_dst = int(pos.self_pos.numel())
    dev = h.device
    mean = torch.empty((max(n_dst, 1), H), dtype=h.dtype, device=dev)
    hself = torch.empty((max(n_dst, 1), H), dtype=h.dtype, device=dev)
    _lib.call("rg_sage_mean_fwd", code, ptr(h), H, h.stride(0), ptr(pos.epos), ptr(pos.self_pos),
              n_dst, pos.d_n_dst, ptr(cnt), pos.fanout, ptr(mean), ptr(hself),
              _lib.stream_handle())
    return mean[:n_dst], hself[:n_dst]


def sage_mean_backward(dself: torch.Tensor, dmean: torch.Tensor, cnt: torch.Tensor,
                       pos: LevelPositions) -> torch.Tensor:
    """dh [n_src, H] (model.py:126-135 order)."""
    dself, dmean = dself.contiguous(), dmean.contiguous()
    if dself.dtype != dmean.dtype:
        raise TypeError("dself and dmean must share a dtype")
    code = _dtype_code(dmean)
    n_dst, H = dmean.shape
    n_src, F = pos.n_src, pos.fanout
    dev = dmean.device
    lib = _lib.device()
    nbytes = int(lib.rg_sage_transpose_scratch(n_src, n_dst, F))
    if nbytes < 0:
        raise ValueError("sage_mean_backward: block too large for the transpose")
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    toff = torch.empty(n_src + 1, dtype=I32, device=dev)
    tdst = torch.empty(max(1, n_dst * F), dtype=I32, device=dev)
    s = _lib.stream_handle()
    _lib.call("rg_sage_transpose", ptr(pos.epos), ptr(cnt), n_dst, F, n_src, ptr(toff), ptr(tdst),
              ptr(scratch), nbytes, s)
    self_of = torch.empty(n_src, dtype=I32, device=dev)
    dh = torch.empty((n_src, H), dtype=dmean.dtype, device=dev)
    _lib.call("rg_sage_mean_bwd", code, ptr(dself), ptr(dmean), n_dst, H, ptr(cnt),
              ptr(pos.self_pos), ptr(toff), ptr(tdst), n_src, pos.d_n_src, pos.d_n_dst,
              ptr(self_of), ptr(dh), s)
    return dh
