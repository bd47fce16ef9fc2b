"""GraphSAGE mean aggregation over a sampled block (model.py:72-81, 126-135).

The consumer of the feature bundle.  Forward: mean[t] = in-order fp32 sum of
h[pos(src)] over t's sampled edges / max(cnt_t, 1), plus the self rows
h[pos(dst_front[t])].  Backward: dh = 0; dh[self_pos] += dself; then for every
edge in (dst, src) order dh[pos(src)] += (dmean / denom)[t].  Both orders are
the reference's, so results are bit-identical for identical inputs; the
dense GEMMs around them stay in torch/cuBLAS (north_star item 5).

Edges are given in the sampler's ELL form (ell[t*F + r], r < cnt[t],
ascending src), i.e. BlockSampler.ell[d] / .cnt[d] directly.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import ptr

I32 = torch.int32


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


def sage_mean(h: torch.Tensor, src_front: torch.Tensor, dst_front: torch.Tensor,
              ell: torch.Tensor, cnt: torch.Tensor, fanout: int, H: int | None = None):
    """(mean [n_dst, H], h_self [n_dst, H], self_pos [n_dst]) on the current stream."""
    n_src, ldh = h.shape
    H = ldh if H is None else H
    n_dst = int(dst_front.numel())
    dev = h.device
    mean = torch.empty((max(n_dst, 1), H), dtype=torch.float32, device=dev)
    hself = torch.empty((max(n_dst, 1), H), dtype=torch.float32, device=dev)
    self_pos = torch.empty(max(n_dst, 1), dtype=I32, device=dev)
    _lib.call("rg_sage_mean_fwd", ptr(h), n_src, H, ldh, ptr(src_front), ptr(dst_front), n_dst,
              ptr(ell), ptr(cnt), fanout, ptr(mean), ptr(hself), ptr(self_pos),
              _lib.stream_handle())
    return mean[:n_dst], hself[:n_dst], self_pos[:n_dst]


def sage_mean_backward(dself: torch.Tensor, dmean: torch.Tensor, cnt: torch.Tensor,
                       self_pos: torch.Tensor, src_front: torch.Tensor, ell: torch.Tensor,
                       fanout: int) -> torch.Tensor:
    """dh [n_src, H] (model.py:126-135 order)."""
    n_dst, H = dmean.shape
    n_src = int(src_front.numel())
    dev = dmean.device
    lib = _lib.device()
    scratch = torch.empty(int(lib.rg_sage_transpose_scratch(n_src, n_dst, fanout)), dtype=I32,
                          device=dev)
    toff = torch.empty(n_src + 1, dtype=I32, device=dev)
    tdst = torch.empty(max(1, n_dst * fanout), dtype=I32, device=dev)
    s = _lib.stream_handle()
    _lib.call("rg_sage_transpose", ptr(src_front), n_src, ptr(ell), ptr(cnt), n_dst, fanout,
              ptr(toff), ptr(tdst), ptr(scratch), s)
    self_of = torch.empty(n_src, dtype=I32, device=dev)
    dh = torch.empty((n_src, H), dtype=torch.float32, device=dev)
    _lib.call("rg_sage_mean_bwd", ptr(dself.contiguous()), ptr(dmean.contiguous()), n_dst, H,
              ptr(cnt), ptr(self_pos), ptr(toff), ptr(tdst), n_src, ptr(self_of), ptr(dh), s)
    return dh
