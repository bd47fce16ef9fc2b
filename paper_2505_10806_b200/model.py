"""GraphSAGE-mean model on the device (model.py:21-172 of the reference).

The bundle consumer: per layer, the sampled-neighbour mean comes from the
bit-exact aggregation kernels (aggregate.py), the two dense products are
fp32 cuBLAS GEMMs (TF32 disabled), and the backward pass is the reference's
analytic one (model.py:107-136), SGD as model.py:139-146.  Parameters are
initialised exactly like init_params (numpy Philox, model.py:38-50).
Dense GEMM rounding differs from numpy's BLAS, so losses agree with the
reference to ~1e-6 relative, not bit-for-bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .aggregate import sage_mean, sage_mean_backward, sage_positions


@dataclass
class LayerParams:
    w_self: torch.Tensor  # d_in x d_out
    w_neigh: torch.Tensor
    bias: torch.Tensor

    def numpy(self):
        return (self.w_self.cpu().numpy(), self.w_neigh.cpu().numpy(), self.bias.cpu().numpy())


def layer_dims(feat_dim: int, hidden_dim: int, num_classes: int, num_layers: int):
    dims = [feat_dim] + [hidden_dim] * (num_layers - 1) + [num_classes]
    return list(zip(dims[:-1], dims[1:]))


def init_params(feat_dim: int, hidden_dim: int, num_classes: int, num_layers: int, seed: int,
                dtype=torch.float32, device="cuda") -> list[LayerParams]:
    """Glorot-scaled normal init from Philox(seed), as model.py:38-50."""
    rng = np.random.Generator(np.random.Philox(seed))
    np_dtype = np.float32 if dtype == torch.float32 else np.float64
    out = []
    for d_in, d_out in layer_dims(feat_dim, hidden_dim, num_classes, num_layers):
        scale = np.sqrt(2.0 / (d_in + d_out))
        ws = (rng.standard_normal((d_in, d_out)) * scale).astype(np_dtype)
        wn = (rng.standard_normal((d_in, d_out)) * scale).astype(np_dtype)
        out.append(LayerParams(torch.from_numpy(ws).to(device), torch.from_numpy(wn).to(device),
                               torch.zeros(d_out, dtype=dtype, device=device)))
    return out


@dataclass
class DeviceBlock:
    """One sampled block on the device: frontiers[d] (int32 ids, sorted),
    ELL edges per level (ell[d]: n_d x F_d, cnt[d]: n_d), fanouts per step,
    and the graph's node count (size of the position-rank scratch)."""

    frontiers: list[torch.Tensor]
    ell: list[torch.Tensor]
    cnt: list[torch.Tensor]
    step_fan: list[int]
    num_nodes: int

    @property
    def num_layers(self) -> int:
        return len(self.ell)


def block_from_slot(smp, slot: int, nfront: np.ndarray) -> DeviceBlock:
    """View slot `slot` of a BlockSampler run (nfront: host copy of its sizes)."""
    fr = [smp.front[d][slot, : int(nfront[d])] for d in range(smp.L + 1)]
    ell = [smp.ell[d][slot] for d in range(smp.L)]
    cnt = [smp.cnt[d][slot, : int(nfront[d])] for d in range(smp.L)]
    return DeviceBlock(fr, ell, cnt, list(smp.step_fan), smp.dg.n)


def _forward(block: DeviceBlock, h: torch.Tensor, params: list[LayerParams]):
    """h: the bundle rows [|input|, >= feat_dim] (a row-strided view is fine)."""
    L = len(params)
    saved = []
    rank = torch.empty(block.num_nodes, dtype=torch.int32, device=h.device)
    for l, p in enumerate(params):
        d = L - 1 - l
        src_front, dst_front = block.frontiers[d + 1], block.frontiers[d]
        pos = sage_positions(src_front, dst_front, block.ell[d], block.cnt[d], block.step_fan[d],
                             block.num_nodes, rank)
        mean, h_self = sage_mean(h, pos, block.cnt[d], H=p.w_self.shape[0])
        z = h_self @ p.w_self + mean @ p.w_neigh + p.bias
        saved.append((h, h_self, mean, z, pos))
        h = torch.clamp_min(z, 0) if l < L - 1 else z
    return h, saved


def loss_and_grad(block: DeviceBlock, rows: torch.Tensor, labels: torch.Tensor,
                  params: list[LayerParams]):
    """Mean softmax cross-entropy over the block's seeds and its exact
    reverse-mode gradient (model.py:107-136)."""
    logits, saved = _forward(block, rows, params)
    y = labels[block.frontiers[0].long()]
    shifted = logits - logits.max(dim=1, keepdim=True).values
    ex = torch.exp(shifted)
    se = ex.sum(dim=1)
    n = y.numel()
    ar = torch.arange(n, device=logits.device)
    nll = -(shifted[ar, y] - torch.log(se))
    dz = ex / se[:, None]
    dz[ar, y] -= 1
    dz = dz / n
    loss = nll.mean()
    L = len(params)
    grads: list[LayerParams | None] = [None] * L
    for l in range(L - 1, -1, -1):
        p = params[l]
        h, h_self, mean, z, pos = saved[l]
        if l < L - 1:
            dz = dz * (z > 0)
        grads[l] = LayerParams(h_self.T @ dz, mean.T @ dz, dz.sum(dim=0))
        if l > 0:
            d = L - 1 - l
            dself = dz @ p.w_self.T
            dmean = dz @ p.w_neigh.T
            dz = sage_mean_backward(dself, dmean, block.cnt[d], pos)
    return loss, grads


def sgd_step(params: list[LayerParams], grads: list[LayerParams], lr: float) -> list[LayerParams]:
    lr_t = torch.tensor(lr, dtype=params[0].w_self.dtype, device=params[0].w_self.device)
    return [LayerParams(p.w_self - lr_t * g.w_self, p.w_neigh - lr_t * g.w_neigh,
                        p.bias - lr_t * g.bias) for p, g in zip(params, grads)]


class FullGraph:
    """Full-neighbourhood mean operator for evaluation (model.py:149-163):
    A[i, j] = 1 / max(deg_i, 1) for each CSR entry, as a CUDA CSR matrix."""

    def __init__(self, g, dtype=torch.float32, device="cuda"):
        deg = np.diff(g.indptr)
        inv = (1.0 / np.maximum(deg, 1)).astype(np.float32 if dtype == torch.float32
                                                   else np.float64)
        vals = torch.from_numpy(np.repeat(inv, deg)).to(device)
        self.adj = torch.sparse_csr_tensor(torch.from_numpy(np.asarray(g.indptr)).to(device),
                                           torch.from_numpy(np.asarray(g.indices, np.int64)).to(
                                               device), vals, size=(g.num_nodes, g.num_nodes),
                                           check_invariants=False)
        self.features = torch.from_numpy(np.ascontiguousarray(g.features)).to(device).to(dtype)
        self.labels = torch.from_numpy(np.asarray(g.labels)).to(device)

    def evaluate(self, params: list[LayerParams], mask: np.ndarray) -> float | None:
        sel = np.flatnonzero(mask)
        if len(sel) == 0:
            return None
        h = self.features
        for l, p in enumerate(params):
            z = h @ p.w_self + (self.adj @ h) @ p.w_neigh + p.bias
            h = torch.clamp_min(z, 0) if l < len(params) - 1 else z
        idx = torch.from_numpy(sel).to(h.device)
        return float((h[idx].argmax(dim=1) == self.labels[idx]).float().mean().item())
