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

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
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


_WGRAD_CHUNK = int(os.environ.get("RG_WGRAD_CHUNK", "256"))


def wgrad(a: torch.Tensor, dz: torch.Tensor) -> torch.Tensor:
    """a.T @ dz for tall operands (the weight gradient over a level's rows,
    model.py:130-131).  cuBLAS runs a [d_in x K] @ [K x d_out] product with a
    tiny output on a couple of CTAs; with K in the thousands the rows are
    split into 256-row chunks multiplied as one batched GEMM (hundreds of
    CTAs) and summed (a different fp32 summation order than one GEMM: parity
    is rel 1e-5).  Products training step, GPU ms per batch: chunk 4096
    0.82, 1024 0.64, 512 0.61, 256 0.59 (tools/train_probe.py)."""
    k = a.shape[0]
    chunk = _WGRAD_CHUNK
    if k < 4 * chunk:
        return a.T @ dz
    n = k // chunk
    head = torch.bmm(a[: n * chunk].view(n, chunk, -1).transpose(1, 2),
                     dz[: n * chunk].view(n, chunk, -1)).sum(dim=0)
    return head + a[n * chunk:].T @ dz[n * chunk:] if n * chunk < k else head


def wgrad_parts(a: torch.Tensor, dz: torch.Tensor) -> torch.Tensor:
    """wgrad's chunk partials, unsummed: [chunks, d_in, d_out] (the sum runs
    inside rg_sgd_apply, in chunk order)."""
    k = a.shape[0]
    chunk = _WGRAD_CHUNK
    if k < 4 * chunk:
        return (a.T @ dz)[None]
    n = k // chunk
    head = torch.bmm(a[: n * chunk].view(n, chunk, -1).transpose(1, 2),
                     dz[: n * chunk].view(n, chunk, -1))
    if n * chunk < k:
        head = torch.cat([head, (a[n * chunk:].T @ dz[n * chunk:])[None]])
    return head


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
        grads[l] = LayerParams(wgrad(h_self, dz), wgrad(mean, dz), dz.sum(dim=0))
        if l > 0:
            d = L - 1 - l
            dself = dz @ p.w_self.T
            dmean = dz @ p.w_neigh.T
            dz = sage_mean_backward(dself, dmean, block.cnt[d], pos)
    return loss, grads


class GraphTrainer:
    """The training step (model.py:107-146: forward, softmax cross-entropy,
    analytic backward, SGD) of one sampler slot's batch b, captured once per
    (slot buffers, b) as a CUDA graph and replayed for every later group that
    lands in that slot.  The step reads the slot's live frontier sizes on the
    device (the aggregation kernels' device counts; rows past them are zero
    padding and the loss / gradients are masked to the live seeds), so a
    replay needs no host sync and ~10 us of host time instead of ~150 eager
    launches.  Parameters are updated in place (the same arithmetic as
    sgd_step); the loss accumulates on the device.  Results equal the eager
    step up to cuBLAS rounding on the padded GEMM shapes."""

    def __init__(self, params: list[LayerParams], labels: torch.Tensor, feat_dim: int,
                 num_nodes: int, lr: float):
        self.params = [LayerParams(p.w_self.clone(), p.w_neigh.clone(), p.bias.clone())
                       for p in params]
        self.dtype = self.params[0].w_self.dtype
        self.dcode = {torch.float32: 0, torch.float64: 1}[self.dtype]
        self.labels = labels.long().contiguous()
        self.lr = float(lr)
        self.feat_dim = int(feat_dim)
        self.n = int(num_nodes)
        self.loss_sum = torch.zeros((), dtype=torch.float64, device=labels.device)
        self.rank = torch.empty(self.n, dtype=torch.int32, device=labels.device)
        self.pool = torch.cuda.graph_pool_handle()
        self.graphs: dict = {}
        self.captures = 0

    def _body(self, smp, rows_buf, b: int) -> None:
        L, G = smp.L, smp.G
        nf = smp.nfront
        dn = [nf.data_ptr() + 4 * (d * G + b) for d in range(L + 1)]
        front = [smp.front[d][b] for d in range(L + 1)]
        rows = rows_buf[b, :, : self.feat_dim]
        h = rows if self.dtype == torch.float32 else rows.to(self.dtype)
        params = self.params
        saved = []
        for l, p in enumerate(params):
            d = L - 1 - l
            cnt = smp.cnt[d][b]
            pos = sage_positions(front[d + 1], front[d], smp.ell[d][b], cnt,
                                 smp.step_fan[d], self.n, self.rank, dn[d + 1], dn[d])
            mean, h_self = sage_mean(h, pos, cnt, H=p.w_self.shape[0])
            # bias + h_self @ Ws + mean @ Wn as two accumulating GEMMs (no
            # separate add launches)
            z = torch.addmm(p.bias, h_self, p.w_self)
            z.addmm_(mean, p.w_neigh)
            saved.append((h_self, mean, z, pos, d, cnt))
            h = torch.clamp_min(z, 0) if l < L - 1 else z
        # softmax cross-entropy over the live seeds and its gradient, one
        # kernel (model.py:107-124); the loss accumulates into loss_sum
        cap0 = front[0].numel()
        h = h.contiguous()
        dz = torch.empty_like(h)
        nll = torch.empty(cap0, dtype=h.dtype, device=h.device)
        s = _lib.stream_handle()
        _lib.call("rg_softmax_xent", self.dcode, h.data_ptr(), h.shape[1], cap0, dn[0],
                  self.labels.data_ptr(), front[0].data_ptr(), dz.data_ptr(), nll.data_ptr(),
                  self.loss_sum.data_ptr(), s)
        for l in range(L - 1, -1, -1):
            p = params[l]
            h_self, mean, z, pos, d, cnt = saved[l]
            if l < L - 1:
                dz = torch.ops.aten.threshold_backward(dz, z, 0)  # dz * (z > 0)
            gws, gwn, gb = wgrad_parts(h_self, dz), wgrad_parts(mean, dz), dz.sum(dim=0)
            if l > 0:
                dself = dz @ p.w_self.T
                dmean = dz @ p.w_neigh.T
                dz = sage_mean_backward(dself, dmean, cnt, pos)
            # SGD on the three tensors in one launch, the weight gradients'
            # chunk partials summed inside (sgd_step, model.py:139-146)
            ws = (p.w_self, p.w_neigh, p.bias)
            gs = (gws, gwn, gb)
            _lib.call("rg_sgd_apply", self.dcode, 3,
                      (ctypes.c_void_p * 3)(*[w.data_ptr() for w in ws]),
                      (ctypes.c_void_p * 3)(*[g.data_ptr() for g in gs]),
                      (ctypes.c_int64 * 3)(*[w.numel() for w in ws]),
                      (ctypes.c_int32 * 3)(gws.shape[0], gwn.shape[0], 1), self.lr, s)

    def step(self, smp, rows_buf, b: int, capture_lock=None) -> None:
        """One batch on the current stream (capturing its graph on first use;
        capture_lock, e.g. GroupProducer.capture_lock, keeps another thread's
        CUDA calls out of the capture)."""
        key = (smp.front[0].data_ptr(), rows_buf.data_ptr(), int(b))
        g = self.graphs.get(key)
        if g is None:
            if capture_lock is not None:
                with capture_lock:
                    self._capture(smp, rows_buf, b, key)
            else:
                self._capture(smp, rows_buf, b, key)
            g = self.graphs[key]
        g.replay()

    def _capture(self, smp, rows_buf, b: int, key) -> None:
        cur = torch.cuda.current_stream()
        if not self.graphs:
            # first capture: let cuBLAS / the allocator initialise outside it,
            # on a side stream, on throw-away copies of the parameters
            keep = [LayerParams(p.w_self.clone(), p.w_neigh.clone(), p.bias.clone())
                    for p in self.params]
            loss0 = self.loss_sum.clone()
            side = torch.cuda.Stream()
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                self._body(smp, rows_buf, b)
            cur.wait_stream(side)
            for p, k in zip(self.params, keep):
                p.w_self.copy_(k.w_self)
                p.w_neigh.copy_(k.w_neigh)
                p.bias.copy_(k.bias)
            self.loss_sum.copy_(loss0)
        g = torch.cuda.CUDAGraph()
        # thread_local + the caller's capture_lock: the GroupProducer thread
        # keeps its GPU work in flight but makes no CUDA calls meanwhile
        with torch.cuda.graph(g, pool=self.pool, capture_error_mode="thread_local"):
            self._body(smp, rows_buf, b)
        self.graphs[key] = g
        self.captures += 1


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
