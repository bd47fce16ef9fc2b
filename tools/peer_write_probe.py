"""Probe: scattered 400-B row WRITES into a peer GPU's buffer vs scattered
row READS from it (one process, 2 GPUs, peer access)."""
import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <torch/extension.h>
__global__ void scat(const float4* __restrict__ src, const int* __restrict__ pos, float4* dst,
                     int n, int nvec, int mode) {
  // warp per row, lanes < nvec copy one float4 each; mode 0: src[i] -> dst[pos[i]] (scatter
  // write), mode 1: src[pos[i]] -> dst[i] (gather read)
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = w; i < n; i += nw) {
    int p = pos[i];
    if (lane < nvec) {
      if (mode == 0) dst[(long)p * nvec + lane] = src[(long)i * nvec + lane];
      else dst[(long)i * nvec + lane] = src[(long)p * nvec + lane];
    }
  }
}
void run(torch::Tensor s, torch::Tensor p, torch::Tensor d, int64_t nvec, int64_t mode) {
  int n = p.numel();
  scat<<<148 * 16, 256>>>((const float4*)s.data_ptr(), p.data_ptr<int>(), (float4*)d.data_ptr(),
                          n, nvec, mode);
}
"""
m = load_inline("peer_probe", cpp_sources="void run(torch::Tensor s, torch::Tensor p, torch::Tensor d, int64_t nvec, int64_t mode);",
                cuda_sources=src, functions=["run"],
                extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"])
torch.cuda.set_device(0)
n, N, d = 4_000_000, 800_000, 100
rows0 = torch.randn((N, d), device="cuda:0")
peer = torch.empty((n, d), device="cuda:1")
peer_src = torch.randn((n, d), device="cuda:1")
local = torch.empty((n, d), device="cuda:0")
out0 = torch.empty((N, d), device="cuda:0")
pos = torch.randperm(n, device="cuda:0")[:N].int()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, s, dd, mode in (("scatter-write local", rows0, local, 0), ("scatter-write peer", rows0, peer, 0),
                          ("gather-read peer", peer_src, out0, 1)):
    for _ in range(2):
        m.run(s, pos, dd, d // 4, mode)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        m.run(s, pos, dd, d // 4, mode)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name:22s}: {N * d * 4 / ms / 1e6:7.1f} GB/s payload")
