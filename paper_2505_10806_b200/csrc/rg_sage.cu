// K8: GraphSAGE mean aggregation over a sampled block, forward and backward.
//
// Reference: gnnpipe/model.py:72-81 (_forward_pass) and model.py:126-135
// (loss_and_grad backward scatter).  The reference sums neighbour rows with
// np.add.at in edge order (dst asc, src asc), divides by max(count, 1) in
// fp32, and in the backward adds dself at the self positions first and then
// (dmean / denom)[dst] into dh[src] in the same edge order.  Both kernels
// reproduce those orders exactly (one sequential fp32 chain per output
// element, parallel over columns), so results are bit-identical to the
// reference for identical inputs; only the dense GEMMs around them (cuBLAS)
// differ in rounding.
#include <climits>

#include "rg_common.cuh"

namespace rg {
namespace {

constexpr int kWarps = 8;
constexpr int kSortCap = 4096;

__device__ __forceinline__ int lower_bound(const int32_t* __restrict__ a, int64_t n, int32_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (int)lo;
}

// warp per destination row t; columns strided over lanes, 4 per lane per tile
__global__ void __launch_bounds__(kWarps * 32)
    sage_fwd_kernel(const float* __restrict__ h, int64_t n_src, int H, int ldh,
                    const int32_t* __restrict__ src_front, const int32_t* __restrict__ dst_front,
                    int64_t n_dst, const int32_t* __restrict__ ell, const int32_t* __restrict__ cnt,
                    int F, float* __restrict__ mean, float* __restrict__ self,
                    int32_t* __restrict__ self_pos) {
  const int lane = lane_id();
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); t < n_dst; t += nw) {
    const int c = cnt[t];
    const float denom = (float)max(c, 1);
    const int ps = lower_bound(src_front, n_src, dst_front[t]);
    if (lane == 0 && self_pos) self_pos[t] = ps;
    int p_lane = 0;
    if (lane < c) p_lane = lower_bound(src_front, n_src, ell[t * F + lane]);
    for (int col0 = 0; col0 < H; col0 += 128) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int r0 = 0; r0 < c; r0 += 32) {
        int p_chunk = p_lane;
        if (r0 > 0) {
          const int r = r0 + lane;
          p_chunk = r < c ? lower_bound(src_front, n_src, ell[t * F + r]) : 0;
        }
        const int nr = min(32, c - r0);
        for (int rr = 0; rr < nr; ++rr) {
          const int p = __shfl_sync(kFull, p_chunk, rr);
          const float* hp = h + (int64_t)p * ldh;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int col = col0 + u * 32 + lane;
            if (col < H) acc[u] += __ldg(hp + col);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int col = col0 + u * 32 + lane;
        if (col < H) {
          mean[t * H + col] = acc[u] / denom;
          if (self) self[t * H + col] = __ldg(h + (int64_t)ps * ldh + col);
        }
      }
    }
  }
}

// edge -> src position (ELL aligned) and per-src in-degree
__global__ void transpose_count_kernel(const int32_t* __restrict__ src_front, int64_t n_src,
                                       const int32_t* __restrict__ ell,
                                       const int32_t* __restrict__ cnt, int64_t n_dst, int F,
                                       int32_t* __restrict__ epos, int32_t* __restrict__ deg) {
  const int64_t total = n_dst * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / F;
    const int r = (int)(i - t * F);
    if (r < cnt[t]) {
      const int p = lower_bound(src_front, n_src, ell[i]);
      epos[i] = p;
      atomicAdd(deg + p, 1);
    }
  }
}

// exclusive scan of deg[0..n) into off[0..n], single pass per 1024-chunk
// with the chunk base taken from a preceding count pass (two kernels).
constexpr int kScanChunk = 1024;
__global__ void __launch_bounds__(256)
    chunk_sum_kernel(const int32_t* __restrict__ x, int64_t n, int32_t* __restrict__ tot) {
  __shared__ int s_red[32];
  const int64_t i0 = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * 4;
  int c = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i0 + i < n) c += x[i0 + i];
  int total;
  block_excl_scan<256>(c, s_red, &total);
  if (threadIdx.x == 0) tot[blockIdx.x] = total;
}

__global__ void __launch_bounds__(256)
    chunk_scan_kernel(const int32_t* __restrict__ x, int64_t n, const int32_t* __restrict__ tot,
                      int64_t nchunks, int32_t* __restrict__ off) {
  __shared__ int s_red[32];
  __shared__ int s_base;
  int before = 0, all = 0;
  for (int64_t c = threadIdx.x; c < nchunks; c += blockDim.x) {
    all += tot[c];
    if (c < (int64_t)blockIdx.x) before += tot[c];
  }
  int t;
  block_excl_scan<256>(before, s_red, &t);
  if (threadIdx.x == 0) s_base = t;
  __syncthreads();
  const int base = s_base;
  __syncthreads();
  int grand;
  block_excl_scan<256>(all, s_red, &grand);
  if (blockIdx.x == 0 && threadIdx.x == 0) off[n] = grand;
  const int64_t i0 = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * 4;
  int v[4], s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = i0 + i < n ? x[i0 + i] : 0;
    s += v[i];
  }
  int dummy;
  int at = base + block_excl_scan<256>(s, s_red, &dummy);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i0 + i < n) off[i0 + i] = at;
    at += v[i];
  }
}

__global__ void transpose_fill_kernel(const int32_t* __restrict__ cnt, int64_t n_dst, int F,
                                      const int32_t* __restrict__ epos,
                                      const int32_t* __restrict__ toff, int32_t* __restrict__ fill,
                                      int32_t* __restrict__ tdst) {
  const int64_t total = n_dst * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / F;
    const int r = (int)(i - t * F);
    if (r < cnt[t]) {
      const int p = epos[i];
      tdst[toff[p] + atomicAdd(fill + p, 1)] = (int32_t)t;
    }
  }
}

// sort every src segment of tdst ascending (restores the reference's edge
// order for each src); warp per segment up to 32, CTA + smem beyond.
__global__ void __launch_bounds__(256)
    segment_sort_kernel(const int32_t* __restrict__ toff, int64_t n_src,
                        int32_t* __restrict__ tdst, int32_t* __restrict__ err) {
  __shared__ int32_t s_val[kSortCap];
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t s = (int64_t)blockIdx.x * 8 + warp; s < n_src; s += nw) {
    const int a = toff[s], len = toff[s + 1] - a;
    if (len <= 1 || len > 32) continue;
    int32_t x = lane < len ? tdst[a + lane] : INT_MAX;
    warp_bitonic_sort_keys(x);
    if (lane < len) tdst[a + lane] = x;
  }
  // long segments: whole CTA, one at a time
  for (int64_t s = blockIdx.x; s < n_src; s += gridDim.x) {
    const int a = toff[s], len = toff[s + 1] - a;
    if (len <= 32) continue;
    if (len > kSortCap) {
      if (threadIdx.x == 0) atomicExch(err, 1);
      continue;
    }
    int P = 1;
    while (P < len) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) s_val[i] = i < len ? tdst[a + i] : INT_MAX;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          const int l = i ^ j;
          if (l > i) {
            const bool up = (i & k) == 0;
            const int32_t x = s_val[i], y = s_val[l];
            if ((x > y) == up) {
              s_val[i] = y;
              s_val[l] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < len; i += blockDim.x) tdst[a + i] = s_val[i];
    __syncthreads();
  }
}

__global__ void self_of_kernel(const int32_t* __restrict__ self_pos, int64_t n_dst,
                               int32_t* __restrict__ self_of) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_dst;
       t += (int64_t)gridDim.x * blockDim.x)
    self_of[self_pos[t]] = (int32_t)t;
}

__global__ void __launch_bounds__(kWarps * 32)
    sage_bwd_kernel(const float* __restrict__ dself, const float* __restrict__ dmean, int H,
                    const int32_t* __restrict__ cnt, const int32_t* __restrict__ self_of,
                    const int32_t* __restrict__ toff, const int32_t* __restrict__ tdst,
                    int64_t n_src, float* __restrict__ dh) {
  const int lane = lane_id();
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t s = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); s < n_src; s += nw) {
    const int a = toff[s], len = toff[s + 1] - a;
    const int so = self_of[s];
    for (int col0 = 0; col0 < H; col0 += 128) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      if (so >= 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = col0 + u * 32 + lane;
          if (col < H) acc[u] += dself[(int64_t)so * H + col];
        }
      }
      for (int k = 0; k < len; ++k) {
        const int t = __ldg(tdst + a + k);
        const float denom = (float)max(__ldg(cnt + t), 1);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = col0 + u * 32 + lane;
          if (col < H) acc[u] += __ldg(dmean + (int64_t)t * H + col) / denom;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int col = col0 + u * 32 + lane;
        if (col < H) dh[s * H + col] = acc[u];
      }
    }
  }
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_sage_mean_fwd(const float* d_h, int64_t n_src, int32_t H, int32_t ldh,
                                const int32_t* d_src_front, const int32_t* d_dst_front,
                                int64_t n_dst, const int32_t* d_ell, const int32_t* d_cnt,
                                int32_t fanout, float* d_mean, float* d_self, int32_t* d_self_pos,
                                void* stream) {
  RG_REQUIRE(H >= 1 && ldh >= H && n_src >= 1 && n_dst >= 0 && fanout >= 1,
             "rg_sage_mean_fwd: bad sizes");
  if (n_dst == 0) return RG_OK;
  const int grid = (int)std::min<int64_t>((n_dst + kWarps - 1) / kWarps, kNumSMs * 16);
  sage_fwd_kernel<<<grid, kWarps * 32, 0, (cudaStream_t)stream>>>(
      d_h, n_src, H, ldh, d_src_front, d_dst_front, n_dst, d_ell, d_cnt, fanout, d_mean, d_self,
      d_self_pos);
  return check_launch("sage_fwd");
}

extern "C" int rg_sage_transpose(const int32_t* d_src_front, int64_t n_src, const int32_t* d_ell,
                                 const int32_t* d_cnt, int64_t n_dst, int32_t fanout,
                                 int32_t* d_toff, int32_t* d_tdst, int32_t* d_scratch,
                                 void* stream) {
  RG_REQUIRE(n_src >= 1 && n_dst >= 0 && fanout >= 1, "rg_sage_transpose: bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  // scratch layout: deg[n_src] | fill[n_src] | err[1] | chunk[nchunks] | epos[n_dst*F]
  const int64_t nchunks = (n_src + kScanChunk - 1) / kScanChunk;
  int32_t* deg = d_scratch;
  int32_t* fill = deg + n_src;
  int32_t* err = fill + n_src;
  int32_t* chunk = err + 1;
  int32_t* epos = chunk + nchunks;
  if (cudaMemsetAsync(deg, 0, sizeof(int32_t) * (2 * n_src + 1), s) != cudaSuccess)
    return check_launch("transpose memset");
  const int g = kNumSMs * 8;
  transpose_count_kernel<<<g, 256, 0, s>>>(d_src_front, n_src, d_ell, d_cnt, n_dst, fanout, epos,
                                           deg);
  int rc = check_launch("transpose_count");
  if (rc) return rc;
  chunk_sum_kernel<<<(unsigned)nchunks, 256, 0, s>>>(deg, n_src, chunk);
  if ((rc = check_launch("chunk_sum"))) return rc;
  chunk_scan_kernel<<<(unsigned)nchunks, 256, 0, s>>>(deg, n_src, chunk, nchunks, d_toff);
  if ((rc = check_launch("chunk_scan"))) return rc;
  transpose_fill_kernel<<<g, 256, 0, s>>>(d_cnt, n_dst, fanout, epos, d_toff, fill, d_tdst);
  if ((rc = check_launch("transpose_fill"))) return rc;
  segment_sort_kernel<<<kNumSMs * 2, 256, 0, s>>>(d_toff, n_src, d_tdst, err);
  return check_launch("segment_sort");
}

extern "C" int64_t rg_sage_transpose_scratch(int64_t n_src, int64_t n_dst, int32_t fanout) {
  return 2 * n_src + 1 + (n_src + kScanChunk - 1) / kScanChunk + n_dst * fanout;
}

extern "C" int rg_sage_mean_bwd(const float* d_dself, const float* d_dmean, int64_t n_dst,
                                int32_t H, const int32_t* d_cnt, const int32_t* d_self_pos,
                                const int32_t* d_toff, const int32_t* d_tdst, int64_t n_src,
                                int32_t* d_self_of, float* d_dh, void* stream) {
  RG_REQUIRE(H >= 1 && n_src >= 1 && n_dst >= 0, "rg_sage_mean_bwd: bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(d_self_of, 0xff, sizeof(int32_t) * n_src, s) != cudaSuccess)
    return check_launch("bwd memset");
  if (n_dst > 0) {
    self_of_kernel<<<kNumSMs * 2, 256, 0, s>>>(d_self_pos, n_dst, d_self_of);
    int rc = check_launch("self_of");
    if (rc) return rc;
  }
  const int grid = (int)std::min<int64_t>((n_src + kWarps - 1) / kWarps, kNumSMs * 16);
  sage_bwd_kernel<<<grid, kWarps * 32, 0, s>>>(d_dself, d_dmean, H, d_cnt, d_self_of, d_toff,
                                               d_tdst, n_src, d_dh);
  return check_launch("sage_bwd");
}
