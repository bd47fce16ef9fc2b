// K9: group prefetch of peer-owned rows over NVLink (north_star item 4).
//
// The reference pulls every mini-batch's fallback rows from their owners
// (prefetch.py:41-88 -> store.py:173-196), one RPC per owner per batch, and
// its Prefetcher runs the producer ahead of the consumer (prefetch.py:91-164).
// A group of G batches touches each input node ~G * |inputs| / n times
// (Products, G = 32: ~8.8x), so pulling per batch moves the same peer rows
// over NVLink many times.  Here, once a group is sampled, the union of its
// input sets (OR of the per-batch level-L bitmaps) restricted to the nodes
// whose route points at a peer GPU's shard is copied ONCE into a local
// shadow of that shard (same row positions), on the sampling stream, ahead
// of the group's gather; the gather then reads those rows from local HBM
// through the unchanged route words.  Per-batch accounting (fallback rows,
// owners, RPCs) is computed from the route words exactly as before.
#include <cstdlib>

#include "rg_common.cuh"

namespace rg {
namespace {

struct RowBases {
  const float* p[16];
};
struct RowDsts {
  float* p[16];
};

// bits[w] bit j = route kind of node 32w+j is in kind_mask
__global__ void __launch_bounds__(256)
    route_kind_bits_kernel(const uint32_t* __restrict__ route, int64_t n, uint32_t kind_mask,
                           uint32_t* __restrict__ bits) {
  const int64_t nwords = (n + 31) / 32;
  const int lane = lane_id();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nwords;
       w += warps) {
    const int64_t v = w * 32 + lane;
    bool in = false;
    if (v < n) {
      const uint32_t rt = route[v];
      in = rt != RG_ROUTE_INVALID && ((kind_mask >> (rt >> RG_KIND_SHIFT)) & 1u);
    }
    const unsigned m = __ballot_sync(kFull, in);
    if (lane == 0) bits[w] = m;
  }
}

// out[w] = mask[w] & OR_{b < G} bm[b * nwords + w]
__global__ void __launch_bounds__(256)
    group_union_kernel(const uint32_t* __restrict__ bm, int64_t nwords, int G,
                       const uint32_t* __restrict__ mask, uint32_t* __restrict__ out) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t m = mask[w];
    uint32_t u = 0;
    if (m) {
      for (int b = 0; b < G; ++b) u |= __ldg(bm + (int64_t)b * nwords + w);
    }
    out[w] = u & m;
  }
}

// rows of ids[0 .. *nids) copied from src[kind] to dst[kind] at the same
// row offset.  One warp per 32 rows; each warp instruction touches one row
// (or a 32-vector slice of it), the mapping NVLink peer reads prefer
// (tools/nvlink_probe.py), 8 loads in flight per lane.
__global__ void __launch_bounds__(256)
    prefetch_rows_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ nids,
                         const uint32_t* __restrict__ route, const __grid_constant__ RowBases src,
                         const __grid_constant__ RowDsts dst, int src_stride, int nvec) {
  constexpr int kU = 8;
  __shared__ const float* s_src[16];
  __shared__ float* s_dst[16];
  if (threadIdx.x < 16) {
    s_src[threadIdx.x] = src.p[threadIdx.x];
    s_dst[threadIdx.x] = dst.p[threadIdx.x];
  }
  __syncthreads();
  const int lane = lane_id();
  const int n = *nids;
  const int chunks = (nvec + 31) >> 5;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5) * 32;
  for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; r0 < n;
       r0 += wstride) {
    const int64_t r = r0 + lane;
    const int nr = (int)(n - r0 < 32 ? n - r0 : 32);
    unsigned long long sp = 0, dp = 0;
    if (r < n) {
      const uint32_t rt = __ldg(route + __ldg(ids + r));
      if (rt != RG_ROUTE_INVALID) {
        const int kind = (int)(rt >> RG_KIND_SHIFT);
        const int64_t off = (int64_t)(rt & RG_ROW_MASK) * src_stride;
        if (s_src[kind] && s_dst[kind]) {
          sp = reinterpret_cast<unsigned long long>(s_src[kind] + off);
          dp = reinterpret_cast<unsigned long long>(s_dst[kind] + off);
        }
      }
    }
    const int items = nr * chunks;
    for (int i0 = 0; i0 < items; i0 += kU) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int it = i0 + u;
        const int rr = chunks == 1 ? it : it / chunks;
        const int c = (it - rr * chunks) * 32 + lane;
        const unsigned long long s = __shfl_sync(kFull, sp, rr & 31);
        v[u] = (it < items && c < nvec && s) ? ld_stream(reinterpret_cast<const float4*>(s) + c)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int it = i0 + u;
        const int rr = chunks == 1 ? it : it / chunks;
        const int c = (it - rr * chunks) * 32 + lane;
        const unsigned long long d = __shfl_sync(kFull, dp, rr & 31);
        if (it < items && c < nvec && d) reinterpret_cast<float4*>(d)[c] = v[u];
      }
    }
  }
}

// rows received from their owners (NCCL transport: rows[i] belongs to
// ids[i]) scattered into the local shadow of their shard, at the row given
// by the route word.  Warp per 32 rows; source rows are contiguous.
__global__ void __launch_bounds__(256)
    scatter_rows_kernel(const int32_t* __restrict__ ids, int64_t n,
                        const uint32_t* __restrict__ route, const float* __restrict__ rows,
                        int rows_stride, const __grid_constant__ RowDsts dst, int dst_stride,
                        int nvec) {
  __shared__ float* s_dst[16];
  if (threadIdx.x < 16) s_dst[threadIdx.x] = dst.p[threadIdx.x];
  __syncthreads();
  const int lane = lane_id();
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5) * 32;
  for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; r0 < n;
       r0 += wstride) {
    const int64_t r = r0 + lane;
    const int nr = (int)(n - r0 < 32 ? n - r0 : 32);
    unsigned long long dp = 0;
    if (r < n) {
      const uint32_t rt = __ldg(route + __ldg(ids + r));
      if (rt != RG_ROUTE_INVALID && s_dst[rt >> RG_KIND_SHIFT])
        dp = reinterpret_cast<unsigned long long>(s_dst[rt >> RG_KIND_SHIFT] +
                                                  (int64_t)(rt & RG_ROW_MASK) * dst_stride);
    }
    const float4* src = reinterpret_cast<const float4*>(rows + r0 * rows_stride);
    const int rs4 = rows_stride / 4;
    const int total = nr * nvec;
    for (int e0 = 0; e0 < total; e0 += 32) {  // warp-uniform trip count
      const int e = e0 + lane;
      const int rr = e / nvec, c = e - rr * nvec;
      const unsigned long long d = __shfl_sync(kFull, dp, rr & 31);
      if (e < total && d) reinterpret_cast<float4*>(d)[c] = ld_stream(src + (int64_t)rr * rs4 + c);
    }
  }
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_route_kind_bits(const uint32_t* d_route, int64_t n, uint32_t kind_mask,
                                  uint32_t* d_bits, void* stream) {
  RG_REQUIRE(n >= 1, "rg_route_kind_bits: bad n");
  route_kind_bits_kernel<<<kNumSMs * 4, 256, 0, (cudaStream_t)stream>>>(d_route, n, kind_mask,
                                                                        d_bits);
  return check_launch("route_kind_bits");
}

extern "C" int rg_group_union(const uint32_t* d_bm, int64_t nwords, int32_t G,
                              const uint32_t* d_mask, uint32_t* d_out, void* stream) {
  RG_REQUIRE(G >= 1 && nwords >= 1, "rg_group_union: bad sizes");
  const int blocks = (int)std::min<int64_t>((nwords + 255) / 256, kNumSMs * 8);
  group_union_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(d_bm, nwords, G, d_mask, d_out);
  return check_launch("group_union");
}

extern "C" int rg_prefetch_rows(const int32_t* d_ids, const int32_t* d_nids, int64_t cap,
                                const uint32_t* d_route, const float* const* h_src,
                                float* const* h_dst, int32_t src_stride, int32_t d,
                                void* stream) {
  RG_REQUIRE(cap >= 1 && d >= 1 && src_stride >= d && src_stride % 4 == 0,
             "rg_prefetch_rows: bad sizes");
  RowBases s;
  RowDsts t;
  for (int i = 0; i < 16; ++i) {
    s.p[i] = h_src[i];
    t.p[i] = h_dst[i];
  }
  const int nvec = (d + 3) / 4;
  // 6 CTAs/SM (1.5 waves at 64 registers), as for the latency-bound peer
  // gather; measured: 2/SM co-running with a split local gather pass was
  // slower end to end
  static const int env_ctas = [] {
    const char* e = getenv("RG_PREFETCH_CTAS_PER_SM");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  const int per_sm = env_ctas ? env_ctas : 6;
  const int64_t want = (cap + 255) / 256;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)kNumSMs * per_sm));
  prefetch_rows_kernel<<<gx, 256, 0, (cudaStream_t)stream>>>(d_ids, d_nids, d_route, s, t,
                                                            src_stride, nvec);
  return check_launch("prefetch_rows");
}

extern "C" int rg_scatter_rows(const int32_t* d_ids, int64_t n, const uint32_t* d_route,
                               const float* d_rows, int32_t rows_stride, float* const* h_dst,
                               int32_t dst_stride, int32_t d, void* stream) {
  RG_REQUIRE(n >= 0 && d >= 1 && rows_stride >= d && dst_stride >= d && rows_stride % 4 == 0 &&
                 dst_stride % 4 == 0,
             "rg_scatter_rows: bad sizes");
  if (n == 0) return RG_OK;
  RowDsts t;
  for (int i = 0; i < 16; ++i) t.p[i] = h_dst[i];
  const int64_t want = (n + 255) / 256;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)kNumSMs * 4));
  scatter_rows_kernel<<<gx, 256, 0, (cudaStream_t)stream>>>(d_ids, n, d_route, d_rows,
                                                            rows_stride, t, dst_stride,
                                                            (d + 3) / 4);
  return check_launch("scatter_rows");
}

// ---- cross-GPU group sequence flags (shared sampling) ------
// Every worker samples every batch (train.py:291-311), so at N > 1 the
// ranks split each group's batches, sample their share and copy the others'
// sampled input sets from the peers over NVLink.  A rank publishes "group
// seq of slot s is sampled / copied" as a 64-bit counter in its own memory;
// peers poll it through the IPC mapping.  Writes of the kernels before the
// signal (stream order) are made visible system-wide before the counter;
// the wait is bounded (a stuck peer sets *d_status instead of hanging the
// GPU).
namespace rg {
namespace {
__global__ void flag_signal_kernel(unsigned long long* flag, unsigned long long value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

__global__ void flag_wait_kernel(const unsigned long long* flag, unsigned long long value,
                                 long long timeout_cycles, int32_t* status) {
  const long long t0 = clock64();
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= value) break;
    if (clock64() - t0 > timeout_cycles) {
      atomicExch(status, 1);
      break;
    }
    __nanosleep(256);
  }
  __threadfence_system();
}
}  // namespace
}  // namespace rg

extern "C" int rg_flag_signal(uint64_t* d_flag, uint64_t value, void* stream) {
  RG_REQUIRE(d_flag != nullptr && ((uintptr_t)d_flag & 7) == 0, "rg_flag_signal: bad flag");
  flag_signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long*)d_flag, value);
  return check_launch("flag_signal");
}

extern "C" int rg_flag_wait(const uint64_t* d_flag, uint64_t value, int32_t timeout_ms,
                            int32_t* d_status, void* stream) {
  RG_REQUIRE(d_flag != nullptr && ((uintptr_t)d_flag & 7) == 0 && d_status != nullptr &&
                 timeout_ms > 0,
             "rg_flag_wait: bad arguments");
  // ~2 GHz SM clock: cycles per ms, generous (the bound only has to stop a hang)
  const long long cycles = (long long)timeout_ms * 2000000ll;
  flag_wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((const unsigned long long*)d_flag, value,
                                                      cycles, d_status);
  return check_launch("flag_wait");
}

