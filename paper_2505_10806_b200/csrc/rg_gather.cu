// K6/K7: feature-bundle gather, cache fill and pull routing.
//
// Reference: gnnpipe/prefetch.py:41-88 (assemble_bundle), cache.py:54-78
// (FeatureCache.lookup), store.py:66-69 (rows_for_local) and
// store.py:173-196 (StoreClient._pull).  The reference splits a request
// into local / cache-hit / fallback ids with searchsorted passes and pulls
// fallback rows per owner through a byte codec.  Here every node carries one
// 32-bit route word (owner or cache kind + row index); a warp
// copies 32 consecutive bundle rows at a time: one coalesced id load, one
// route load per row, then the rows' 16-byte vectors are streamed with all
// 32 lanes busy (flattened row x vector index) and written back contiguously.
// Source rows may live in this GPU's HBM or in a peer GPU's shard (NVLink
// P2P pointer); the kernel does not distinguish.
#include <atomic>
#include <cstdlib>

#include "rg_common.cuh"

namespace rg {
namespace {

constexpr int kGatherWarps = 8;
constexpr int kUnroll = 8;
#ifndef RG_UNROLL_PEER
#define RG_UNROLL_PEER 8
#endif
constexpr int kUnrollPeer = RG_UNROLL_PEER;  // loads in flight per lane, peer path

struct Bases {
  const float* p[16];
};

// kRowAligned (used when some shards live on peer GPUs): one row (or a
// 32-vector slice of one) per warp instruction, so every load is a single
// row-local segment — NVLink peer reads of 400-B rows run ~12 % faster that
// way (tools/nvlink_probe.py) while HBM-local rows prefer the flattened
// all-lanes-busy mapping of the default instantiation.
template <bool kRowAligned>
__global__ void __launch_bounds__(kGatherWarps * 32, 4)
    gather_bundle_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ nids,
                         int64_t cap, const uint32_t* __restrict__ route, const __grid_constant__ Bases bases,
                         int src_stride, int stride, int nvec, int dq, int dr, int my_part,
                         uint32_t peer_mask, float* __restrict__ out,
                         uint32_t* __restrict__ counters) {
  __shared__ uint32_t s_cnt[RG_NCOUNTERS];
  __shared__ const float* s_base[16];
  const int b = blockIdx.y;
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x < RG_NCOUNTERS) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x < 16) s_base[threadIdx.x] = bases.p[threadIdx.x];
  __syncthreads();
  const int nrows = nids[b];
  uint32_t c_local = 0, c_hit = 0, c_fb = 0, c_bad = 0, c_peer = 0, omask = 0;
  const int64_t warp_stride = (int64_t)gridDim.x * kGatherWarps * 32;
  for (int64_t r0 = ((int64_t)blockIdx.x * kGatherWarps + warp) * 32; r0 < nrows;
       r0 += warp_stride) {
    const int64_t row = r0 + lane;
    const bool valid = row < nrows;
    const int nr = (int)(nrows - r0 < 32 ? nrows - r0 : 32);
    uint32_t rt = RG_ROUTE_INVALID;
    if (valid) rt = __ldg(route + __ldg(ids + (int64_t)b * cap + row));
    const int kind = (int)(rt >> RG_KIND_SHIFT);
    const float* bp = (valid && rt != RG_ROUTE_INVALID) ? s_base[kind] : nullptr;
    const bool bad = valid && bp == nullptr;
    const bool local = valid && !bad && kind == my_part;
    const bool hit = valid && !bad && kind == (int)RG_KIND_CACHE;
    const bool fb = valid && !bad && !local && !hit;
    c_local += __popc(__ballot_sync(kFull, local));
    c_hit += __popc(__ballot_sync(kFull, hit));
    c_fb += __popc(__ballot_sync(kFull, fb));
    c_bad += __popc(__ballot_sync(kFull, bad));
    c_peer += __popc(__ballot_sync(kFull, fb && ((peer_mask >> kind) & 1u)));
    omask |= __reduce_or_sync(kFull, fb ? (1u << kind) : 0u);
    const float* src = nullptr;
    if (bp) src = bp + (int64_t)(rt & RG_ROW_MASK) * src_stride;
    const unsigned long long srcu = reinterpret_cast<unsigned long long>(src);
    float4* dst = reinterpret_cast<float4*>(out + ((int64_t)b * cap + r0) * stride);
    if (kRowAligned) {
      constexpr int kU = kUnrollPeer;
      const int chunks = (nvec + 31) >> 5;
      const int items = nr * chunks;
      for (int i0 = 0; i0 < items; i0 += kU) {
        float4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int it = i0 + u;
          const int rr = chunks == 1 ? it : it / chunks;
          const int c = (it - rr * chunks) * 32 + lane;
          const unsigned long long sp = __shfl_sync(kFull, srcu, rr & 31);
          v[u] = (it < items && c < nvec && sp)
                     ? ld_stream(reinterpret_cast<const float4*>(sp) + c)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int it = i0 + u;
          const int rr = chunks == 1 ? it : it / chunks;
          const int c = (it - rr * chunks) * 32 + lane;
          if (it < items && c < nvec) st_stream(dst + rr * nvec + c, v[u]);
        }
      }
      continue;
    }
    const int total = nr * nvec;
    // lane handles flattened vectors e = lane, lane+32, ...: row e/nvec, col e%nvec
    int er = lane / nvec, ec = lane - (lane / nvec) * nvec;
    for (int e0 = 0; e0 < total; e0 += 32 * kUnroll) {
      float4 v[kUnroll];
      int rr[kUnroll], cc[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        rr[u] = er;
        cc[u] = ec;
        ec += dr;
        er += dq;
        if (ec >= nvec) {
          ec -= nvec;
          ++er;
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const unsigned long long sp = __shfl_sync(kFull, srcu, rr[u] & 31);
        const int e = e0 + u * 32 + lane;
        if (e < total && sp)
          v[u] = ld_stream(reinterpret_cast<const float4*>(sp) + cc[u]);
        else
          v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int e = e0 + u * 32 + lane;
        if (e < total) st_stream(dst + e, v[u]);
      }
    }
  }
  if (lane == 0) {
    atomicAdd(&s_cnt[RG_CNT_LOCAL], c_local);
    atomicAdd(&s_cnt[RG_CNT_HIT], c_hit);
    atomicAdd(&s_cnt[RG_CNT_FALLBACK], c_fb);
    atomicAdd(&s_cnt[RG_CNT_BAD], c_bad);
    atomicAdd(&s_cnt[RG_CNT_PEER], c_peer);
    atomicOr(&s_cnt[RG_CNT_OWNER_MASK], omask);
  }
  __syncthreads();
  if (threadIdx.x < RG_NCOUNTERS) {
    const uint32_t x = s_cnt[threadIdx.x];
    if (x) {
      uint32_t* g = counters + (int64_t)b * RG_NCOUNTERS + threadIdx.x;
      if (threadIdx.x == RG_CNT_OWNER_MASK)
        atomicOr(g, x);
      else
        atomicAdd(g, x);
    }
  }
}

// ---- launch-wide work queue (local rows) -----------------------------------
// Same copy as the flattened path above, but 32-row chunks are pulled from a
// launch-wide queue instead of each CTA striding over one batch: items
// k = c*G + b (chunk c of batch b) chunk-major, so the work in flight at any
// time spans every batch at the same chunk index (hub rows, low ids, are
// shared across batches and stay in L2) and the tail balances across SMs.
// Provenance counters accumulate per CTA per batch in shared memory.
constexpr int kQueueMaxG = 128;  // batches with shared-memory counters
constexpr unsigned kGatherClaim = 4;

__global__ void __launch_bounds__(kGatherWarps * 32, 4)
    gather_queue_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ nids,
                        int64_t cap, int G, const uint32_t* __restrict__ route,
                        const __grid_constant__ Bases bases, int src_stride, int stride,
                        int nvec, int dq, int dr, int my_part, uint32_t peer_mask,
                        float* __restrict__ out, uint32_t* __restrict__ counters,
                        unsigned* __restrict__ queue) {
  __shared__ uint32_t s_cnt[kQueueMaxG][RG_NCOUNTERS];
  __shared__ int32_t s_nr[kQueueMaxG];
  __shared__ const float* s_base[16];
  __shared__ unsigned s_maxc;
  const int lane = lane_id();
  for (int i = threadIdx.x; i < kQueueMaxG * RG_NCOUNTERS; i += blockDim.x)
    (&s_cnt[0][0])[i] = 0;
  if (threadIdx.x < 16) s_base[threadIdx.x] = bases.p[threadIdx.x];
  if (threadIdx.x == 0) s_maxc = 0;
  __syncthreads();
  unsigned mc = 0;
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    const int n = nids[i];
    s_nr[i] = n;
    mc = max(mc, (unsigned)((n + 31) / 32));
  }
  atomicMax(&s_maxc, mc);
  __syncthreads();
  const unsigned items = s_maxc * (unsigned)G;
  for (;;) {
    unsigned t0 = 0;
    if (lane == 0) t0 = atomicAdd(queue, kGatherClaim);
    t0 = __shfl_sync(kFull, t0, 0);
    if (t0 >= items) break;
    int c = (int)(t0 / (unsigned)G);  // one division per claim
    int b = (int)(t0 - (unsigned)c * (unsigned)G) - 1;
#pragma unroll 1
    for (unsigned k = t0; k < t0 + kGatherClaim && k < items; ++k) {
      if (++b == G) {
        b = 0;
        ++c;
      }
      const int nrows = s_nr[b];
      const int64_t r0 = (int64_t)c * 32;
      if (r0 >= nrows) continue;
      const int64_t row = r0 + lane;
      const bool valid = row < nrows;
      const int nr = (int)(nrows - r0 < 32 ? nrows - r0 : 32);
      uint32_t rt = RG_ROUTE_INVALID;
      if (valid) rt = __ldg(route + __ldg(ids + (int64_t)b * cap + row));
      const int kind = (int)(rt >> RG_KIND_SHIFT);
      const float* bp = (valid && rt != RG_ROUTE_INVALID) ? s_base[kind] : nullptr;
      const bool bad = valid && bp == nullptr;
      const bool local = valid && !bad && kind == my_part;
      const bool hit = valid && !bad && kind == (int)RG_KIND_CACHE;
      const bool fb = valid && !bad && !local && !hit;
      const unsigned n_local = __popc(__ballot_sync(kFull, local));
      const unsigned n_hit = __popc(__ballot_sync(kFull, hit));
      const unsigned n_fb = __popc(__ballot_sync(kFull, fb));
      const unsigned n_bad = __popc(__ballot_sync(kFull, bad));
      const unsigned om = __reduce_or_sync(kFull, fb ? (1u << kind) : 0u);
      const unsigned n_peer =
          peer_mask ? __popc(__ballot_sync(kFull, fb && ((peer_mask >> kind) & 1u))) : 0u;
      if (lane == 0) {
        uint32_t* sc = s_cnt[b];
        if (n_peer) atomicAdd(sc + RG_CNT_PEER, n_peer);
        if (n_local) atomicAdd(sc + RG_CNT_LOCAL, n_local);
        if (n_hit) atomicAdd(sc + RG_CNT_HIT, n_hit);
        if (n_fb) atomicAdd(sc + RG_CNT_FALLBACK, n_fb);
        if (n_bad) atomicAdd(sc + RG_CNT_BAD, n_bad);
        if (om) atomicOr(sc + RG_CNT_OWNER_MASK, om);
      }
      const float* src = nullptr;
      if (bp) src = bp + (int64_t)(rt & RG_ROW_MASK) * src_stride;
      const unsigned long long srcu = reinterpret_cast<unsigned long long>(src);
      float4* dst = reinterpret_cast<float4*>(out + ((int64_t)b * cap + r0) * stride);
      const int total = nr * nvec;
      int er = lane / nvec, ec = lane - (lane / nvec) * nvec;
      for (int e0 = 0; e0 < total; e0 += 32 * kUnroll) {
        float4 v[kUnroll];
        int rr[kUnroll], cc[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          rr[u] = er;
          cc[u] = ec;
          ec += dr;
          er += dq;
          if (ec >= nvec) {
            ec -= nvec;
            ++er;
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const unsigned long long sp = __shfl_sync(kFull, srcu, rr[u] & 31);
          const int e = e0 + u * 32 + lane;
          if (e < total && sp)
            v[u] = ld_stream(reinterpret_cast<const float4*>(sp) + cc[u]);
          else
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int e = e0 + u * 32 + lane;
          if (e < total) st_stream(dst + e, v[u]);
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * RG_NCOUNTERS; i += blockDim.x) {
    const int b = i / RG_NCOUNTERS, k = i - b * RG_NCOUNTERS;
    const uint32_t x = s_cnt[b][k];
    if (x) {
      uint32_t* g = counters + (int64_t)b * RG_NCOUNTERS + k;
      if (k == RG_CNT_OWNER_MASK)
        atomicOr(g, x);
      else
        atomicAdd(g, x);
    }
  }
}

// ---- group gather from the input bitmaps -----------------------------------
// The group's input sets as the sampler leaves them: bm[b][w] (bit j of word
// w = node 32w+j is in batch b's input set) and wpre[b][w] (rank of node 32w
// in that sorted set).  No id list is read: a window's set bits give the
// ids, its wpre entry the output rank of its first row.
#ifndef RG_STAGED_MIN_CTAS
#define RG_STAGED_MIN_CTAS 4
#endif

// ---- staged union gather: each source row read once per group -------------
// A gather that reads every batch's rows separately moves each bundle row
// through L2 twice (the source read — an L2 hit for all but the first batch
// — and the write): 68.8 GB of L2 traffic per G = 128 Products launch, while
// the bundle writes alone (34.4 GB) need ~4.6 ms at the measured write-only
// HBM rate (7.5 TB/s, tools/hbm_probe.py).  Here a CTA owns a window of
// 32*kW ids for ALL G batches: phase 1 stages every present source row of
// the window in shared memory (each row read from HBM once per group);
// phase 2 writes, batch by batch, that batch's rows of the window as one
// contiguous run (ranks wpre[b][w0] ..).  (A warp-per-id scatter — each row
// stored straight to every batch holding it — reads once too but scatters
// 400-B writes over all G bundles at once and measured 11.7 ms: HBM write
// locality matters more than the reads.)
// kBulk: phase 2 hands each run of consecutive present ids to the TMA engine
// as one bulk shared->global copy (cp.async.bulk; rows are 16-B multiples),
// issued by the lane that owns the run's first id, instead of moving 16-B
// vectors through registers; the staging buffer is double-buffered so
// window k+1 is loaded while the bulk copies of window k drain.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* gdst, const void* ssrc, uint32_t bytes,
                                              uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int kW, bool kBulk>
__global__ void __launch_bounds__(kGatherWarps * 32, RG_STAGED_MIN_CTAS)
    gather_staged_kernel(const uint32_t* __restrict__ bm, const int32_t* __restrict__ wpre,
                         int64_t nwords, int G, int64_t cap, const uint32_t* __restrict__ route,
                         const __grid_constant__ Bases bases, int src_stride, int stride,
                         int nvec, int dq, int dr, int my_part, uint32_t peer_mask,
                         float* __restrict__ out, uint32_t* __restrict__ counters,
                         unsigned* __restrict__ queue, int hint) {
  constexpr int kIds = 32 * kW;
  // bulk stores marked evict-first: the bundle is not re-read here (Products
  // G = 128: 5.81 vs 5.87 ms per launch; evict_last 5.90, evict_unchanged 5.86)
  uint64_t pol = 0;
  if (hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  extern __shared__ float4 s_rows[];  // [kIds][nvec]
  __shared__ uint32_t s_cnt[kQueueMaxG][RG_NCOUNTERS];
  __shared__ const float* s_base[16];
  __shared__ unsigned long long s_src[kIds];
  __shared__ uint32_t s_present[kW], s_mloc[kW], s_mhit[kW], s_mfb[kW], s_mbad[kW], s_mpeer[kW];
  __shared__ uint32_t s_mq[16][kW];  // fallback ids per owner kind
  __shared__ uint32_t s_fbkinds;
  __shared__ uint32_t s_words[kQueueMaxG * kW];  // bm[b][w0 + q] of every batch
  __shared__ int32_t s_rbase[kQueueMaxG];         // wpre[b][w0]
  __shared__ unsigned s_win;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int i = threadIdx.x; i < kQueueMaxG * RG_NCOUNTERS; i += blockDim.x)
    (&s_cnt[0][0])[i] = 0;
  if (threadIdx.x < 16) s_base[threadIdx.x] = bases.p[threadIdx.x];
  const int64_t nwin = (nwords + kW - 1) / kW;
  const uint32_t row_bytes = (uint32_t)nvec * 16u;
  for (unsigned it = 0;; ++it) {
    // kBulk: the bulk copies that read this window's staging buffer (issued
    // two windows ago) have finished reading it
    if constexpr (kBulk) bulk_wait_read1();
    __syncthreads();  // previous window fully written out; counters zeroed
    float4* rows = s_rows + (kBulk ? (it & 1u) * (unsigned)(kIds * nvec) : 0u);
    if (threadIdx.x == 0) s_win = atomicAdd(queue, 1u);
    if (threadIdx.x < kW) s_present[threadIdx.x] = 0;
    if (threadIdx.x < 16 * kW) (&s_mq[0][0])[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_fbkinds = 0;
    __syncthreads();
    const int64_t win = s_win;
    if (win >= nwin) break;
    const int64_t w0 = win * kW;
    // phase 1a: the group's words of the window (kept for phase 2), their
    // union, and every batch's rank base
    for (int i = threadIdx.x; i < G * kW; i += blockDim.x) {
      const int bb = i / kW, q = i - bb * kW;
      uint32_t x = 0;
      if (w0 + q < nwords) x = __ldg(bm + (int64_t)bb * nwords + w0 + q);
      s_words[i] = x;
      if (x) atomicOr(&s_present[q], x);
    }
    for (int bb = threadIdx.x; bb < G; bb += blockDim.x) s_rbase[bb] = __ldg(wpre + (int64_t)bb * nwords + w0);
    __syncthreads();
    // phase 1b: route / kind / source address per id (warp q <-> word q)
    if (warp < kW) {
      const uint32_t pres = s_present[warp];
      const bool here = (pres >> lane) & 1u;
      const int64_t id = (w0 + warp) * 32 + lane;
      const uint32_t rt = here ? __ldg(route + id) : RG_ROUTE_INVALID;
      const int kind = (int)(rt >> RG_KIND_SHIFT);
      const float* bp = (here && rt != RG_ROUTE_INVALID) ? s_base[kind] : nullptr;
      const bool bad = here && bp == nullptr;
      const bool local = here && !bad && kind == my_part;
      const bool hit = here && !bad && kind == (int)RG_KIND_CACHE;
      const bool fb = here && !bad && !local && !hit;
      const unsigned mfb = __ballot_sync(kFull, fb);
      const unsigned mloc = __ballot_sync(kFull, local), mhit = __ballot_sync(kFull, hit);
      const unsigned mbad = __ballot_sync(kFull, bad);
      const unsigned mpeer = __ballot_sync(kFull, fb && ((peer_mask >> kind) & 1u));
      if (lane == 0) {
        s_mloc[warp] = mloc;
        s_mhit[warp] = mhit;
        s_mfb[warp] = mfb;
        s_mbad[warp] = mbad;
        s_mpeer[warp] = mpeer;
      }
      if (fb) atomicOr(&s_mq[kind][warp], 1u << lane);
      const unsigned kinds = __reduce_or_sync(kFull, fb ? (1u << kind) : 0u);
      s_src[warp * 32 + lane] = reinterpret_cast<unsigned long long>(
          bp ? bp + (int64_t)(rt & RG_ROW_MASK) * src_stride : nullptr);
      if (lane == 0 && kinds) atomicOr(&s_fbkinds, kinds);
    }
    __syncthreads();
    // phase 1c: stage the present rows; warp w copies ids 4w.. (row-aligned:
    // lane c moves vector c, four rows' loads in flight per lane)
    {
      constexpr int kR = 4;
      for (int r0 = warp * kR; r0 < kIds; r0 += kGatherWarps * kR) {
        unsigned long long sp[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) sp[u] = s_src[r0 + u];
        for (int c = lane; c < nvec; c += 32) {
          float4 v[kR];
#pragma unroll
          for (int u = 0; u < kR; ++u)
            v[u] = sp[u] ? ld_stream(reinterpret_cast<const float4*>(sp[u]) + c)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < kR; ++u) rows[(r0 + u) * nvec + c] = v[u];
        }
      }
    }
    if constexpr (kBulk) fence_proxy_async_smem();  // staged rows -> the TMA's view
    __syncthreads();
    // phase 2a: provenance of the window for this warp's batches, one batch
    // per lane (batch w + 8l belongs to lane l of warp w in every window, so
    // the CTA's per-batch counters need no atomics)
    {
      const int bb = warp + kGatherWarps * lane;
      if (bb < G) {
        const uint32_t fbk = s_fbkinds;
        unsigned n_loc = 0, n_hit = 0, n_fb = 0, n_bad = 0, n_peer = 0, om = 0;
#pragma unroll
        for (int q = 0; q < kW; ++q) {
          const uint32_t word = s_words[bb * kW + q];
          n_loc += __popc(word & s_mloc[q]);
          n_hit += __popc(word & s_mhit[q]);
          n_fb += __popc(word & s_mfb[q]);
          n_bad += __popc(word & s_mbad[q]);
          n_peer += __popc(word & s_mpeer[q]);
          for (unsigned kk = fbk; kk; kk &= kk - 1) {
            const int kq = __ffs(kk) - 1;
            if (word & s_mq[kq][q]) om |= 1u << kq;
          }
        }
        uint32_t* sc = s_cnt[bb];
        sc[RG_CNT_LOCAL] += n_loc;
        sc[RG_CNT_HIT] += n_hit;
        sc[RG_CNT_FALLBACK] += n_fb;
        sc[RG_CNT_BAD] += n_bad;
        sc[RG_CNT_PEER] += n_peer;
        sc[RG_CNT_OWNER_MASK] |= om;
      }
    }
    // phase 2b: each batch's run of the window, contiguous
    if constexpr (kBulk) {
      // lane l owns id 32q + l.  Consecutive ids of the batch are
      // consecutive rows both in the staging buffer and in the batch's run,
      // so each maximal run of set bits (across word boundaries) is one bulk
      // copy, issued by the lane of its first id; its output rank is the
      // popcount of the batch's bits below it.
      for (int bb = warp; bb < G; bb += kGatherWarps) {
        uint32_t wd[kW];
#pragma unroll
        for (int q = 0; q < kW; ++q) wd[q] = s_words[bb * kW + q];
        int r = s_rbase[bb];
        float* dstb = out + (int64_t)bb * cap * stride;
#pragma unroll
        for (int q = 0; q < kW; ++q) {
          const uint32_t word = wd[q];
          const bool prev = lane ? (word >> (lane - 1)) & 1u : (q ? wd[q - 1] >> 31 : 0u);
          if (((word >> lane) & 1u) && !prev) {
            // trailing ones from this id on, continued into the next words
            int len = __clz(__brev(~(word >> lane)));
            bool open = len == 32 - lane;
#pragma unroll
            for (int q2 = q + 1; q2 < kW; ++q2) {
              if (open) {
                const int t = __clz(__brev(~wd[q2]));
                len += t;
                open = t == 32;
              }
            }
            if (hint)
              bulk_s2g_hint(dstb + (int64_t)(r + __popc(word & lt)) * stride,
                            rows + (q * 32 + lane) * nvec, row_bytes * (uint32_t)len, pol);
            else
              bulk_s2g(dstb + (int64_t)(r + __popc(word & lt)) * stride, rows + (q * 32 + lane) * nvec,
                       row_bytes * (uint32_t)len);
          }
          r += __popc(word);
        }
      }
      bulk_commit();
      continue;
    }
    for (int bb = warp; bb < G; bb += kGatherWarps) {
      const uint32_t wd = lane < kW ? s_words[bb * kW + lane] : 0u;
      if (__reduce_or_sync(kFull, wd) == 0u) continue;
      const int base = s_rbase[bb];
      // the batch's rows in id order = consecutive output rows; four rows per
      // step, lane c moves vector c of each (no per-element index math)
      float4* dst = reinterpret_cast<float4*>(out + ((int64_t)bb * cap + base) * stride);
      int k = 0;
#pragma unroll 1
      for (int q = 0; q < kW; ++q) {
        uint32_t word = __shfl_sync(kFull, wd, q);
        while (word) {
          int j[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            j[u] = word ? q * 32 + __ffs(word) - 1 : -1;
            word &= word - 1;
          }
          for (int c = lane; c < nvec; c += 32) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (j[u] >= 0) v[u] = rows[j[u] * nvec + c];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (j[u] >= 0) st_stream(dst + (int64_t)(k + u) * nvec + c, v[u]);
          }
          k += (j[0] >= 0) + (j[1] >= 0) + (j[2] >= 0) + (j[3] >= 0);
        }
      }
    }
  }
  if constexpr (kBulk) bulk_wait_all();  // the staging buffers outlive every copy
  __syncthreads();
  for (int i = threadIdx.x; i < G * RG_NCOUNTERS; i += blockDim.x) {
    const int bb = i / RG_NCOUNTERS, k = i - bb * RG_NCOUNTERS;
    const uint32_t x = s_cnt[bb][k];
    if (x) {
      uint32_t* g = counters + (int64_t)bb * RG_NCOUNTERS + k;
      if (k == RG_CNT_OWNER_MASK)
        atomicOr(g, x);
      else
        atomicAdd(g, x);
    }
  }
}

// per-device ring of queue counters: one slot per launch (zeroed on the
// launch stream), so concurrent gathers on different streams never share
unsigned* queue_slot(cudaStream_t s) {
  constexpr int kSlots = 1024;
  static unsigned* ring[16] = {};
  static std::atomic<unsigned> next{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  if (!ring[dev] && cudaMalloc(&ring[dev], kSlots * sizeof(unsigned)) != cudaSuccess) {
    ring[dev] = nullptr;
    return nullptr;
  }
  unsigned* q = ring[dev] + (next.fetch_add(1) % kSlots);
  if (cudaMemsetAsync(q, 0, sizeof(unsigned), s) != cudaSuccess) return nullptr;
  return q;
}

__global__ void route_copy_kernel(const uint32_t* __restrict__ base, int64_t n,
                                  uint32_t* __restrict__ route) {
  const int64_t n4 = n / 4;
  const uint4* b4 = reinterpret_cast<const uint4*>(base);
  uint4* r4 = reinterpret_cast<uint4*>(route);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    r4[i] = b4[i];
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    route[i] = base[i];
}

__global__ void route_scatter_kernel(const int32_t* __restrict__ hot, int64_t n_hot,
                                     uint32_t* __restrict__ route) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_hot;
       i += (int64_t)gridDim.x * blockDim.x)
    route[hot[i]] = (RG_KIND_CACHE << RG_KIND_SHIFT) | (uint32_t)i;
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_gather_bundle(const int32_t* d_ids, const int32_t* d_nids, int64_t cap,
                                int32_t G, const uint32_t* d_route, const float* const* h_bases,
                                int32_t src_stride, int32_t stride, int32_t my_part,
                                uint32_t peer_mask, float* d_out, uint32_t* d_counters,
                                void* stream) {
  RG_REQUIRE(G >= 1 && G <= 65535 && cap >= 1, "rg_gather_bundle: bad sizes");
  RG_REQUIRE(stride >= 4 && stride % 4 == 0, "rg_gather_bundle: stride %d not a multiple of 4",
             stride);
  RG_REQUIRE(src_stride >= stride && src_stride % 4 == 0,
             "rg_gather_bundle: src_stride %d < stride %d or not a multiple of 4", src_stride,
             stride);
  RG_REQUIRE(((uintptr_t)d_out & 15) == 0, "rg_gather_bundle: output not 16-byte aligned");
  Bases bases;
  for (int i = 0; i < 16; ++i) {
    bases.p[i] = h_bases[i];
    RG_REQUIRE(((uintptr_t)bases.p[i] & 15) == 0, "rg_gather_bundle: base %d misaligned", i);
  }
  const int nvec = stride / 4;
  const int dq = 32 / nvec, dr = 32 % nvec;

  // enough CTAs for ~4 resident per SM on the largest slot; extra CTAs of a
  // short batch exit after one bounds check.
  // One wave: (SMs x 3) CTAs split evenly over the G batches (each CTA
  // grid-strides over its batch's rows).  Measured (profiles/r01_summary.md):
  // 3/SM single wave 6.39 TB/s; 4/SM (a 16-CTA second wave at G=32) 5.15;
  // 8/SM (two waves) 5.94.  Inside the overlapped step (the next group's
  // sampling on a second stream) 4/SM is ~2 % faster end to end (8,080 vs
  // 7,920 batches/s) though the gather alone drops to ~6.2 TB/s: 4/SM is
  // the default.
  // With peer (NVLink) shards the gather is latency-bound on remote reads:
  // 6 CTAs/SM (1.5 waves) measured best at N = 2 (9,355 vs 8,930 batches/s
  // at 3/SM; 8/SM 9,129).
  // knobs read per call (diagnostic sweeps set them between launches)
  auto env_int = [](const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
  };
  const int env_ctas = std::max(0, env_int("RG_GATHER_CTAS_PER_SM", 0));
  const int ctas_per_sm = env_ctas ? env_ctas : (peer_mask ? 6 : 4);
  const int64_t want = (cap + kGatherWarps * 32 - 1) / (kGatherWarps * 32);
  const int gx = (int)std::max<int64_t>(
      1, std::min<int64_t>(want, ((int64_t)kNumSMs * ctas_per_sm) / G));
  const bool use_queue = env_int("RG_GATHER_QUEUE", 1) != 0;
  // peer shards: the per-batch row-aligned kernel below.  The queue (opt-in
  // with RG_GATHER_PEER_QUEUE=1, rows of 32 vectors only, where its
  // flattened mapping is row-aligned too) measured slower with NVLink rows:
  // papers100M-shaped N = 2, 1,991 (3 CTAs/SM) / 1,981 (4) vs 2,152 batches/s
  const bool peer_queue = peer_mask == 0 || (nvec == 32 && env_int("RG_GATHER_PEER_QUEUE", 0));
  if (peer_queue && G <= kQueueMaxG && use_queue &&
      (uint64_t)G * (uint64_t)((cap + 31) / 32) < (1ull << 32) - kGatherClaim) {
    unsigned* q = queue_slot((cudaStream_t)stream);
    if (!q) return check_launch("gather queue");
    // 3 CTAs/SM measured best for the queue (Products G = 128: 3 -> 11,877,
    // 4 -> 11,753, 2 -> 11,249 batches/s)
    const int qctas = env_ctas ? env_ctas : 3;
    gather_queue_kernel<<<kNumSMs * qctas, kGatherWarps * 32, 0, (cudaStream_t)stream>>>(
        d_ids, d_nids, cap, G, d_route, bases, src_stride, stride, nvec, dq, dr, my_part,
        peer_mask, d_out, d_counters, q);
    return check_launch("gather_queue");
  }
  if (peer_mask != 0)
    gather_bundle_kernel<true><<<dim3(gx, G), kGatherWarps * 32, 0, (cudaStream_t)stream>>>(
        d_ids, d_nids, cap, d_route, bases, src_stride, stride, nvec, dq, dr, my_part, peer_mask,
        d_out, d_counters);
  else
    gather_bundle_kernel<false><<<dim3(gx, G), kGatherWarps * 32, 0, (cudaStream_t)stream>>>(
        d_ids, d_nids, cap, d_route, bases, src_stride, stride, nvec, dq, dr, my_part, peer_mask,
        d_out, d_counters);
  return check_launch("gather_bundle");
}

extern "C" int rg_gather_window(const uint32_t* d_bm, const int32_t* d_wpre, int64_t nwords,
                                int32_t G, int64_t cap, const uint32_t* d_route,
                                const float* const* h_bases, int32_t src_stride, int32_t stride,
                                int32_t my_part, uint32_t peer_mask, float* d_out,
                                uint32_t* d_counters, void* stream) {
  RG_REQUIRE(G >= 1 && G <= kQueueMaxG && cap >= 1 && nwords >= 1,
             "rg_gather_window: bad sizes (G <= %d)", kQueueMaxG);
  RG_REQUIRE(nwords < (1ll << 32) - 1, "rg_gather_window: too many bitmap words");
  RG_REQUIRE(stride >= 4 && stride % 4 == 0, "rg_gather_window: stride %d not a multiple of 4",
             stride);
  RG_REQUIRE(src_stride >= stride && src_stride % 4 == 0,
             "rg_gather_window: src_stride %d < stride %d or not a multiple of 4", src_stride,
             stride);
  RG_REQUIRE(((uintptr_t)d_out & 15) == 0, "rg_gather_window: output not 16-byte aligned");
  Bases bases;
  for (int i = 0; i < 16; ++i) {
    bases.p[i] = h_bases[i];
    RG_REQUIRE(((uintptr_t)bases.p[i] & 15) == 0, "rg_gather_window: base %d misaligned", i);
  }
  const int nvec = stride / 4;
  const int dq = 32 / nvec, dr = 32 % nvec;
  unsigned* q = queue_slot((cudaStream_t)stream);
  if (!q) return check_launch("gather window queue");
  // Phase 2 by TMA bulk copies (default) or through registers
  // (RG_GATHER_BULK=0).  Products G = 128, ms per launch: bulk 128-id windows
  // 5.87, 64-id 5.99; registers 64-id 6.04, 128-id 5.97.  With the row
  // reads removed (diagnostic build) the bulk kernel still needs 5.41 ms:
  // the bundle write pattern (~6.4 TB/s here), not instruction issue (bulk
  // executes 3x fewer instructions than the register copy), bounds it.
  static const int hint = [] {
    const char* e = getenv("RG_GATHER_HINT");  // 0: no L2 policy on the bulk stores
    return e ? atoi(e) : 1;
  }();
  static const int bulk_env = [] {
    const char* e = getenv("RG_GATHER_BULK");
    return e ? atoi(e) : -1;  // -1: by size
  }();
  static const int kw_env = [] {
    const char* e = getenv("RG_GATHER_KW");  // ids per window / 32
    return e ? std::max(1, std::min(4, atoi(e))) : 0;
  }();
  // staged rows per window <= ~56 KB
  auto window_words = [&](int kw) {
    while (kw > 1 && (int64_t)32 * kw * nvec * 16 > 56 * 1024) kw >>= 1;
    return kw;
  };
  int kw = window_words(kw_env ? kw_env : 4);
  // bulk needs the staging buffer twice and enough windows per CTA for the
  // double buffer to pay (BASELINE config 0, ~6 windows per CTA: registers
  // 0.129 vs bulk 0.137 ms)
  bool bulk = bulk_env != 0 && 2 * (size_t)32 * kw * nvec * 16 <= 200 * 1024 &&
              (bulk_env == 1 || (nwords + kw - 1) / kw >= (int64_t)16 * kNumSMs);
  if (!bulk) kw = window_words(kw_env ? kw_env : 2);
  const size_t sbuf = (size_t)32 * kw * nvec * 16;  // one window's staged rows
  RG_REQUIRE(sbuf <= 200 * 1024, "rg_gather_window: rows of %d floats too wide to stage",
             stride);
  const size_t srows = bulk ? 2 * sbuf : sbuf;
  {
    cudaStream_t st = (cudaStream_t)stream;
    auto go = [&](auto kern) {
      // every call: the attribute is per kernel and per device, and all the
      // instantiations share this lambda's type (a static flag here would
      // only ever cover the first one)
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
          cudaSuccess)
        return check_launch("gather_staged attribute");
      static const int cap_sm = [] {
        const char* e = getenv("RG_GATHER_STAGED_CTAS");
        return e ? std::max(1, atoi(e)) : 0;
      }();
      static const bool reserve = [] {
        const char* e = getenv("RG_GATHER_RESERVE");
        return e ? atoi(e) != 0 : true;
      }();
      size_t dyn = srows;
      if (bulk && reserve) {
        // the TMA engine drains the stores, so 2 CTAs per SM carry the
        // launch; the rest of the SM's shared memory is reserved too, so no
        // other kernel (the next group's sampler on the other stream) lands
        // beside it: a co-resident sampler stretches the gather's
        // latency-bound staging phase (Products: 12.96 vs 9.26 ms per step)
        const int want_sm = cap_sm ? cap_sm : 2;
        int dev = 0, smem_sm = 0, reserved = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        const int64_t fill = (int64_t)smem_sm / want_sm - reserved - (int64_t)fa.sharedSizeBytes;
        dyn = (size_t)std::max<int64_t>((int64_t)srows, std::min<int64_t>(fill, 200 * 1024));
      }
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGatherWarps * 32, dyn);
      if (cap_sm) per_sm = std::min(per_sm, cap_sm);
      kern<<<kNumSMs * std::max(1, per_sm), kGatherWarps * 32, dyn, st>>>(
          d_bm, d_wpre, nwords, G, cap, d_route, bases, src_stride, stride, nvec, dq, dr, my_part,
          peer_mask, d_out, d_counters, q, hint);
      return check_launch("gather_staged");
    };
    if (bulk) {
      if (kw == 4) return go(gather_staged_kernel<4, true>);
      if (kw == 2) return go(gather_staged_kernel<2, true>);
      return go(gather_staged_kernel<1, true>);
    }
    if (kw == 4) return go(gather_staged_kernel<4, false>);
    if (kw == 2) return go(gather_staged_kernel<2, false>);
    return go(gather_staged_kernel<1, false>);
  }
}

extern "C" int rg_route_with_cache(const uint32_t* d_base_route, int64_t n, const int32_t* d_hot,
                                   int64_t n_hot, uint32_t* d_route, void* stream) {
  RG_REQUIRE(n >= 1 && n_hot >= 0, "rg_route_with_cache: bad sizes");
  RG_REQUIRE(n_hot <= (int64_t)RG_ROW_MASK, "rg_route_with_cache: n_hot too large");
  cudaStream_t s = (cudaStream_t)stream;
  if (d_route != d_base_route) {
    route_copy_kernel<<<kNumSMs * 4, 256, 0, s>>>(d_base_route, n, d_route);
    int rc = check_launch("route_copy");
    if (rc) return rc;
  }
  if (n_hot == 0) return RG_OK;
  route_scatter_kernel<<<kNumSMs * 2, 256, 0, s>>>(d_hot, n_hot, d_route);
  return check_launch("route_scatter");
}
