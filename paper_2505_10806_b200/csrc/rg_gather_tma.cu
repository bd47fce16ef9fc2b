// K7 variant: bundle gather with TMA bulk copies (cp.async.bulk).
//
// Same contract as rg_gather_bundle (prefetch.py:41-88 semantics, route
// words, provenance counters), but each row moves global -> shared ->
// global through the Tensor Memory Accelerator: one warp per CTA, every lane
// owns a private ring of kSlots shared-memory row slots and runs a software
// pipeline (bulk load with mbarrier completion -> bulk store with bulk-group
// completion).  The bytes in flight live in shared memory, not registers, so
// the kernel needs one warp per SM and leaves the SM's warp slots and
// register file to the concurrently running sampler (the two-stream overlap
// of WorkerPipeline.step_overlapped).
#include <cstdlib>

#include "rg_common.cuh"

namespace rg {
namespace {

struct TBases {
  const float* p[16];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(uint32_t dst_smem, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst_smem),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(src_smem), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

constexpr int kS = 2;           // loads in flight per lane
constexpr int kSlots = 2 * kS;  // + stores in flight per lane

// rows of batch b: [0, nids[b]); CTA c of the batch's CTAs owns rows
// r = (c*32 + lane) + t*(ctas*32).  Per lane: row L is loaded into slot
// L % kSlots; at the same time row L - kS (loaded kS rows ago) is stored
// from its slot; a slot is reloaded only after the store that used it, kS
// stores back, has finished reading shared memory (wait_group.read kS).
__global__ void __launch_bounds__(32)
    gather_tma_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ nids,
                      int64_t cap, const uint32_t* __restrict__ route,
                      const __grid_constant__ TBases bases, int src_stride, int stride,
                      int my_part, float* __restrict__ out, uint32_t* __restrict__ counters) {
  extern __shared__ __align__(128) uint8_t s_rows[];
  __shared__ __align__(8) uint64_t s_bar[32 * kSlots];
  __shared__ int32_t s_dst[32 * kSlots];  // destination row of each slot (-1: none)
  const int lane = threadIdx.x;
  const int b = blockIdx.y;
  const uint32_t row_bytes = (uint32_t)stride * 4u;
  const uint32_t slot_bytes = (row_bytes + 127u) & ~127u;
  for (int i = 0; i < kSlots; ++i) mbar_init(smem_u32(&s_bar[lane * kSlots + i]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int nrows = nids[b];
  const int64_t step = (int64_t)gridDim.x * 32;
  uint32_t c_local = 0, c_hit = 0, c_fb = 0, c_bad = 0, omask = 0;
  uint32_t parity = 0;  // per-slot phase parity of the next wait
  float* outb = out + (int64_t)b * cap * stride;
  auto store_slot = [&](int slot) {
    const uint32_t bar = smem_u32(&s_bar[lane * kSlots + slot]);
    mbar_wait(bar, (parity >> slot) & 1u);
    parity ^= 1u << slot;
    const int32_t dr = s_dst[lane * kSlots + slot];
    if (dr >= 0)
      bulk_store(outb + (int64_t)dr * stride,
                 smem_u32(s_rows + (lane * kSlots + slot) * slot_bytes), row_bytes);
    bulk_commit();  // one group per stored slot (empty groups keep the count exact)
  };
  int64_t L = 0;  // rows loaded by this lane
  for (int64_t r = (int64_t)blockIdx.x * 32 + lane; r < nrows; r += step) {
    const int32_t id = __ldg(ids + (int64_t)b * cap + r);
    const uint32_t rt = __ldg(route + id);
    const int kind = (int)(rt >> RG_KIND_SHIFT);
    const float* bp = rt != RG_ROUTE_INVALID ? bases.p[kind] : nullptr;
    if (L >= kS) store_slot((int)((L - kS) % kSlots));
    const int slot = (int)(L % kSlots);
    if (L >= kSlots) bulk_wait_read<kS>();  // the store that used `slot` is done reading
    const uint32_t bar = smem_u32(&s_bar[lane * kSlots + slot]);
    s_dst[lane * kSlots + slot] = bp ? (int32_t)r : -1;
    if (bp) {
      mbar_expect_tx(bar, row_bytes);
      bulk_load(smem_u32(s_rows + (lane * kSlots + slot) * slot_bytes),
                bp + (int64_t)(rt & RG_ROW_MASK) * src_stride, row_bytes, bar);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
      // invalid route word: zero row, as rg_gather_bundle writes it
      float4* z = reinterpret_cast<float4*>(outb + r * stride);
      for (int c = 0; c < stride / 4; ++c) z[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    ++L;
    if (!bp) {
      ++c_bad;
    } else if (kind == my_part) {
      ++c_local;
    } else if (kind == (int)RG_KIND_CACHE) {
      ++c_hit;
    } else {
      ++c_fb;
      omask |= 1u << kind;
    }
  }
  for (int64_t k = L < kS ? 0 : L - kS; k < L; ++k) store_slot((int)(k % kSlots));
  bulk_wait_all();
  __syncwarp();
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    c_local += __shfl_xor_sync(kFull, c_local, o);
    c_hit += __shfl_xor_sync(kFull, c_hit, o);
    c_fb += __shfl_xor_sync(kFull, c_fb, o);
    c_bad += __shfl_xor_sync(kFull, c_bad, o);
    omask |= __shfl_xor_sync(kFull, omask, o);
  }
  if (lane == 0) {
    uint32_t* g = counters + (int64_t)b * RG_NCOUNTERS;
    if (c_local) atomicAdd(g + RG_CNT_LOCAL, c_local);
    if (c_hit) atomicAdd(g + RG_CNT_HIT, c_hit);
    if (c_fb) atomicAdd(g + RG_CNT_FALLBACK, c_fb);
    if (c_bad) atomicAdd(g + RG_CNT_BAD, c_bad);
    if (omask) atomicOr(g + RG_CNT_OWNER_MASK, omask);
  }
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_gather_bundle_tma(const int32_t* d_ids, const int32_t* d_nids, int64_t cap,
                                    int32_t G, const uint32_t* d_route,
                                    const float* const* h_bases, int32_t src_stride,
                                    int32_t stride, int32_t my_part, float* d_out,
                                    uint32_t* d_counters, int32_t ctas_per_sm, void* stream) {
  RG_REQUIRE(G >= 1 && G <= 65535 && cap >= 1, "rg_gather_bundle_tma: bad sizes");
  RG_REQUIRE(stride >= 4 && stride % 4 == 0 && src_stride >= stride && src_stride % 4 == 0,
             "rg_gather_bundle_tma: bad strides");
  RG_REQUIRE(((uintptr_t)d_out & 15) == 0, "rg_gather_bundle_tma: output not 16-byte aligned");
  TBases bases;
  for (int i = 0; i < 16; ++i) {
    bases.p[i] = h_bases[i];
    RG_REQUIRE(((uintptr_t)bases.p[i] & 15) == 0, "rg_gather_bundle_tma: base %d misaligned", i);
  }
  const int slot_bytes = (stride * 4 + 127) & ~127;
  const int smem = 32 * kSlots * slot_bytes;
  if (smem > 200 * 1024) {
    set_error("rg_gather_bundle_tma: row of %d floats too large", stride);
    return RG_ERR_UNSUPPORTED;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gather_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_set = true;
  }
  const int per_sm = ctas_per_sm > 0 ? ctas_per_sm : 4;
  const int64_t want = (cap + 31) / 32;
  const int gx = (int)std::max<int64_t>(
      1, std::min<int64_t>(want, ((int64_t)kNumSMs * per_sm + G - 1) / G));
  gather_tma_kernel<<<dim3(gx, G), 32, smem, (cudaStream_t)stream>>>(
      d_ids, d_nids, cap, d_route, bases, src_stride, stride, my_part, d_out, d_counters);
  return check_launch("gather_tma");
}
