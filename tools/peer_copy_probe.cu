// Peer (NVLink) -> local copy rates on B200, for choosing the group
// prefetch's copy mechanism:
//   ld16     : SM kernel, contiguous, 16-B loads/stores, 8 in flight per lane
//   bulk     : cp.async.bulk global(peer) -> smem -> global(local), 16 KB chunks
//   bulk-runs: same, runs of R 400-B rows at random row offsets (the sorted
//              union of a group is mostly such runs)
//   rows16   : SM kernel, random single 400-B rows, row-aligned warp mapping
//   ce       : cudaMemcpyPeerAsync (copy engine), contiguous
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o peer_copy_probe \
//        tools/peer_copy_probe.cu ; needs 2 GPUs.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

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
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(256) ld16_kernel(const float4* __restrict__ s, float4* __restrict__ d,
                                                   int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) v[u] = __ldg(s + i);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) d[i] = v[u];
    }
  }
}

// one thread per CTA drives a ring of kSlots chunk slots; chunk k of the
// CTA's list: (src offset, dst offset, bytes)
constexpr int kSlots = 4;
__global__ void __launch_bounds__(32) bulk_kernel(const uint8_t* __restrict__ s, uint8_t* __restrict__ d,
                                                  const int64_t* __restrict__ off, const int32_t* __restrict__ len,
                                                  int64_t nchunks, int slot_bytes) {
  extern __shared__ __align__(128) uint8_t buf[];
  __shared__ __align__(8) uint64_t bar[kSlots];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kSlots; ++i) mbar_init(smem_u32(&bar[i]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t parity = 0;
  int64_t mine[kSlots];
  int32_t mlen[kSlots];
  int64_t k = blockIdx.x, issued = 0, done = 0;
  const int64_t step = gridDim.x;
  constexpr int kAhead = kSlots / 2;
  while (done < issued || k < nchunks) {
    // issue loads while fewer than kAhead outstanding
    while (k < nchunks && issued - done < kAhead) {
      const int slot = (int)(issued % kSlots);
      if (issued >= kSlots) bulk_wait_read<kAhead - 1>();  // slot's old store read out
      const uint32_t sb = smem_u32(buf + (size_t)slot * slot_bytes);
      const uint32_t b = smem_u32(&bar[slot]);
      mbar_expect_tx(b, (uint32_t)len[k]);
      bulk_load(sb, s + off[k], (uint32_t)len[k], b);
      mine[slot] = off[k];
      mlen[slot] = len[k];
      ++issued;
      k += step;
    }
    if (done < issued) {
      const int slot = (int)(done % kSlots);
      mbar_wait(smem_u32(&bar[slot]), (parity >> slot) & 1u);
      parity ^= 1u << slot;
      bulk_store(d + mine[slot], smem_u32(buf + (size_t)slot * slot_bytes), (uint32_t)mlen[slot]);
      bulk_commit();
      ++done;
    }
  }
  bulk_wait_all();
}

// random single rows (400 B = 25 float4), row-aligned warp mapping
__global__ void __launch_bounds__(256) rows16_kernel(const float4* __restrict__ s, float4* __restrict__ d,
                                                     const int64_t* __restrict__ rows, int64_t nrows) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r0 = w * 8; r0 < nrows; r0 += nw * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (r0 + u < nrows && lane < 25) v[u] = __ldg(s + rows[r0 + u] * 25 + lane);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (r0 + u < nrows && lane < 25) d[rows[r0 + u] * 25 + lane] = v[u];
  }
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  const int64_t bytes = 1ll << 30;
  CK(cudaSetDevice(1));
  uint8_t* src;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  uint8_t* dst;
  CK(cudaMalloc(&dst, bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, double nbytes, auto&& fn) {
    fn();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) fn();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("%-28s %8.1f GB/s\n", name, 5 * nbytes / (ms / 1e3) / 1e9);
  };
  timeit("ce contiguous", bytes, [&] { CK(cudaMemcpyPeerAsync(dst, 0, src, 1, bytes)); });
  for (int ctas : {148 * 2, 148 * 4, 148 * 8})
    timeit(ctas == 296 ? "ld16 contiguous 2/SM" : ctas == 592 ? "ld16 contiguous 4/SM"
                                                              : "ld16 contiguous 8/SM",
           bytes, [&] {
             ld16_kernel<<<ctas, 256>>>((const float4*)src, (float4*)dst, bytes / 16);
           });
  // bulk: contiguous 16 KB chunks, and runs of R 400-B rows at random offsets
  const int64_t nrow_total = bytes / 400;
  for (int R : {0, 1, 6, 32}) {
    std::vector<int64_t> off;
    std::vector<int32_t> len;
    double tot = 0;
    if (R == 0) {
      for (int64_t o = 0; o + 16384 <= bytes; o += 16384) {
        off.push_back(o);
        len.push_back(16384);
      }
      tot = (double)off.size() * 16384;
    } else {
      srand(7);
      const int64_t nruns = nrow_total / R / 2;
      for (int64_t i = 0; i < nruns; ++i) {
        const int64_t r = ((int64_t)rand() * 32768 + rand()) % (nrow_total - R);
        off.push_back(r * 400);
        len.push_back(R * 400);
        tot += R * 400.0;
      }
    }
    int64_t* d_off;
    int32_t* d_len;
    CK(cudaMalloc(&d_off, off.size() * 8));
    CK(cudaMalloc(&d_len, len.size() * 4));
    CK(cudaMemcpy(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_len, len.data(), len.size() * 4, cudaMemcpyHostToDevice));
    const int slot_bytes = R == 0 ? 16384 : ((R * 400 + 127) / 128) * 128;
    const int smem = kSlots * slot_bytes;
    CK(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int per_sm : {2, 8}) {
      char name[64];
      snprintf(name, sizeof name, "bulk %s%d x%d/SM", R == 0 ? "16KB" : "runs R=", R, per_sm);
      timeit(name, tot, [&] {
        bulk_kernel<<<148 * per_sm, 32, smem>>>(src, dst, d_off, d_len, (int64_t)off.size(),
                                                slot_bytes);
      });
    }
    if (R == 1) {
      std::vector<int64_t> rows(off.size());
      for (size_t i = 0; i < off.size(); ++i) rows[i] = off[i] / 400;
      int64_t* d_rows;
      CK(cudaMalloc(&d_rows, rows.size() * 8));
      CK(cudaMemcpy(d_rows, rows.data(), rows.size() * 8, cudaMemcpyHostToDevice));
      timeit("rows16 random 400-B rows", tot, [&] {
        rows16_kernel<<<148 * 6, 256>>>((const float4*)src, (float4*)dst, d_rows,
                                        (int64_t)rows.size());
      });
      CK(cudaFree(d_rows));
    }
    CK(cudaFree(d_off));
    CK(cudaFree(d_len));
  }
  return 0;
}
