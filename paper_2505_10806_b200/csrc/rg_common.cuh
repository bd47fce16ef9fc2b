// Shared device helpers for the RapidGNN B200 kernels.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "../../include/rapidgnn_b200.h"

namespace rg {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;  // rng.py:19
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ull;    // rng.py:20
constexpr uint64_t MIX2 = 0x94D049BB133111EBull;    // rng.py:21
constexpr int kNumSMs = 148;
constexpr unsigned kFull = 0xffffffffu;

// SplitMix64 finalizer (rng.py:28-33); a bijection on uint64.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= MIX1;
  x ^= x >> 27;
  x *= MIX2;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// streaming 16-byte global load that does not allocate in L1
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(float4* p, const float4& v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w));
}

// block-wide exclusive scan of one int per thread; returns the exclusive
// prefix, *total receives the block sum.  smem: >= 32 ints.
template <int kThreads>
__device__ __forceinline__ int block_excl_scan(int v, int* smem, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    constexpr int kWarps = kThreads / 32;
    int w = lane < kWarps ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kWarps) smem[lane] = w;  // inclusive warp prefixes
  }
  __syncthreads();
  int warp_base = warp ? smem[warp - 1] : 0;
  *total = smem[kThreads / 32 - 1];
  __syncthreads();
  return warp_base + x - v;
}

// ascending bitonic sort of one (key, val) pair per lane across the warp
template <typename K, typename V>
__device__ __forceinline__ void warp_bitonic_sort(K& key, V& val) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      K ok = __shfl_xor_sync(kFull, key, j);
      V ov = __shfl_xor_sync(kFull, val, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      const bool take = (lower == up) ? (ok < key) : (ok > key);
      if (take) {
        key = ok;
        val = ov;
      }
    }
  }
}

template <typename K>
__device__ __forceinline__ void warp_bitonic_sort_keys(K& key) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      K ok = __shfl_xor_sync(kFull, key, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      const bool take = (lower == up) ? (ok < key) : (ok > key);
      if (take) key = ok;
    }
  }
}

}  // namespace rg

// error plumbing shared by the ABI translation units
namespace rg {
void set_error(const char* fmt, ...);
int check_launch(const char* what);
}  // namespace rg

#define RG_REQUIRE(cond, ...)      \
  do {                             \
    if (!(cond)) {                 \
      ::rg::set_error(__VA_ARGS__); \
      return RG_ERR_INVALID;       \
    }                              \
  } while (0)
