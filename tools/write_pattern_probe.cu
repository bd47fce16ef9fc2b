// Write-pattern probe for the bundle gather's store stream (no reads):
// G interleaved output regions, each CTA claims a "window" w and writes, for
// every region b, a contiguous run of R bytes at b * region + w * R (the
// staged union gather's pattern: one run per batch per id window), versus one
// sequential stream.  Prints TB/s per pattern.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/write_pattern_probe \
//        tools/write_pattern_probe.cu && tools/write_pattern_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// incompressible payload (the bundle rows are random floats; B200's L2 tries
// to compress every written sector, and constant data would compress)
__device__ __forceinline__ float4 noise(int64_t i) {
  uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull;
  x ^= x >> 31;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 29;
  return make_float4(__uint_as_float((uint32_t)x), __uint_as_float((uint32_t)(x >> 32)),
                     __uint_as_float((uint32_t)(x >> 7)), __uint_as_float((uint32_t)(x >> 19)));
}

__global__ void runs_kernel(float4* out, int64_t region_vec, int G, int run_vec, int64_t nwin,
                            unsigned* queue) {
  __shared__ unsigned s_w;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_w = atomicAdd(queue, 1u);
    __syncthreads();
    const int64_t w = s_w;
    if (w >= nwin) break;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = warp; b < G; b += blockDim.x >> 5) {
      float4* dst = out + (int64_t)b * region_vec + w * run_vec;
      for (int e = lane; e < run_vec; e += 32) dst[e] = noise(w * run_vec + e + b);
    }
  }
}

__global__ void seq_kernel(float4* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = noise(i);
}

int main() {
  const int G = 128;
  const int64_t total = 34ll << 30;  // ~ the G = 128 Products bundle bytes
  const int64_t region = total / G / 16 * 16;
  float4* out;
  unsigned* q;
  if (cudaMalloc(&out, G * region) != cudaSuccess || cudaMalloc(&q, 4) != cudaSuccess) return 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    seq_kernel<<<148 * 8, 256>>>(out, G * region / 16);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("{\"pattern\": \"sequential\", \"tbs\": %.3f}\n", G * region / (ms * 1e-3) / 1e12);
  const int runs[] = {1600, 3400, 6800, 13600, 27200, 65536};
  for (int R : runs) {
    const int run_vec = R / 16;
    const int64_t nwin = region / R;
    for (int ctas : {2, 3, 4}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(q, 0, 4);
        cudaEventRecord(a);
        runs_kernel<<<148 * ctas, 256>>>(out, region / 16, G, run_vec, nwin, q);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      printf("{\"pattern\": \"runs\", \"run_bytes\": %d, \"ctas_per_sm\": %d, \"tbs\": %.3f}\n", R,
             ctas, (double)G * nwin * R / (ms * 1e-3) / 1e12);
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
