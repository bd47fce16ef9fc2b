// The GraphSAGE training step's small fused kernels (the consumer of the
// bundle; model.GraphTrainer).
//
// Reference: gnnpipe/model.py:107-146 (loss_and_grad, sgd_step).  The
// graph-captured step ran the softmax cross-entropy head as ~25 elementwise
// and reduction launches and the SGD update as two launches per tensor; at
// Products shape those tiny kernels were a third of the step's GPU time.
//   rg_softmax_xent: loss and d(loss)/d(logits) of the live seed rows in one
//     CTA (deterministic: fixed-order sums, no atomics);
//   rg_sgd_apply: w -= lr * sum_c g[c] for up to three tensors per launch,
//     the chunk partials of the batched weight-gradient GEMM summed in chunk
//     order inside the update.
// Rounding follows the reference's expression order (lr * g rounded, then
// subtracted; no contraction into FMA).
#include <cmath>

#include "rg_common.cuh"

namespace rg {
namespace {

constexpr int kXentThreads = 1024;

template <typename T>
struct Ops;
template <>
struct Ops<float> {
  __device__ static float exp_(float x) { return expf(x); }
  __device__ static float log_(float x) { return logf(x); }
  __device__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ static float div(float a, float b) { return __fdiv_rn(a, b); }
};
template <>
struct Ops<double> {
  __device__ static double exp_(double x) { return exp(x); }
  __device__ static double log_(double x) { return log(x); }
  __device__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ static double div(double a, double b) { return __ddiv_rn(a, b); }
};

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// fixed-order warp sum: lane 0 ends with ((x0 + x1) + (x2 + x3)) + ...
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v = Ops<T>::add(v, __shfl_down_sync(kFull, v, o));
  return v;
}

// One CTA; warp w handles rows w, w + 32, ...; classes C <= 64 (two per lane).
template <typename T>
__global__ void __launch_bounds__(kXentThreads)
    softmax_xent_kernel(const T* __restrict__ logits, int C, int64_t cap,
                        const int32_t* __restrict__ d_n, const int64_t* __restrict__ labels,
                        const int32_t* __restrict__ front0, T* __restrict__ dz,
                        double* __restrict__ loss_acc) {
  using O = Ops<T>;
  __shared__ T s_part[kXentThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = d_n ? min((int64_t)*d_n, cap) : cap;
  const T nt = (T)n;
  T acc = 0;  // this warp's rows, in row order (lane 0)
  for (int64_t r = warp; r < cap; r += kXentThreads / 32) {
    const T* lr = logits + r * C;
    T* dr = dz + r * C;
    if (r >= n) {  // padding rows: no loss, no gradient
      for (int j = lane; j < C; j += 32) dr[j] = 0;
      continue;
    }
    const int y = (int)labels[front0[r]];
    const T l0 = lane < C ? lr[lane] : -INFINITY;
    const T l1 = lane + 32 < C ? lr[lane + 32] : -INFINITY;
    const T m = warp_max(max(l0, l1));
    const T s0 = O::sub(l0, m), s1 = O::sub(l1, m);
    const T e0 = lane < C ? O::exp_(s0) : (T)0;
    const T e1 = lane + 32 < C ? O::exp_(s1) : (T)0;
    const T se = __shfl_sync(kFull, warp_sum(O::add(e0, e1)), 0);
    const T sy = __shfl_sync(kFull, y < 32 ? s0 : s1, y & 31);
    const T nll = -O::sub(sy, O::log_(se));
    if (lane == 0) acc = O::add(acc, nll);
    if (lane < C) {
      T g = O::div(e0, se);
      if (lane == y) g = O::sub(g, (T)1);
      dr[lane] = O::div(g, nt);
    }
    if (lane + 32 < C) {
      T g = O::div(e1, se);
      if (lane + 32 == y) g = O::sub(g, (T)1);
      dr[lane + 32] = O::div(g, nt);
    }
  }
  if (lane == 0) s_part[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    T tot = 0;
    for (int w = 0; w < kXentThreads / 32; ++w) tot = O::add(tot, s_part[w]);
    if (n > 0) *loss_acc += (double)O::div(tot, nt);
  }
}

struct SgdArgs {
  void* w[3];
  const void* g[3];
  int64_t n[3];
  int32_t chunks[3];
  int64_t chunk_stride[3];
};

template <typename T>
__global__ void sgd_apply_kernel(const __grid_constant__ SgdArgs a, int nt, T lr) {
  using O = Ops<T>;
  for (int t = 0; t < nt; ++t) {
    T* w = static_cast<T*>(a.w[t]);
    const T* g = static_cast<const T*>(a.g[t]);
    const int64_t n = a.n[t];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      T s = g[i];
      for (int c = 1; c < a.chunks[t]; ++c) s = O::add(s, g[c * a.chunk_stride[t] + i]);
      w[i] = O::sub(w[i], O::mul(lr, s));
    }
  }
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_softmax_xent(int32_t dtype, const void* d_logits, int32_t C, int64_t cap,
                               const int32_t* d_n, const int64_t* d_labels,
                               const int32_t* d_front0, void* d_dz, double* d_loss_acc,
                               void* stream) {
  RG_REQUIRE(dtype == RG_DTYPE_F32 || dtype == RG_DTYPE_F64, "rg_softmax_xent: dtype %d", dtype);
  RG_REQUIRE(C >= 1 && C <= 64 && cap >= 0, "rg_softmax_xent: C=%d (1..64) cap=%lld", C,
             (long long)cap);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == RG_DTYPE_F32)
    softmax_xent_kernel<float><<<1, kXentThreads, 0, s>>>(
        static_cast<const float*>(d_logits), C, cap, d_n, d_labels, d_front0,
        static_cast<float*>(d_dz), d_loss_acc);
  else
    softmax_xent_kernel<double><<<1, kXentThreads, 0, s>>>(
        static_cast<const double*>(d_logits), C, cap, d_n, d_labels, d_front0,
        static_cast<double*>(d_dz), d_loss_acc);
  return check_launch("softmax_xent");
}

extern "C" int rg_sgd_apply(int32_t dtype, int32_t n_tensors, void* const* h_w,
                            const void* const* h_g, const int64_t* h_n, const int32_t* h_chunks,
                            double lr, void* stream) {
  RG_REQUIRE(dtype == RG_DTYPE_F32 || dtype == RG_DTYPE_F64, "rg_sgd_apply: dtype %d", dtype);
  RG_REQUIRE(n_tensors >= 1 && n_tensors <= 3, "rg_sgd_apply: 1..3 tensors, got %d", n_tensors);
  SgdArgs a{};
  int64_t most = 1;
  for (int t = 0; t < n_tensors; ++t) {
    RG_REQUIRE(h_n[t] >= 0 && h_chunks[t] >= 1, "rg_sgd_apply: bad size / chunks");
    a.w[t] = h_w[t];
    a.g[t] = h_g[t];
    a.n[t] = h_n[t];
    a.chunks[t] = h_chunks[t];
    a.chunk_stride[t] = h_n[t];  // partials [chunks, n] contiguous
    most = std::max(most, h_n[t]);
  }
  const int blocks = (int)std::min<int64_t>((most + 255) / 256, kNumSMs * 4);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == RG_DTYPE_F32)
    sgd_apply_kernel<float><<<blocks, 256, 0, s>>>(a, n_tensors, (float)lr);
  else
    sgd_apply_kernel<double><<<blocks, 256, 0, s>>>(a, n_tensors, lr);
  return check_launch("sgd_apply");
}
