// The GraphSAGE training step's small fused kernels (the consumer of the
// bundle; model.GraphTrainer).
//
// Reference: gnnpipe/model.py:107-146 (loss_and_grad, sgd_step).  The
// graph-captured step ran the softmax cross-entropy head as ~25 elementwise
// and reduction launches and the SGD update as two launches per tensor; at
// Products shape those tiny kernels were a third of the step's GPU time.
//   rg_softmax_xent: loss and d(loss)/d(logits) of the live seed rows, warp
//     per row, then one CTA sums the rows' losses in a fixed order
//     (deterministic, no atomics);
//   rg_sgd_apply: w -= lr * sum_c g[c] for up to three tensors per launch,
//     the chunk partials of the batched weight-gradient GEMM summed inside
//     the update (eight interleaved in-order sums, combined pairwise: a
//     fixed order, so runs are reproducible).
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

// Warp per row (classes C <= 64, two per lane): the row's nll goes to
// nll[r] (0 for padding rows), the gradient to dz.
constexpr int kXentWarps = 8;

template <typename T>
__global__ void __launch_bounds__(kXentWarps * 32)
    softmax_xent_kernel(const T* __restrict__ logits, int C, int64_t cap,
                        const int32_t* __restrict__ d_n, const int64_t* __restrict__ labels,
                        const int32_t* __restrict__ front0, T* __restrict__ dz,
                        T* __restrict__ nll_out) {
  using O = Ops<T>;
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)kXentWarps + (threadIdx.x >> 5);
  if (r >= cap) return;
  const int64_t n = d_n ? min((int64_t)*d_n, cap) : cap;
  const T* lr = logits + r * C;
  T* dr = dz + r * C;
  if (r >= n) {  // padding rows: no loss, no gradient
    for (int j = lane; j < C; j += 32) dr[j] = 0;
    if (lane == 0) nll_out[r] = 0;
    return;
  }
  const T nt = (T)n;
  const int y = (int)labels[front0[r]];
  const T l0 = lane < C ? lr[lane] : -INFINITY;
  const T l1 = lane + 32 < C ? lr[lane + 32] : -INFINITY;
  const T m = warp_max(max(l0, l1));
  const T s0 = O::sub(l0, m), s1 = O::sub(l1, m);
  const T e0 = lane < C ? O::exp_(s0) : (T)0;
  const T e1 = lane + 32 < C ? O::exp_(s1) : (T)0;
  const T se = __shfl_sync(kFull, warp_sum(O::add(e0, e1)), 0);
  const T sy = __shfl_sync(kFull, y < 32 ? s0 : s1, y & 31);
  if (lane == 0) nll_out[r] = -O::sub(sy, O::log_(se));
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

// loss_acc += (sum of nll in a fixed order) / n: thread t sums rows t,
// t + 1024, ... in order, then the 1024 partials are added pairwise.
template <typename T>
__global__ void __launch_bounds__(kXentThreads)
    xent_loss_kernel(const T* __restrict__ nll, int64_t cap, const int32_t* __restrict__ d_n,
                     double* __restrict__ loss_acc) {
  using O = Ops<T>;
  __shared__ T s_part[kXentThreads];
  const int64_t n = d_n ? min((int64_t)*d_n, cap) : cap;
  T acc = 0;
  for (int64_t r = threadIdx.x; r < cap; r += kXentThreads) acc = O::add(acc, nll[r]);
  s_part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kXentThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      s_part[threadIdx.x] = O::add(s_part[threadIdx.x], s_part[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0 && n > 0) *loss_acc += (double)O::div(s_part[0], (T)n);
}

struct SgdArgs {
  void* w[3];
  const void* g[3];
  int64_t n[3];
  int32_t chunks[3];
  int64_t chunk_stride[3];
};

// CTA = 32 elements of one tensor x 8 warps; warp w sums the partials
// c = w, w + 8, ... in order (lane = element), then the eight warp sums are
// combined as ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)) and the
// element updated.  Blocks [0, b0) cover tensor 0, then tensor 1, ...
constexpr int kSgdWarps = 8;

template <typename T>
__global__ void __launch_bounds__(kSgdWarps * 32)
    sgd_apply_kernel(const __grid_constant__ SgdArgs a, int nt, T lr) {
  using O = Ops<T>;
  __shared__ T s_part[kSgdWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t blk = blockIdx.x;
  int t = 0;
  for (; t < nt; ++t) {
    const int64_t nb = (a.n[t] + 31) / 32;
    if (blk < nb) break;
    blk -= nb;
  }
  if (t >= nt) return;
  const int64_t i = blk * 32 + lane;
  const bool ok = i < a.n[t];
  const T* g = static_cast<const T*>(a.g[t]);
  T s = 0;
  if (ok) {
    const int chunks = a.chunks[t];
    const int64_t cs = a.chunk_stride[t];
    if (warp < chunks) s = g[warp * cs + i];
    for (int c = warp + kSgdWarps; c < chunks; c += kSgdWarps) s = O::add(s, g[c * cs + i]);
  }
  s_part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && ok) {
    const T a01 = O::add(s_part[0][lane], s_part[1][lane]);
    const T a23 = O::add(s_part[2][lane], s_part[3][lane]);
    const T a45 = O::add(s_part[4][lane], s_part[5][lane]);
    const T a67 = O::add(s_part[6][lane], s_part[7][lane]);
    const T sum = O::add(O::add(a01, a23), O::add(a45, a67));
    T* w = static_cast<T*>(a.w[t]);
    w[i] = O::sub(w[i], O::mul(lr, sum));
  }
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_softmax_xent(int32_t dtype, const void* d_logits, int32_t C, int64_t cap,
                               const int32_t* d_n, const int64_t* d_labels,
                               const int32_t* d_front0, void* d_dz, void* d_nll,
                               double* d_loss_acc, void* stream) {
  RG_REQUIRE(dtype == RG_DTYPE_F32 || dtype == RG_DTYPE_F64, "rg_softmax_xent: dtype %d", dtype);
  RG_REQUIRE(C >= 1 && C <= 64 && cap >= 1, "rg_softmax_xent: C=%d (1..64) cap=%lld", C,
             (long long)cap);
  RG_REQUIRE((cap + kXentWarps - 1) / kXentWarps < (1ll << 31), "rg_softmax_xent: cap too large");
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned blocks = (unsigned)((cap + kXentWarps - 1) / kXentWarps);
  if (dtype == RG_DTYPE_F32) {
    softmax_xent_kernel<float><<<blocks, kXentWarps * 32, 0, s>>>(
        static_cast<const float*>(d_logits), C, cap, d_n, d_labels, d_front0,
        static_cast<float*>(d_dz), static_cast<float*>(d_nll));
    if (int rc = check_launch("softmax_xent")) return rc;
    xent_loss_kernel<float><<<1, kXentThreads, 0, s>>>(static_cast<const float*>(d_nll), cap,
                                                        d_n, d_loss_acc);
  } else {
    softmax_xent_kernel<double><<<blocks, kXentWarps * 32, 0, s>>>(
        static_cast<const double*>(d_logits), C, cap, d_n, d_labels, d_front0,
        static_cast<double*>(d_dz), static_cast<double*>(d_nll));
    if (int rc = check_launch("softmax_xent")) return rc;
    xent_loss_kernel<double><<<1, kXentThreads, 0, s>>>(static_cast<const double*>(d_nll), cap,
                                                         d_n, d_loss_acc);
  }
  return check_launch("xent_loss");
}

extern "C" int rg_sgd_apply(int32_t dtype, int32_t n_tensors, void* const* h_w,
                            const void* const* h_g, const int64_t* h_n, const int32_t* h_chunks,
                            double lr, void* stream) {
  RG_REQUIRE(dtype == RG_DTYPE_F32 || dtype == RG_DTYPE_F64, "rg_sgd_apply: dtype %d", dtype);
  RG_REQUIRE(n_tensors >= 1 && n_tensors <= 3, "rg_sgd_apply: 1..3 tensors, got %d", n_tensors);
  SgdArgs a{};
  for (int t = 0; t < n_tensors; ++t) {
    RG_REQUIRE(h_n[t] >= 0 && h_chunks[t] >= 1, "rg_sgd_apply: bad size / chunks");
    a.w[t] = h_w[t];
    a.g[t] = h_g[t];
    a.n[t] = h_n[t];
    a.chunks[t] = h_chunks[t];
    a.chunk_stride[t] = h_n[t];  // partials [chunks, n] contiguous
  }
  int64_t blocks = 0;
  for (int t = 0; t < n_tensors; ++t) blocks += (h_n[t] + 31) / 32;
  RG_REQUIRE(blocks < (1ll << 31), "rg_sgd_apply: tensors too large");
  if (blocks == 0) return RG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == RG_DTYPE_F32)
    sgd_apply_kernel<float><<<(unsigned)blocks, kSgdWarps * 32, 0, s>>>(a, n_tensors, (float)lr);
  else
    sgd_apply_kernel<double><<<(unsigned)blocks, kSgdWarps * 32, 0, s>>>(a, n_tensors, lr);
  return check_launch("sgd_apply");
}
