// K8: GraphSAGE mean aggregation over a sampled block, forward and backward.
//
// Reference: gnnpipe/model.py:72-81 (_forward_pass) and model.py:126-135
// (loss_and_grad backward scatter).  The reference sums neighbour rows with
// np.add.at in edge order (dst asc, src asc), divides by max(count, 1) in
// the parameter dtype, and in the backward adds dself at the self positions
// first and then (dmean / denom)[dst] into dh[src] in the same edge order.
// Both kernels reproduce those orders exactly (one sequential chain per
// output element, parallel over columns), so results are bit-identical to
// the reference for identical inputs in fp32 and fp64 (RunConfig.precision,
// train.py:117); only the dense GEMMs around them (cuBLAS) differ in rounding.
//
// Positions (model.py:53-55, 74-75: searchsorted of src / dst into the
// sorted src frontier) are resolved ONCE per level by rg_sage_positions —
// a scatter of frontier ranks into an n-node rank table, then one load per
// edge — and shared by the forward and the backward.  The backward's
// transposed index (edges grouped by src, ascending dst inside a group =
// the reference's edge order for that src) is a stable radix sort of the
// edges by src position, so any in-sample in-degree is handled exactly.
#include <climits>

#include <cub/device/device_radix_sort.cuh>

#include "rg_common.cuh"

namespace rg {
namespace {

constexpr int kWarps = 8;

// live count: the device word when given (a sampler slot's nfront entry, so
// the call needs no host sync and can be captured in a CUDA graph; the host
// size is then the capacity), else the host size itself
__device__ __forceinline__ int64_t live_count(const int32_t* d_n, int64_t cap) {
  return d_n ? min((int64_t)__ldg(d_n), cap) : cap;
}

// ---------------------------------------------------------------- positions
__global__ void rank_scatter_kernel(const int32_t* __restrict__ front, int64_t cap,
                                    const int32_t* __restrict__ d_n, int32_t* __restrict__ rank) {
  const int64_t n = live_count(d_n, cap);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    rank[front[j]] = (int32_t)j;
}

// epos[t*F + r] = rank of ell[t*F + r] (r < cnt[t]), -1 past the row's count;
// self_pos[t] = rank of dst_front[t] (frontiers are nested: dst ⊂ src)
// rows past the live count (capacity padding) get no edges and self row 0
__global__ void edge_pos_kernel(const int32_t* __restrict__ rank,
                                const int32_t* __restrict__ dst_front, int64_t cap_dst,
                                const int32_t* __restrict__ d_ndst,
                                const int32_t* __restrict__ ell, const int32_t* __restrict__ cnt,
                                int F, int32_t* __restrict__ epos,
                                int32_t* __restrict__ self_pos) {
  const int64_t n_dst = live_count(d_ndst, cap_dst);
  const int64_t total = cap_dst * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / F;
    const int r = (int)(i - t * F);
    const bool live = t < n_dst;
    epos[i] = live && r < __ldg(cnt + t) ? __ldg(rank + __ldg(ell + i)) : -1;
    if (r == 0) self_pos[t] = live ? __ldg(rank + __ldg(dst_front + t)) : 0;
  }
}

// ---------------------------------------------------------------- row tiles
// N elements of T moved as one aligned load (16 B for float4 / double2)
template <typename T, int N>
struct alignas(sizeof(T) * N) Vec {
  T v[N];
};

// A group of SW lanes owns one output row; lane j of the group handles the
// row's vectors j, j + SW, ... (up to V per pass over the columns; V is
// chosen per launch as ceil(nvec / SW), so registers match the row width).
template <typename T, int N, int V>
__device__ __forceinline__ void load_vecs(const T* __restrict__ row, int nvec, int j0, int SW,
                                          Vec<T, N> (&x)[V]) {
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const int vi = j0 + u * SW;
    if (vi < nvec) x[u] = *reinterpret_cast<const Vec<T, N>*>(row + (int64_t)vi * N);
  }
}

// mean[t] = (((0 + h[p_1]) + h[p_2]) + ...) / max(cnt_t, 1); self[t] = h[self_pos[t]]
template <typename T, int N, int V>
__global__ void __launch_bounds__(kWarps * 32)
    sage_fwd_kernel(const T* __restrict__ h, int ldh, int H, const int32_t* __restrict__ epos,
                    const int32_t* __restrict__ self_pos, int64_t cap_dst,
                    const int32_t* __restrict__ d_ndst, const int32_t* __restrict__ cnt, int F,
                    int SW, T* __restrict__ mean, T* __restrict__ self) {
  const int64_t n_live = live_count(d_ndst, cap_dst);
  const int lane = lane_id();
  const int rpw = 32 / SW;  // rows per warp
  const int grp = lane / SW, j0 = lane % SW;
  const int nvec = H / N;
  const int64_t nrow_step = (int64_t)gridDim.x * kWarps * rpw;
  for (int64_t t = ((int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5)) * rpw + grp; t < cap_dst;
       t += nrow_step) {
    const bool live = t < n_live;  // padding rows: mean = self = 0
    const int c = live ? __ldg(cnt + t) : 0;
    const T denom = (T)max(c, 1);
    const int32_t* ep = epos + t * F;
    const int ps = __ldg(self_pos + t);
    for (int vb = 0; vb < nvec; vb += SW * V) {
      const int jb = vb + j0;
      Vec<T, N> acc[V];
#pragma unroll
      for (int u = 0; u < V; ++u)
#pragma unroll
        for (int k = 0; k < N; ++k) acc[u].v[k] = (T)0;
      constexpr int R = V == 1 ? 4 : 2;  // rows' loads in flight; adds stay in edge order
      int r = 0;
      for (; r + R <= c; r += R) {
        Vec<T, N> x[R][V];
#pragma unroll
        for (int q = 0; q < R; ++q)
          load_vecs<T, N, V>(h + (int64_t)__ldg(ep + r + q) * ldh, nvec, jb, SW, x[q]);
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
          for (int u = 0; u < V; ++u)
#pragma unroll
            for (int k = 0; k < N; ++k) acc[u].v[k] += x[q][u].v[k];
      }
      for (; r < c; ++r) {
        Vec<T, N> x0[V];
        load_vecs<T, N, V>(h + (int64_t)__ldg(ep + r) * ldh, nvec, jb, SW, x0);
#pragma unroll
        for (int u = 0; u < V; ++u)
#pragma unroll
          for (int k = 0; k < N; ++k) acc[u].v[k] += x0[u].v[k];
      }
      Vec<T, N> sv[V];
#pragma unroll
      for (int u = 0; u < V; ++u)
#pragma unroll
        for (int k = 0; k < N; ++k) sv[u].v[k] = (T)0;
      if (self && live) load_vecs<T, N, V>(h + (int64_t)ps * ldh, nvec, jb, SW, sv);
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int vi = jb + u * SW;
        if (vi < nvec) {
#pragma unroll
          for (int k = 0; k < N; ++k) acc[u].v[k] = acc[u].v[k] / denom;
          *reinterpret_cast<Vec<T, N>*>(mean + t * H + (int64_t)vi * N) = acc[u];
          if (self) *reinterpret_cast<Vec<T, N>*>(self + t * H + (int64_t)vi * N) = sv[u];
        }
      }
    }
  }
}

// ---------------------------------------------------------------- transpose
// toff[s] = first sorted index with key >= s (keys ascending, holes keyed
// n_src), s = 0..n_src: a binary search per s.  (Filling each key gap from
// the key that ends it put the whole gap between the last live row and the
// capacity on one thread: 27 us at Products layer 1.)
__global__ void segment_bounds_kernel(const int32_t* __restrict__ keys, int64_t nkeys,
                                      int64_t n_src, int32_t* __restrict__ toff) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= n_src;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nkeys;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)__ldg(keys + mid) < s)
        lo = mid + 1;
      else
        hi = mid;
    }
    toff[s] = (int32_t)lo;
  }
}

// radix-sort input: key = src position (holes -> n_src, sorted last),
// value = dst row; input order is the reference's edge order (t asc, r asc)
__global__ void transpose_keys_kernel(const int32_t* __restrict__ epos, int64_t total, int F,
                                      int32_t n_src, int32_t* __restrict__ keys,
                                      int32_t* __restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = epos[i];
    keys[i] = p >= 0 ? p : n_src;
    vals[i] = (int32_t)(i / F);
  }
}

__global__ void self_of_kernel(const int32_t* __restrict__ self_pos, int64_t cap_dst,
                               const int32_t* __restrict__ d_ndst,
                               int32_t* __restrict__ self_of) {
  const int64_t n_dst = live_count(d_ndst, cap_dst);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_dst;
       t += (int64_t)gridDim.x * blockDim.x)
    self_of[self_pos[t]] = (int32_t)t;
}

// dh[s] = ((0 + dself[self_of[s]]) + dmean[t_1]/denom_1) + dmean[t_2]/denom_2 ...
template <typename T, int N, int V>
__global__ void __launch_bounds__(kWarps * 32)
    sage_bwd_kernel(const T* __restrict__ dself, const T* __restrict__ dmean, int H,
                    const int32_t* __restrict__ cnt, const int32_t* __restrict__ self_of,
                    const int32_t* __restrict__ toff, const int32_t* __restrict__ tdst,
                    int64_t cap_src, const int32_t* __restrict__ d_nsrc, int SW,
                    T* __restrict__ dh) {
  const int64_t n_live = live_count(d_nsrc, cap_src);
  const int lane = lane_id();
  const int rpw = 32 / SW;
  const int grp = lane / SW, j0 = lane % SW;
  const int nvec = H / N;
  const int64_t nrow_step = (int64_t)gridDim.x * kWarps * rpw;
  for (int64_t s = ((int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5)) * rpw + grp; s < cap_src;
       s += nrow_step) {
    const bool live = s < n_live;  // padding rows: dh = 0
    const int a = live ? __ldg(toff + s) : 0, len = live ? __ldg(toff + s + 1) - a : 0;
    const int so = live ? __ldg(self_of + s) : -1;
    for (int vb = 0; vb < nvec; vb += SW * V) {
      const int jb = vb + j0;
      Vec<T, N> acc[V];
#pragma unroll
      for (int u = 0; u < V; ++u)
#pragma unroll
        for (int k = 0; k < N; ++k) acc[u].v[k] = (T)0;
      if (so >= 0) {
        Vec<T, N> x[V];
        load_vecs<T, N, V>(dself + (int64_t)so * H, nvec, jb, SW, x);
#pragma unroll
        for (int u = 0; u < V; ++u)
#pragma unroll
          for (int k = 0; k < N; ++k) acc[u].v[k] += x[u].v[k];
      }
      // long segments (hub srcs with thousands of in-sample edges) are one
      // sequential chain per column: keep R rows' loads in flight
      constexpr int R = V == 1 ? 8 : 2;
      int q = 0;
      for (; q + R <= len; q += R) {
        int t[R];
        T dn[R];
        Vec<T, N> x[R][V];
#pragma unroll
        for (int i = 0; i < R; ++i) t[i] = __ldg(tdst + a + q + i);
#pragma unroll
        for (int i = 0; i < R; ++i) {
          dn[i] = (T)max(__ldg(cnt + t[i]), 1);
          load_vecs<T, N, V>(dmean + (int64_t)t[i] * H, nvec, jb, SW, x[i]);
        }
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
          for (int u = 0; u < V; ++u)
#pragma unroll
            for (int k = 0; k < N; ++k) acc[u].v[k] += x[i][u].v[k] / dn[i];
      }
      for (; q < len; ++q) {
        const int t0 = __ldg(tdst + a + q);
        const T d0 = (T)max(__ldg(cnt + t0), 1);
        Vec<T, N> x0[V];
        load_vecs<T, N, V>(dmean + (int64_t)t0 * H, nvec, jb, SW, x0);
#pragma unroll
        for (int u = 0; u < V; ++u)
#pragma unroll
          for (int k = 0; k < N; ++k) acc[u].v[k] += x0[u].v[k] / d0;
      }
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int vi = jb + u * SW;
        if (vi < nvec) *reinterpret_cast<Vec<T, N>*>(dh + s * H + (int64_t)vi * N) = acc[u];
      }
    }
  }
}

// widest vector (<= 16 B) that divides H and the row pitch and keeps the
// base pointers aligned
template <typename T>
int vec_width(int H, int64_t pitch, std::initializer_list<const void*> ptrs) {
  for (int n = 16 / (int)sizeof(T); n > 1; n >>= 1) {
    bool ok = H % n == 0 && pitch % n == 0;
    for (const void* p : ptrs)
      if (p && (reinterpret_cast<uintptr_t>(p) % (n * sizeof(T))) != 0) ok = false;
    if (ok) return n;
  }
  return 1;
}

int sub_warp(int nvec) {
  int sw = 1;
  while (sw < 32 && sw < nvec) sw <<= 1;
  return sw;
}

template <typename T, int N>
int launch_fwd(const void* h, int ldh, int H, const int32_t* epos, const int32_t* self_pos,
               int64_t n_dst, const int32_t* d_ndst, const int32_t* cnt, int F, void* mean,
               void* self, cudaStream_t s) {
  const int SW = sub_warp(H / N);
  const int vpl = (H / N + SW - 1) / SW;
  const int64_t rows_per_cta = (int64_t)kWarps * (32 / SW);
  const int grid = (int)std::min<int64_t>((n_dst + rows_per_cta - 1) / rows_per_cta, kNumSMs * 16);
  auto go = [&](auto kern) {
    kern<<<grid, kWarps * 32, 0, s>>>((const T*)h, ldh, H, epos, self_pos, n_dst, d_ndst, cnt, F,
                                      SW, (T*)mean, (T*)self);
    return check_launch("sage_fwd");
  };
  if (vpl <= 1) return go(sage_fwd_kernel<T, N, 1>);
  if (vpl <= 2) return go(sage_fwd_kernel<T, N, 2>);
  return go(sage_fwd_kernel<T, N, 4>);
}

template <typename T, int N>
int launch_bwd(const void* dself, const void* dmean, int H, const int32_t* cnt,
               const int32_t* self_of, const int32_t* toff, const int32_t* tdst, int64_t n_src,
               const int32_t* d_nsrc, void* dh, cudaStream_t s) {
  const int SW = sub_warp(H / N);
  const int vpl = (H / N + SW - 1) / SW;
  const int64_t rows_per_cta = (int64_t)kWarps * (32 / SW);
  const int grid = (int)std::min<int64_t>((n_src + rows_per_cta - 1) / rows_per_cta, kNumSMs * 16);
  auto go = [&](auto kern) {
    kern<<<grid, kWarps * 32, 0, s>>>((const T*)dself, (const T*)dmean, H, cnt, self_of, toff,
                                      tdst, n_src, d_nsrc, SW, (T*)dh);
    return check_launch("sage_bwd");
  };
  if (vpl <= 1) return go(sage_bwd_kernel<T, N, 1>);
  if (vpl <= 2) return go(sage_bwd_kernel<T, N, 2>);
  return go(sage_bwd_kernel<T, N, 4>);
}

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

size_t cub_temp_bytes(int64_t nitems, int end_bit) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)nitems, 0,
                                  end_bit);
  return bytes;
}

int key_bits(int64_t n_src) {
  int b = 1;
  while (b < 31 && (int64_t(1) << b) <= n_src) ++b;
  return b;
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_sage_positions(const int32_t* d_src_front, int64_t n_src,
                                 const int32_t* d_dst_front, int64_t n_dst, const int32_t* d_ell,
                                 const int32_t* d_cnt, int32_t fanout, int64_t n_nodes,
                                 const int32_t* d_n_src, const int32_t* d_n_dst, int32_t* d_rank,
                                 int32_t* d_epos, int32_t* d_self_pos, void* stream) {
  RG_REQUIRE(n_src >= 1 && n_src <= INT32_MAX && n_dst >= 0 && fanout >= 1 && n_nodes >= n_src,
             "rg_sage_positions: bad sizes");
  RG_REQUIRE(n_dst * (int64_t)fanout < INT32_MAX, "rg_sage_positions: n_dst * fanout overflows");
  if (n_dst == 0) return RG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  rank_scatter_kernel<<<(unsigned)std::min<int64_t>((n_src + 255) / 256, kNumSMs * 8), 256, 0, s>>>(
      d_src_front, n_src, d_n_src, d_rank);
  int rc = check_launch("rank_scatter");
  if (rc) return rc;
  const int64_t total = n_dst * fanout;
  edge_pos_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, kNumSMs * 8), 256, 0, s>>>(
      d_rank, d_dst_front, n_dst, d_n_dst, d_ell, d_cnt, fanout, d_epos, d_self_pos);
  return check_launch("edge_pos");
}

extern "C" int rg_sage_mean_fwd(int32_t dtype, const void* d_h, int32_t H, int32_t ldh,
                                const int32_t* d_epos, const int32_t* d_self_pos, int64_t n_dst,
                                const int32_t* d_n_dst, const int32_t* d_cnt, int32_t fanout,
                                void* d_mean, void* d_self, void* stream) {
  RG_REQUIRE(H >= 1 && ldh >= H && n_dst >= 0 && fanout >= 1, "rg_sage_mean_fwd: bad sizes");
  RG_REQUIRE(dtype == RG_DTYPE_F32 || dtype == RG_DTYPE_F64, "rg_sage_mean_fwd: bad dtype");
  if (n_dst == 0) return RG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == RG_DTYPE_F32) {
    switch (vec_width<float>(H, ldh, {d_h, d_mean, d_self})) {
      case 4: return launch_fwd<float, 4>(d_h, ldh, H, d_epos, d_self_pos, n_dst, d_n_dst, d_cnt, fanout, d_mean, d_self, s);
      case 2: return launch_fwd<float, 2>(d_h, ldh, H, d_epos, d_self_pos, n_dst, d_n_dst, d_cnt, fanout, d_mean, d_self, s);
      default: return launch_fwd<float, 1>(d_h, ldh, H, d_epos, d_self_pos, n_dst, d_n_dst, d_cnt, fanout, d_mean, d_self, s);
    }
  }
  if (vec_width<double>(H, ldh, {d_h, d_mean, d_self}) == 2)
    return launch_fwd<double, 2>(d_h, ldh, H, d_epos, d_self_pos, n_dst, d_n_dst, d_cnt, fanout, d_mean, d_self, s);
  return launch_fwd<double, 1>(d_h, ldh, H, d_epos, d_self_pos, n_dst, d_n_dst, d_cnt, fanout, d_mean, d_self, s);
}

extern "C" int64_t rg_sage_transpose_scratch(int64_t n_src, int64_t n_dst, int32_t fanout) {
  const int64_t total = n_dst * fanout;
  if (n_src < 1 || total < 0 || total >= INT32_MAX) return -1;
  return (int64_t)(3 * align_up(sizeof(int32_t) * std::max<int64_t>(total, 1)) +
                   align_up(cub_temp_bytes(total, key_bits(n_src))));
}

extern "C" int rg_sage_transpose(const int32_t* d_epos, const int32_t* d_cnt, int64_t n_dst,
                                 int32_t fanout, int64_t n_src, int32_t* d_toff, int32_t* d_tdst,
                                 void* d_scratch, int64_t scratch_bytes, void* stream) {
  (void)d_cnt;
  RG_REQUIRE(n_src >= 1 && n_src < INT32_MAX && n_dst >= 0 && fanout >= 1,
             "rg_sage_transpose: bad sizes");
  const int64_t need = rg_sage_transpose_scratch(n_src, n_dst, fanout);
  RG_REQUIRE(need >= 0 && scratch_bytes >= need, "rg_sage_transpose: scratch %lld < %lld bytes",
             (long long)scratch_bytes, (long long)need);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t total = n_dst * fanout;
  char* base = (char*)d_scratch;
  const size_t arr = align_up(sizeof(int32_t) * std::max<int64_t>(total, 1));
  int32_t* keys_in = (int32_t*)base;
  int32_t* vals_in = (int32_t*)(base + arr);
  int32_t* keys_out = (int32_t*)(base + 2 * arr);
  void* temp = base + 3 * arr;
  int rc;
  if (total > 0) {
    const unsigned g = (unsigned)std::min<int64_t>((total + 255) / 256, kNumSMs * 8);
    transpose_keys_kernel<<<g, 256, 0, s>>>(d_epos, total, fanout, (int32_t)n_src, keys_in,
                                            vals_in);
    if ((rc = check_launch("transpose_keys"))) return rc;
    const int bits = key_bits(n_src);
    size_t temp_bytes = cub_temp_bytes(total, bits);
    // stable LSD radix sort: per src the dst rows keep their edge order
    if (cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, d_tdst,
                                        (int)total, 0, bits, s) != cudaSuccess)
      return check_launch("transpose radix sort");
  }
  const unsigned g = (unsigned)std::min<int64_t>((n_src + 1 + 255) / 256, kNumSMs * 8);
  segment_bounds_kernel<<<g, 256, 0, s>>>(keys_out, total, n_src, d_toff);
  return check_launch("segment_bounds");
}

extern "C" int rg_sage_mean_bwd(int32_t dtype, const void* d_dself, const void* d_dmean,
                                int64_t n_dst, int32_t H, const int32_t* d_cnt,
                                const int32_t* d_self_pos, const int32_t* d_toff,
                                const int32_t* d_tdst, int64_t n_src, const int32_t* d_n_src,
                                const int32_t* d_n_dst, int32_t* d_self_of, void* d_dh,
                                void* stream) {
  RG_REQUIRE(H >= 1 && n_src >= 1 && n_dst >= 0, "rg_sage_mean_bwd: bad sizes");
  RG_REQUIRE(dtype == RG_DTYPE_F32 || dtype == RG_DTYPE_F64, "rg_sage_mean_bwd: bad dtype");
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(d_self_of, 0xff, sizeof(int32_t) * n_src, s) != cudaSuccess)
    return check_launch("bwd memset");
  if (n_dst > 0) {
    self_of_kernel<<<kNumSMs * 2, 256, 0, s>>>(d_self_pos, n_dst, d_n_dst, d_self_of);
    int rc = check_launch("self_of");
    if (rc) return rc;
  }
  if (dtype == RG_DTYPE_F32) {
    switch (vec_width<float>(H, H, {d_dself, d_dmean, d_dh})) {
      case 4: return launch_bwd<float, 4>(d_dself, d_dmean, H, d_cnt, d_self_of, d_toff, d_tdst, n_src, d_n_src, d_dh, s);
      case 2: return launch_bwd<float, 2>(d_dself, d_dmean, H, d_cnt, d_self_of, d_toff, d_tdst, n_src, d_n_src, d_dh, s);
      default: return launch_bwd<float, 1>(d_dself, d_dmean, H, d_cnt, d_self_of, d_toff, d_tdst, n_src, d_n_src, d_dh, s);
    }
  }
  if (vec_width<double>(H, H, {d_dself, d_dmean, d_dh}) == 2)
    return launch_bwd<double, 2>(d_dself, d_dmean, H, d_cnt, d_self_of, d_toff, d_tdst, n_src, d_n_src, d_dh, s);
  return launch_bwd<double, 1>(d_dself, d_dmean, H, d_cnt, d_self_of, d_toff, d_tdst, n_src, d_n_src, d_dh, s);
}
