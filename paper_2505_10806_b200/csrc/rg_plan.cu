// K1/K4/K5: epoch shuffle keys, access histogram, hot-set selection.
//
// Reference: gnnpipe/rng.py:28-62 (mix64, stream_keys), plan.py:108-141
// (_count, collect_access, top_hot).
//
// collect_access counts, per node, the batches of the scope whose input set
// holds it, restricted to remote nodes (plan.py:117-130).  The per-batch
// input sets are the level-L sampler bitmaps, so the count is a dense
// bit-plane sum (one word read per 32 nodes per batch) instead of the
// reference's concatenate + np.unique over ~1e9 ids per epoch.  The count
// is the same for every worker; the remote mask is applied when the
// candidates are extracted.
//
// top_hot (plan.py:133-141) = lexsort by (-count, id), first n_hot, sorted
// by id.  Equivalently: with c* the largest count c
// such that #{count >= c} >= n_hot, take every candidate with count > c*
// plus the lowest-id (n_hot - #{count > c*}) candidates with count == c*.
// The device side provides the count histogram and the two threshold
// bitmaps; the host picks c* from the histogram and the ordered tie quota is
// a prefix of the (sorted) compaction of bm_eq.
#include "rg_common.cuh"

namespace rg {
namespace {

__global__ void mix64_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                             int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mix64(in[i]);
}

__global__ void stream_keys_kernel(uint64_t master, int64_t count, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mix64((uint64_t)(i + 1) * GOLDEN + master);
}

// thread per node: counts[v] += sum_b bit(bm_b, v).  A warp covers exactly
// one bitmap word per batch (broadcast load).
__global__ void count_inputs_kernel(const uint32_t* __restrict__ bm, int64_t nwords, int G,
                                    int64_t n, uint32_t* __restrict__ counts) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = v >> 5;
    const int bit = (int)(v & 31);
    uint32_t c = 0;
    for (int b = 0; b < G; ++b) c += (__ldg(bm + (int64_t)b * nwords + w) >> bit) & 1u;
    if (c) counts[v] += c;
  }
}

__global__ void count_histogram_kernel(const uint32_t* __restrict__ counts,
                                       const uint8_t* __restrict__ owner, int my_part, int64_t n,
                                       uint32_t* __restrict__ hist, int max_count,
                                       uint32_t* __restrict__ bm_cand) {
  const int lane = lane_id();
  // grid-stride in whole warps so each warp owns one bitmap word
  const int64_t nwarps_total = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nwords = (n + 31) >> 5;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += nwarps_total) {
    const int64_t v = w * 32 + lane;
    bool cand = false;
    uint32_t c = 0;
    if (v < n) {
      c = counts[v];
      cand = c > 0 && (int)owner[v] != my_part;
    }
    const unsigned m = __ballot_sync(kFull, cand);
    if (lane == 0) bm_cand[w] = m;
    if (cand) atomicAdd(hist + (c < (uint32_t)max_count ? c : (uint32_t)max_count), 1u);
  }
}

__global__ void threshold_split_kernel(const uint32_t* __restrict__ counts,
                                       const uint32_t* __restrict__ bm_cand, int64_t n,
                                       uint32_t c_star, uint32_t* __restrict__ bm_gt,
                                       uint32_t* __restrict__ bm_eq) {
  const int lane = lane_id();
  const int64_t nwarps_total = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nwords = (n + 31) >> 5;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += nwarps_total) {
    const int64_t v = w * 32 + lane;
    const uint32_t cw = bm_cand[w];
    const bool cand = (cw >> lane) & 1u;
    const uint32_t c = (cand && v < n) ? counts[v] : 0u;
    const unsigned gt = __ballot_sync(kFull, cand && c > c_star);
    const unsigned eq = __ballot_sync(kFull, cand && c == c_star);
    if (lane == 0) {
      bm_gt[w] = gt;
      bm_eq[w] = eq;
    }
  }
}

__global__ void gather_counts_kernel(const uint32_t* __restrict__ counts,
                                     const int32_t* __restrict__ ids, const int32_t* __restrict__ n,
                                     int64_t cap, uint32_t* __restrict__ out) {
  const int64_t cnt = (int64_t)*n < cap ? (int64_t)*n : cap;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = counts[ids[i]];
}

// seeds of batches i0 .. i0+G-1 of an epoch permutation plus their batch
// seeds mix64(s0 ^ (e<<32 | i)) (sampler.py:40, 57)
__global__ void fill_seeds_kernel(const int32_t* __restrict__ perm, int64_t n_perm,
                                  int32_t batch_size, int64_t i0, int32_t* __restrict__ seeds,
                                  int32_t* __restrict__ nseeds, int seed_cap, uint64_t s0,
                                  uint64_t epoch, uint64_t* __restrict__ rng) {
  const int b = blockIdx.x;
  const int64_t i = i0 + b;
  const int64_t start = i * batch_size;
  const int64_t left = n_perm - start;
  const int cnt = left <= 0 ? 0 : (int)(left < batch_size ? left : batch_size);
  for (int t = threadIdx.x; t < cnt; t += blockDim.x)
    seeds[(int64_t)b * seed_cap + t] = perm[start + t];
  if (threadIdx.x == 0) {
    nseeds[b] = cnt;
    rng[b] = mix64(s0 ^ ((epoch << 32) | (uint64_t)i));
  }
}

// Synthetic feature rows for graphs too large for the reference's numpy
// generator (config X): value(v, c) = Box-Muller normal of two 24-bit
// uniforms from mix64(seed ^ ((v * d + c + 1) * GOLDEN)).  Row of node ids[i]
// goes to out[i * stride]; padding columns are zero.
__global__ void fill_features_kernel(const int32_t* __restrict__ ids, int64_t n, int d,
                                     int stride, uint64_t seed, float* __restrict__ out) {
  const int64_t total = n * stride;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / stride;
    const int c = (int)(e - i * stride);
    float val = 0.f;
    if (c < d) {
      const uint64_t v = (uint64_t)ids[i];
      const uint64_t h = mix64(seed ^ ((v * (uint64_t)d + (uint64_t)c + 1ull) * GOLDEN));
      const float u1 = ((float)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
      const float u2 = (float)((h >> 16) & 0xFFFFFFull) * (1.0f / 16777216.0f);
      val = sqrtf(-2.0f * __logf(u1)) * __cosf(6.283185307179586f * u2);
    }
    out[e] = val;
  }
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_mix64(const uint64_t* d_in, uint64_t* d_out, int64_t n, void* stream) {
  RG_REQUIRE(n >= 0, "rg_mix64: n < 0");
  if (n == 0) return RG_OK;
  mix64_kernel<<<kNumSMs * 4, 256, 0, (cudaStream_t)stream>>>(d_in, d_out, n);
  return check_launch("mix64");
}

extern "C" int rg_stream_keys(uint64_t master, int64_t count, uint64_t* d_out, void* stream) {
  RG_REQUIRE(count >= 0, "rg_stream_keys: count < 0");
  if (count == 0) return RG_OK;
  stream_keys_kernel<<<kNumSMs * 4, 256, 0, (cudaStream_t)stream>>>(master, count, d_out);
  return check_launch("stream_keys");
}

extern "C" int rg_count_inputs(const uint32_t* d_bm, int64_t nwords, int32_t G, int64_t n,
                               uint32_t* d_counts, void* stream) {
  RG_REQUIRE(G >= 1 && n >= 1 && nwords * 32 >= n, "rg_count_inputs: bad sizes");
  count_inputs_kernel<<<kNumSMs * 8, 256, 0, (cudaStream_t)stream>>>(d_bm, nwords, G, n,
                                                                      d_counts);
  return check_launch("count_inputs");
}

extern "C" int rg_count_histogram(const uint32_t* d_counts, const uint8_t* d_owner,
                                  int32_t my_part, int64_t n, uint32_t* d_hist, int32_t max_count,
                                  uint32_t* d_bm_cand, void* stream) {
  RG_REQUIRE(n >= 1 && max_count >= 1, "rg_count_histogram: bad sizes");
  count_histogram_kernel<<<kNumSMs * 8, 256, 0, (cudaStream_t)stream>>>(
      d_counts, d_owner, my_part, n, d_hist, max_count, d_bm_cand);
  return check_launch("count_histogram");
}

extern "C" int rg_threshold_split(const uint32_t* d_counts, const uint32_t* d_bm_cand, int64_t n,
                                  uint32_t c_star, uint32_t* d_bm_gt, uint32_t* d_bm_eq,
                                  void* stream) {
  RG_REQUIRE(n >= 1, "rg_threshold_split: bad sizes");
  threshold_split_kernel<<<kNumSMs * 8, 256, 0, (cudaStream_t)stream>>>(d_counts, d_bm_cand, n,
                                                                         c_star, d_bm_gt, d_bm_eq);
  return check_launch("threshold_split");
}

extern "C" int rg_gather_counts(const uint32_t* d_counts, const int32_t* d_ids,
                                const int32_t* d_n, int64_t cap, uint32_t* d_out, void* stream) {
  RG_REQUIRE(cap >= 0, "rg_gather_counts: bad cap");
  if (cap == 0) return RG_OK;
  gather_counts_kernel<<<kNumSMs * 2, 256, 0, (cudaStream_t)stream>>>(d_counts, d_ids, d_n, cap,
                                                                       d_out);
  return check_launch("gather_counts");
}

extern "C" int rg_fill_seeds(const int32_t* d_perm, int64_t n_perm, int32_t batch_size, int64_t i0,
                             int32_t G, int32_t* d_seeds, int32_t* d_nseeds, int32_t seed_cap,
                             uint64_t s0, int64_t epoch, uint64_t* d_rng, void* stream) {
  RG_REQUIRE(G >= 1 && batch_size >= 1 && batch_size <= seed_cap && i0 >= 0 && epoch >= 0,
             "rg_fill_seeds: bad sizes");
  fill_seeds_kernel<<<G, 256, 0, (cudaStream_t)stream>>>(d_perm, n_perm, batch_size, i0, d_seeds,
                                                         d_nseeds, seed_cap, s0, (uint64_t)epoch,
                                                         d_rng);
  return check_launch("fill_seeds");
}

extern "C" int rg_fill_features(const int32_t* d_ids, int64_t n, int32_t d, int32_t stride,
                                uint64_t seed, float* d_out, void* stream) {
  RG_REQUIRE(n >= 0 && d >= 1 && stride >= d, "rg_fill_features: bad sizes");
  if (n == 0) return RG_OK;
  fill_features_kernel<<<kNumSMs * 8, 256, 0, (cudaStream_t)stream>>>(d_ids, n, d, stride, seed,
                                                                       d_out);
  return check_launch("fill_features");
}
