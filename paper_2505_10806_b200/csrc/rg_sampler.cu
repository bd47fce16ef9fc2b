// K2/K3: multi-hop neighbour sampling for G mini-batches at once.
//
// Reference: gnnpipe/sampler.py:86-152 (_sample_neighbors, sample_block).
// For frontier node v with degree D at expansion step d the reference keys
// every position p < D with mix64(nk_v + (p+1)*GOLDEN), nk_v =
// mix64((v+1)*GOLDEN ^ s_d), and keeps the take = min(D, F) smallest
// (sampler.py:102-113).  Keys are pairwise distinct inside a node (mix64 is
// a bijection and GOLDEN is odd) so the selected set is unique and this
// device version is bit-exact.
//
// Layout: one warp per frontier node; the selected neighbour
// ids are emitted ascending into a fixed-stride ELL row (stride = fanout)
// with a per-row count, which is exactly the (dst, src)-sorted edge list of
// sampler.py:145-146 with the dst implied by the row.  The new frontier
// F_{d+1} = F_d U src (np.union1d, sampler.py:148) is a per-batch bitmap
// over all n nodes that accumulates across steps; rg_bitmap_compact turns it
// into the sorted-unique id list.
#include <climits>
#include <cstdlib>

#include "rg_common.cuh"
#include "rg_prng.cuh"

namespace rg {
namespace {

constexpr int kSampleWarps = 8;           // 256-thread CTAs
constexpr int kSlowCap = 4096;            // largest take handled (fanout cap)
constexpr int kCompactWords = 1024;       // bitmap words per compaction CTA
constexpr int kCompactThreads = 256;
constexpr int kScanElems = 1024;          // elements per ELL-scan CTA
constexpr int kFloydBits = 65536;         // PRNG slow path: largest degree with fanout > 32
constexpr int kQueueBatches = 128;        // largest group G of one rg_sample_level call
// items a warp claims from the launch queue per atomic, decoded one per lane
// (Products G = 128, batches/s: 8 12,386; 12 12,404; 16 12,321; 20 12,236;
// 24 12,148; 32 11,924; the earlier per-item warp decode at 8: 12,054;
// another box: 10 12,796; 12 12,716; 14 12,698)
constexpr unsigned kClaim = 10;
constexpr unsigned kClaimLarge = 16;  // groups of >= 64 batches

__device__ __forceinline__ void mark(uint32_t* bm, int32_t v) {
  atomicOr(bm + (v >> 5), 1u << (v & 31));
}

// Selection for D > F, F <= 32: lanes 0..T-1 end up holding the positions of
// the T smallest keys.  Chunk 0 is bitonic-sorted; later chunks only touch
// the list when a key beats the current T-th smallest (ballot filter), which
// for uniform keys happens ~T*ln(D/32) times in total.
__device__ __forceinline__ int select_positions(uint64_t nk, int D, int T) {
  const int lane = lane_id();
  uint64_t kk = nk + (uint64_t)(lane + 1) * GOLDEN;
  uint64_t key = lane < D ? mix64(kk) : ~0ull;
  int pos = lane;
  warp_bitonic_sort(key, pos);
  uint64_t thr = __shfl_sync(kFull, key, T - 1);
  const uint64_t step = 32ull * GOLDEN;
  for (int base = 32; base < D; base += 32) {
    kk += step;
    const bool valid = base + lane < D;
    const uint64_t k2 = mix64(kk);
    unsigned m = __ballot_sync(kFull, valid && k2 < thr);
    while (m) {
      const int s = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t ck = __shfl_sync(kFull, k2, s);
      if (ck < thr) {
        const int i = __popc(__ballot_sync(kFull, key < ck));
        const uint64_t uk = __shfl_up_sync(kFull, key, 1);
        const int up = __shfl_up_sync(kFull, pos, 1);
        if (lane > i) {
          key = uk;
          pos = up;
        }
        if (lane == i) {
          key = ck;
          pos = base + s;
        }
        thr = __shfl_sync(kFull, key, T - 1);
      }
    }
  }
  return pos;
}

// D <= 32 < ... : the take smallest of (at most) 32 distinct keys, one per
// lane, by an MSB-first radix select on ballots; returns the lane mask.
// Distinct keys make it terminate after ~log2(32) informative bits.
__device__ __forceinline__ unsigned select_mask32(uint64_t key, unsigned cand, int need,
                                                  int top_bit = 63) {
  // two key bits per iteration: the candidates split into four buckets
  // (00, 01, 10, 11) by two ballots; whole buckets below the cut are taken,
  // the bucket holding the cut stays the candidate set.  All quantities are
  // warp-uniform, so the branches do not diverge.
  unsigned sel = 0;
  int bit = top_bit;
#pragma unroll 1
  for (; bit >= 1; bit -= 2) {
    const uint32_t two = (uint32_t)(key >> (bit - 1)) & 3u;
    const unsigned b1 = __ballot_sync(kFull, two & 2u);
    const unsigned b0 = __ballot_sync(kFull, two & 1u);
    const unsigned m0 = cand & ~b1 & ~b0;
    const int n0 = __popc(m0);
    if (n0 >= need) {
      cand = m0;
    } else {
      sel |= m0;
      need -= n0;
      const unsigned m1 = cand & ~b1 & b0;
      const int n1 = __popc(m1);
      if (n1 >= need) {
        cand = m1;
      } else {
        sel |= m1;
        need -= n1;
        const unsigned m2 = cand & b1 & ~b0;
        const int n2 = __popc(m2);
        if (n2 >= need) {
          cand = m2;
        } else {
          sel |= m2;
          need -= n2;
          cand &= b1 & b0;
        }
      }
    }
    if (__popc(cand) == need) return sel | cand;
  }
  if (bit == 0) {  // odd number of bits: the last one alone
    const unsigned ones = __ballot_sync(kFull, (uint32_t)key & 1u);
    const unsigned zeros = cand & ~ones;
    const int nz = __popc(zeros);
    if (nz >= need) {
      cand = zeros;
    } else {
      sel |= zeros;
      need -= nz;
      cand &= ones;
    }
    if (__popc(cand) == need) return sel | cand;
  }
  return sel;
}

// Same over up to 64 keys, two per lane (k0: candidate lane, k1: 32+lane),
// two key bits per iteration.
__device__ __forceinline__ void select_mask64(uint64_t k0, uint64_t k1, unsigned c0, unsigned c1,
                                              int need, unsigned& s0, unsigned& s1,
                                              int top_bit = 63) {
  s0 = 0;
  s1 = 0;
  int bit = top_bit;
#pragma unroll 1
  for (; bit >= 1; bit -= 2) {
    const uint32_t t0 = (uint32_t)(k0 >> (bit - 1)) & 3u;
    const uint32_t t1 = (uint32_t)(k1 >> (bit - 1)) & 3u;
    const unsigned a1 = __ballot_sync(kFull, t0 & 2u), a0 = __ballot_sync(kFull, t0 & 1u);
    const unsigned b1 = __ballot_sync(kFull, t1 & 2u), b0 = __ballot_sync(kFull, t1 & 1u);
    // buckets in key order: (~x1 & ~x0), (~x1 & x0), (x1 & ~x0), (x1 & x0)
    unsigned q0 = c0 & ~a1 & ~a0, q1 = c1 & ~b1 & ~b0;
    int n = __popc(q0) + __popc(q1);
    if (n >= need) {
      c0 = q0;
      c1 = q1;
    } else {
      s0 |= q0;
      s1 |= q1;
      need -= n;
      q0 = c0 & ~a1 & a0;
      q1 = c1 & ~b1 & b0;
      n = __popc(q0) + __popc(q1);
      if (n >= need) {
        c0 = q0;
        c1 = q1;
      } else {
        s0 |= q0;
        s1 |= q1;
        need -= n;
        q0 = c0 & a1 & ~a0;
        q1 = c1 & b1 & ~b0;
        n = __popc(q0) + __popc(q1);
        if (n >= need) {
          c0 = q0;
          c1 = q1;
        } else {
          s0 |= q0;
          s1 |= q1;
          need -= n;
          c0 &= a1 & a0;
          c1 &= b1 & b0;
        }
      }
    }
    if (__popc(c0) + __popc(c1) == need) {
      s0 |= c0;
      s1 |= c1;
      return;
    }
  }
  if (bit == 0) {
    const unsigned o0 = __ballot_sync(kFull, (uint32_t)k0 & 1u);
    const unsigned o1 = __ballot_sync(kFull, (uint32_t)k1 & 1u);
    const unsigned z0 = c0 & ~o0, z1 = c1 & ~o1;
    const int nz = __popc(z0) + __popc(z1);
    if (nz >= need) {
      c0 = z0;
      c1 = z1;
    } else {
      s0 |= z0;
      s1 |= z1;
      need -= nz;
      c0 &= o0;
      c1 &= o1;
    }
    if (__popc(c0) + __popc(c1) == need) {
      s0 |= c0;
      s1 |= c1;
    }
  }
}

// D > 32 >= T: a threshold t0 with E[#keys < t0] = T + 3 sqrt(T) + 3 (keys
// are uniform 64-bit values) keeps ~T..T+20 candidates; they are streamed
// into shared memory in position order and the T smallest are radix-
// selected among them.  Exact whenever T <= #candidates <= 64 (every
// non-candidate key is >= t0 > every candidate key); otherwise (rare)
// returns false and the caller uses the running top-T list.
// On success lanes hold the selected positions compacted in position
// order: *nsel = T, selected position r is returned by lane r (r < T).
__device__ __forceinline__ bool select_threshold(uint64_t nk, int D, int T, uint64_t* s_key,
                                                 int32_t* s_pos, int& pos_out) {
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  const float mu = (float)T + 3.0f * sqrtf((float)T) + 3.0f;  // T = F here: loop-invariant
  const float frac = __fdividef(mu, (float)D);  // approximate: only the candidate count moves
  const uint64_t t0 = frac >= 1.0f ? ~0ull : (uint64_t)(frac * 18446744073709551616.0f);
  int count = 0;
  uint64_t kk = nk + (uint64_t)(lane + 1) * GOLDEN;
  const uint64_t step = 32ull * GOLDEN;
  for (int base = 0; base < D; base += 32) {
    const uint64_t key = mix64(kk);
    kk += step;
    const bool c = base + lane < D && key < t0;
    const unsigned m = __ballot_sync(kFull, c);
    if (c) {
      const int off = count + __popc(m & lt);
      if (off < 64) {
        s_key[off] = key;
        s_pos[off] = base + lane;
      }
    }
    count += __popc(m);
  }
  __syncwarp();
  if (count < T || count > 64) return false;
  const uint64_t k0 = lane < count ? s_key[lane] : ~0ull;
  const unsigned c0 = __ballot_sync(kFull, lane < count);
  unsigned s0, s1 = 0u;
  if (count <= 32) {
    // every candidate is < t0: the bits above t0's top bit are zero for all
    s0 = select_mask32(k0, c0, T, 63 - __clzll((long long)t0));  // one ballot per bit
  } else {
    const uint64_t k1 = 32 + lane < count ? s_key[32 + lane] : ~0ull;
    const unsigned c1 = __ballot_sync(kFull, 32 + lane < count);
    // every candidate is < t0: the bits above t0's top bit are zero for all
    select_mask64(k0, k1, c0, c1, T, s0, s1, 63 - __clzll((long long)t0));
  }
  // compact the selected candidates (already in position order) to lanes
  const int n0 = __popc(s0);
  if ((s0 >> lane) & 1u) s_pos[64 + __popc(s0 & lt)] = s_pos[lane];
  if ((s1 >> lane) & 1u) s_pos[64 + n0 + __popc(s1 & lt)] = s_pos[32 + lane];
  __syncwarp();
  pos_out = lane < T ? s_pos[64 + lane] : 0;
  __syncwarp();
  return true;
}

// Lane-parallel Floyd for the PRNG variants: each lane runs the generator of
// its own node; the n-th drawn position goes to col[n * kFloydStride] (a
// per-warp [n][lane] table padded to 33 columns, so both this per-lane
// column and the per-node row read back in phase B are bank-conflict free).
constexpr int kFloydStride = 33;
constexpr unsigned kVariantClaim = 32;  // one node per lane (pcg32: 8 12,322; 16 13,203; 32 13,585)

template <typename Gen>
__device__ __forceinline__ void floyd_lane(Gen& g, int D, int T, int32_t* col) {
#pragma unroll 1
  for (int j = D - T, n = 0; j < D; ++j, ++n) {
    const int t = (int)g.bounded((uint32_t)(j + 1));
    bool dup = false;
#pragma unroll 1
    for (int i = 0; i < n; ++i) dup |= col[i * kFloydStride] == t;
    col[n * kFloydStride] = dup ? j : t;
  }
}

__device__ __forceinline__ void prng_floyd_lane(int prng, uint64_t nk, uint64_t sd, int D, int T,
                                                int32_t* col) {
  if (prng == kPcg32) {
    Pcg32 g;
    g.seed(nk, sd);
    floyd_lane(g, D, T, col);
  } else if (prng == kSfc64) {
    Sfc64 g;
    g.seed(nk, sd);
    floyd_lane(g, D, T, col);
  } else {
    Xoshiro256pp g;
    g.seed(nk, sd);
    floyd_lane(g, D, T, col);
  }
}

// Per-node metadata (CSR row start, degree, id) for every frontier slot,
// one thread per node: the front -> indptr loads then run lane-parallel and
// the warp-per-node kernel starts from one independent 16-B load instead of
// a two-hop dependent chain.
__global__ void __launch_bounds__(256)
    node_meta_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ front,
                     int64_t cap_in, const int32_t* __restrict__ nfront, int4* __restrict__ meta) {
  const int b = blockIdx.y;
  const int nfb = nfront[b];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nfb; j += gridDim.x * blockDim.x) {
    const int64_t r = (int64_t)b * cap_in + j;
    const int32_t v = front[r];
    const int64_t a = indptr[v];
    const int64_t e = indptr[v + 1];
    meta[r] = make_int4((int)(uint32_t)a, (int)(a >> 32), (int)(e - a), v);
  }
}

template <bool kVariants>
__global__ void __launch_bounds__(kSampleWarps * 32)
    sample_level_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                        int G, const int32_t* __restrict__ front, const int4* __restrict__ meta,
                        int64_t cap_in,
                        const int32_t* __restrict__ nfront, int F, uint64_t level_mix,
                        const uint64_t* __restrict__ rng_seed, int32_t* __restrict__ ell,
                        int32_t* __restrict__ cnt, uint32_t* __restrict__ bm, int64_t nwords,
                        int32_t* __restrict__ slow, int sorted_rows, int prng,
                        unsigned* __restrict__ queue, unsigned claim) {
  __shared__ uint64_t s_key[kSampleWarps][64];
  __shared__ int32_t s_pos[kSampleWarps][96];
  __shared__ uint64_t s_seed[kQueueBatches];  // step seed s_d of every batch
  __shared__ int32_t s_nf[kQueueBatches];     // frontier size of every batch
  __shared__ unsigned s_items;
  __shared__ int32_t s_fl[kVariants ? kSampleWarps * 32 * kFloydStride : 1];  // Floyd draws
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  if (threadIdx.x == 0) s_items = 0;
  __syncthreads();
  int mx = 0;
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    const int nf = nfront[i];
    if (i < kQueueBatches) {
      s_seed[i] = mix64(rng_seed[i] ^ level_mix);
      s_nf[i] = nf;
    }
    mx = max(mx, nf);
  }
  atomicMax(&s_items, (unsigned)mx);
  __syncthreads();
  // one launch-wide queue of items k = j*G + b (frontier rank j of batch b):
  // rank-major, so the low (hub-heavy) ranks of every batch go first and the
  // light tail balances across all SMs; warps claim kClaim items at a time
  // (strided, below)
  const unsigned items = s_items * (unsigned)G;
  // batches past the shared-memory tables (G > kQueueBatches: API callers
  // sampling thousands of seeds sets at once) read / derive theirs
  auto step_seed = [&](int b) {
    return b < kQueueBatches ? s_seed[b] : mix64(__ldg(rng_seed + b) ^ level_mix);
  };
  // one frontier node, warp-cooperative: select, emit ascending, mark
  auto sample_node = [&](int64_t row, int64_t a, int D, int b, int32_t v) {
    const int T = min(D, F);
      int32_t* out = ell + row * F;
      uint32_t* bmb = bm + (int64_t)b * nwords;
      if (D <= 32) {
        // one chunk: lane p owns position p.  The row (<= 128 B, the same
        // sectors a selective load would touch) is loaded before the keys are
        // computed, so its latency hides under the selection ALU work.
        const int32_t row_nb = lane < D ? __ldg(indices + a + lane) : INT_MAX;
        unsigned sel;
        if (D <= F) {
          sel = D == 32 ? kFull : ((1u << D) - 1u);
        } else {
          const uint64_t sd = step_seed(b);
          const uint64_t nk = mix64(((uint64_t)v + 1ull) * GOLDEN ^ sd);
          const uint64_t key = lane < D ? mix64(nk + (uint64_t)(lane + 1) * GOLDEN) : ~0ull;
          sel = select_mask32(key, __ballot_sync(kFull, lane < D), T);
        }
        const bool mine = (sel >> lane) & 1u;
        int32_t nb = mine ? row_nb : INT_MAX;
        if (sorted_rows) {
          // ascending CSR row: position order is id order
          if (mine) {
            out[__popc(sel & lt_mask)] = nb;
            mark(bmb, nb);
          }
          return;
        }
        warp_bitonic_sort_keys(nb);
        if (lane < T) {
          out[lane] = nb;
          mark(bmb, nb);
        }
        return;
      }
      // D > 32 (> F): threshold candidates, else the running top-T list
      const uint64_t sd = step_seed(b);
      const uint64_t nk = mix64(((uint64_t)v + 1ull) * GOLDEN ^ sd);
      int pos;
      const bool ordered = select_threshold(nk, D, F, s_key[warp], s_pos[warp], pos);  // T == F here
      if (!ordered) pos = select_positions(nk, D, T);
      int32_t nb = INT_MAX;
      if (sorted_rows) {
        int p = lane < T ? pos : INT_MAX;
        if (!ordered) warp_bitonic_sort_keys(p);
        if (lane < T) {
          nb = __ldg(indices + a + p);
          out[lane] = nb;
          mark(bmb, nb);
        }
        return;
      }
      if (lane < T) nb = __ldg(indices + a + pos);
      warp_bitonic_sort_keys(nb);
      if (lane < T) {
        out[lane] = nb;
        mark(bmb, nb);
      }
  };
  // Claim c takes items c, c + M, c + 2M, ... (M = number of claims) of
  // the rank-major order: each claim holds one item of every tenth of the
  // ranks, so the lowest ranks — the hubs (frontiers are id-sorted and the
  // generator's hubs have low ids) — land one per claim, in the first
  // claims.  Contiguous claims strung several top hubs through one warp
  // when the group is small (Products G = 2: level 1 160 us, the ten top
  // hubs in the first claim).
  const unsigned nclaims = (items + claim - 1) / claim;
  for (;;) {
    unsigned t0 = 0;
    if (lane == 0) t0 = atomicAdd(queue, claim);
    t0 = __shfl_sync(kFull, t0, 0);
    if (t0 >= items) break;
    // phase A, one item per lane: decode, meta load and count for the
    // claim's items at once (and, for the PRNG variants, Floyd's draws in
    // the lane's own generator: they are sequential per node, so a
    // warp-uniform generator would run them 32 times over)
    const unsigned k = (unsigned)lane * nclaims + t0 / claim;
    bool live = false;
    int D = 0, b = 0;
    int32_t v = 0;
    int64_t row = 0, a = 0;
    if (lane < (int)claim && k < items) {
      const int j = (int)(k / (unsigned)G);
      b = (int)(k - (unsigned)j * (unsigned)G);
      if (j < (b < kQueueBatches ? s_nf[b] : __ldg(nfront + b))) {
        row = (int64_t)b * cap_in + j;
        if (meta) {
          const int4 m = __ldg(meta + row);
          a = (int64_t)(((uint64_t)(uint32_t)m.y << 32) | (uint32_t)m.x);
          D = m.z;
          v = m.w;
        } else {
          v = front[row];
          a = indptr[v];
          D = (int)(indptr[v + 1] - a);
        }
        const int T = min(D, F);
        cnt[row] = T;
        if (T > 32) {  // only reachable with fanout > 32: block path
          const int at = atomicAdd(slow, 1);
          slow[1 + at] = (int)k;
        } else {
          live = true;
        }
      }
    }
    unsigned todo = __ballot_sync(kFull, live);
    if constexpr (!kVariants) {
      // phase B: the warp samples the live items one by one
      while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        sample_node(__shfl_sync(kFull, row, src), __shfl_sync(kFull, a, src),
                    __shfl_sync(kFull, D, src), __shfl_sync(kFull, b, src),
                    __shfl_sync(kFull, v, src));
      }
    } else {
      int32_t* s_flw = s_fl + warp * (32 * kFloydStride);
      if (live && D > F) {
        const uint64_t sd = step_seed(b);
        const uint64_t nk = mix64(((uint64_t)v + 1ull) * GOLDEN ^ sd);
        prng_floyd_lane(prng, nk, sd, D, F, s_flw + lane);  // T == F here
      }
      __syncwarp();
      // phase B, warp per item: neighbour loads, ascending emission, marks
      while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const int64_t r_row = __shfl_sync(kFull, row, src);
        const int64_t r_a = __shfl_sync(kFull, a, src);
        const int r_D = __shfl_sync(kFull, D, src);
        const int r_b = __shfl_sync(kFull, b, src);
        const int r_T = min(r_D, F);
        int32_t x = INT_MAX;
        if (r_D > F) {
          int p = lane < r_T ? s_flw[lane * kFloydStride + src] : INT_MAX;
          if (sorted_rows) {
            warp_bitonic_sort_keys(p);
            if (lane < r_T) x = __ldg(indices + r_a + p);
          } else {
            if (lane < r_T) x = __ldg(indices + r_a + p);
            warp_bitonic_sort_keys(x);
          }
        } else {  // D <= F <= 32: the whole row
          if (lane < r_D) x = __ldg(indices + r_a + lane);
          if (!sorted_rows) warp_bitonic_sort_keys(x);
        }
        if (lane < r_T) {
          ell[r_row * F + lane] = x;
          mark(bm + (int64_t)r_b * nwords, x);
        }
      }
      __syncwarp();  // the next claim reuses s_flw
    }
  }  // claims
}

// ---- take > 32 (fanout > 32): one CTA per node, shared-memory sort -------
__device__ void block_sort_smem(int32_t* s, int n) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = n + threadIdx.x; i < P; i += blockDim.x) s[i] = INT_MAX;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const int32_t x = s[i], y = s[l];
          if ((x > y) == up) {
            s[i] = y;
            s[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(256)
    sample_slow_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                       int G, const int32_t* __restrict__ front, int64_t cap_in, int F,
                       uint64_t level_mix, const uint64_t* __restrict__ rng_seed,
                       int32_t* __restrict__ ell, uint32_t* __restrict__ bm, int64_t nwords,
                       const int32_t* __restrict__ slow, int prng) {
  __shared__ int32_t s_val[2 * kSlowCap];
  __shared__ uint32_t s_pick[kFloydBits / 32];
  __shared__ uint32_t s_hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int s_rank, s_fill;
  const int nslow = slow[0];
  for (int it = blockIdx.x; it < nslow; it += gridDim.x) {
    const int64_t k = (uint32_t)slow[1 + it];  // queue items are < 2^32 (host check)
    const int j = (int)(k / G), b = (int)(k - (int64_t)j * G);
    const int64_t row = (int64_t)b * cap_in + j;
    const int32_t v = front[row];
    const int64_t a = indptr[v];
    const int D = (int)(indptr[v + 1] - a);
    const int T = min(D, F);
    if (D <= F) {
      for (int p = threadIdx.x; p < D; p += blockDim.x) s_val[p] = indices[a + p];
    } else if (prng != kSplitMix) {
      // Floyd's k-subset: for j = D-T .. D-1 draw t in [0, j]; keep t unless
      // already picked, else keep j.  Membership over a D-bit shared bitmap
      // (D <= kFloydBits), or by scanning the <= T picks so far (any D); one
      // thread draws, then the picked positions become neighbour ids.
      const bool bitmap = D <= kFloydBits;
      if (bitmap)
        for (int i = threadIdx.x; i < (D + 31) / 32; i += blockDim.x) s_pick[i] = 0u;
      if (threadIdx.x == 0) s_fill = 0;
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint64_t sd = mix64(rng_seed[b] ^ level_mix);
        const uint64_t nk = mix64(((uint64_t)v + 1ull) * GOLDEN ^ sd);
        Pcg32 g1;
        Sfc64 g2;
        Xoshiro256pp g3;
        g1.seed(nk, sd);
        g2.seed(nk, sd);
        g3.seed(nk, sd);
        int n = 0;
        for (int j = D - T; j < D; ++j) {
          const uint32_t n1 = (uint32_t)(j + 1);
          const int t = (int)(prng == kPcg32 ? g1.bounded(n1)
                                              : prng == kSfc64 ? g2.bounded(n1) : g3.bounded(n1));
          bool seen;
          if (bitmap) {
            seen = (s_pick[t >> 5] >> (t & 31)) & 1u;
          } else {
            seen = false;
            for (int q = 0; q < n; ++q) seen |= s_val[q] == t;
          }
          const int pick = seen ? j : t;
          if (bitmap)
            s_pick[pick >> 5] |= 1u << (pick & 31);
          else
            s_val[n++] = pick;
        }
      }
      __syncthreads();
      if (bitmap) {
        for (int p = threadIdx.x; p < D; p += blockDim.x)
          if ((s_pick[p >> 5] >> (p & 31)) & 1u) s_val[atomicAdd(&s_fill, 1)] = indices[a + p];
      } else {
        for (int i = threadIdx.x; i < T; i += blockDim.x) s_val[i] = indices[a + s_val[i]];
      }
    } else {
      // radix-select the T-th smallest key (8 passes of 8 bits), then keep
      // every position whose key is <= it: exactly T positions.
      const uint64_t sd = mix64(rng_seed[b] ^ level_mix);
      const uint64_t nk = mix64(((uint64_t)v + 1ull) * GOLDEN ^ sd);
      if (threadIdx.x == 0) {
        s_prefix = 0;
        s_rank = T;  // 1-based rank still to find inside the prefix class
        s_fill = 0;
      }
      for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_hist[i] = 0;
        __syncthreads();
        const uint64_t hi_mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
        const uint64_t prefix = s_prefix;
        for (int p = threadIdx.x; p < D; p += blockDim.x) {
          const uint64_t key = mix64(nk + (uint64_t)(p + 1) * GOLDEN);
          if ((key & hi_mask) == prefix) atomicAdd(&s_hist[(key >> shift) & 255], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          int r = s_rank;
          int dgt = 0;
          while ((int)s_hist[dgt] < r) r -= s_hist[dgt++];
          s_rank = r;
          s_prefix = prefix | ((uint64_t)dgt << shift);
        }
        __syncthreads();
      }
      const uint64_t kth = s_prefix;
      for (int p = threadIdx.x; p < D; p += blockDim.x) {
        const uint64_t key = mix64(nk + (uint64_t)(p + 1) * GOLDEN);
        if (key <= kth) s_val[atomicAdd(&s_fill, 1)] = indices[a + p];
      }
    }
    __syncthreads();
    block_sort_smem(s_val, T);
    int32_t* out = ell + row * F;
    uint32_t* bmb = bm + (int64_t)b * nwords;
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
      out[i] = s_val[i];
      mark(bmb, s_val[i]);
    }
    __syncthreads();
  }
}

__global__ void mark_seeds_kernel(const int32_t* __restrict__ seeds,
                                  const int32_t* __restrict__ nseeds, int seed_cap,
                                  uint32_t* __restrict__ bm, int64_t nwords) {
  const int b = blockIdx.y;
  const int ns = nseeds[b];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x)
    mark(bm + (int64_t)b * nwords, seeds[(int64_t)b * seed_cap + i]);
}

// ---- bitmap -> sorted unique ids ----------------------------------------
__global__ void __launch_bounds__(kCompactThreads)
    bitmap_count_kernel(const uint32_t* __restrict__ bm, int64_t nwords, int64_t nchunks,
                        int32_t* __restrict__ chunk_tot) {
  __shared__ int s_red[32];
  const int b = blockIdx.y;
  const uint32_t* w = bm + (int64_t)b * nwords;
  const int64_t w0 = (int64_t)blockIdx.x * kCompactWords + threadIdx.x * 4;
  int c = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (w0 + i < nwords) c += __popc(w[w0 + i]);
  int tot;
  block_excl_scan<kCompactThreads>(c, s_red, &tot);
  if (threadIdx.x == 0) chunk_tot[(int64_t)b * nchunks + blockIdx.x] = tot;
}

// Exclusive prefix of the chunk totals per batch, in place, and the batch
// total: one CTA per batch.  Used when there are many chunks (papers100M
// shape: ~3,400 per batch); with few, the emit kernel sums the totals before
// its chunk itself (one pass, no extra launch).
constexpr int64_t kEmitScanMax = 256;
constexpr int kChunkScanThreads = 1024;

__global__ void __launch_bounds__(kChunkScanThreads)
    chunk_scan_kernel(int32_t* __restrict__ chunk, int64_t nchunks, int32_t* __restrict__ nout) {
  __shared__ int s_red[32];
  int32_t* c = chunk + (int64_t)blockIdx.x * nchunks;
  int carry = 0;
  for (int64_t base = 0; base < nchunks; base += kChunkScanThreads) {
    const int64_t i = base + threadIdx.x;
    const int v = i < nchunks ? c[i] : 0;
    int tot;
    const int ex = block_excl_scan<kChunkScanThreads>(v, s_red, &tot);
    if (i < nchunks) c[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) nout[blockIdx.x] = carry;
}

// Emission is warp-cooperative: each warp owns kCompactWords/8 consecutive
// words; for every word the 32 lanes test one bit each and the set bits are
// written with one coalesced store (ballot + prefix popcount).
// prescanned: chunk_tot already holds exclusive prefixes (chunk_scan_kernel,
// which also wrote nout); else every CTA sums the totals before its chunk
// (quadratic in the chunk count: only for few chunks).
__global__ void __launch_bounds__(kCompactThreads)
    bitmap_emit_kernel(const uint32_t* __restrict__ bm, int64_t nwords, int64_t nchunks,
                       const int32_t* __restrict__ chunk_tot, int32_t* __restrict__ out,
                       int64_t cap_out, int32_t* __restrict__ nout, int32_t* __restrict__ wpre,
                       int prescanned) {
  constexpr int kWarps = kCompactThreads / 32;
  constexpr int kPerWarp = kCompactWords / kWarps;  // 128 words
  __shared__ int s_red[32];
  __shared__ int s_base;
  __shared__ int s_warp[kWarps];
  __shared__ int32_t s_ids[kWarps][32 * 32];  // one 32-word group's ids per warp
  const int b = blockIdx.y;
  const int64_t chunk = blockIdx.x;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  if (prescanned) {
    if (threadIdx.x == 0) s_base = chunk_tot[(int64_t)b * nchunks + chunk];
    __syncthreads();
  } else {
    int before = 0, all = 0;
    for (int64_t c = threadIdx.x; c < nchunks; c += blockDim.x) {
      const int t = chunk_tot[(int64_t)b * nchunks + c];
      all += t;
      if (c < chunk) before += t;
    }
    int tot;
    block_excl_scan<kCompactThreads>(before, s_red, &tot);
    if (threadIdx.x == 0) s_base = tot;
    __syncthreads();
    if (chunk == 0) {
      int grand;
      block_excl_scan<kCompactThreads>(all, s_red, &grand);
      if (threadIdx.x == 0) nout[b] = grand;
    }
  }
  const uint32_t* w = bm + (int64_t)b * nwords;
  const int64_t wbase = chunk * kCompactWords + (int64_t)warp * kPerWarp;
  uint32_t words[kPerWarp / 32];
  int wsum = 0;
#pragma unroll
  for (int g = 0; g < kPerWarp / 32; ++g) {
    const int64_t wi = wbase + g * 32 + lane;
    words[g] = wi < nwords ? w[wi] : 0u;
    wsum += __popc(words[g]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(kFull, wsum, o);
  if (lane == 0) s_warp[warp] = wsum;
  __syncthreads();
  int at = s_base;
  for (int i = 0; i < warp; ++i) at += s_warp[i];
  int32_t* o = out + (int64_t)b * cap_out;
  int32_t* sid = s_ids[warp];
#pragma unroll
  for (int g = 0; g < kPerWarp / 32; ++g) {
    // exclusive prefix of this group's word popcounts
    const int c = __popc(words[g]);
    int x = c;
#pragma unroll
    for (int s2 = 1; s2 < 32; s2 <<= 1) {
      const int y = __shfl_up_sync(kFull, x, s2);
      if (lane >= s2) x += y;
    }
    const int64_t wi = wbase + g * 32 + lane;
    if (wpre && wi < nwords) wpre[(int64_t)b * nwords + wi] = at + x - c;
    const int gsum = __shfl_sync(kFull, x, 31);
    // each lane writes its own word's ids (ascending) into the warp's run,
    // then the run goes out with coalesced stores
    uint32_t word = words[g];
    int p = x - c;
    const int32_t idbase = (int32_t)(wi * 32);
    while (word) {
      sid[p++] = idbase + (__ffs(word) - 1);
      word &= word - 1u;
    }
    __syncwarp();
    for (int i = lane; i < gsum; i += 32) {
      const int pos = at + i;
      if (pos < cap_out) o[pos] = sid[i];
    }
    __syncwarp();
    at += gsum;
  }
}

__global__ void bitmap_set_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ n,
                                  uint32_t* __restrict__ bm) {
  const int cnt = *n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    mark(bm, ids[i]);
}

// ---- ELL -> flat (src, dst) edges for the numpy API ----------------------
__global__ void __launch_bounds__(256)
    ell_count_kernel(const int32_t* __restrict__ nfront, int64_t cap_in,
                     const int32_t* __restrict__ cnt, int64_t nchunks,
                     int32_t* __restrict__ chunk_tot) {
  __shared__ int s_red[32];
  const int b = blockIdx.y;
  const int nf = nfront[b];
  const int64_t j0 = (int64_t)blockIdx.x * kScanElems + threadIdx.x * 4;
  int c = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (j0 + i < nf) c += cnt[(int64_t)b * cap_in + j0 + i];
  int tot;
  block_excl_scan<256>(c, s_red, &tot);
  if (threadIdx.x == 0) chunk_tot[(int64_t)b * nchunks + blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256)
    ell_emit_kernel(const int32_t* __restrict__ front, const int32_t* __restrict__ nfront,
                    int64_t cap_in, const int32_t* __restrict__ ell,
                    const int32_t* __restrict__ cnt, int F, int64_t nchunks,
                    const int32_t* __restrict__ chunk_tot, int32_t* __restrict__ eoff,
                    int32_t* __restrict__ src, int32_t* __restrict__ dst, int64_t cap_e,
                    int32_t* __restrict__ nedge) {
  __shared__ int s_red[32];
  __shared__ int s_base;
  const int b = blockIdx.y;
  const int nf = nfront[b];
  const int64_t chunk = blockIdx.x;
  int before = 0, all = 0;
  for (int64_t c = threadIdx.x; c < nchunks; c += blockDim.x) {
    const int t = chunk_tot[(int64_t)b * nchunks + c];
    all += t;
    if (c < chunk) before += t;
  }
  int tot;
  block_excl_scan<256>(before, s_red, &tot);
  if (threadIdx.x == 0) s_base = tot;
  __syncthreads();
  const int base = s_base;
  __syncthreads();
  int grand;
  block_excl_scan<256>(all, s_red, &grand);
  if (chunk == 0 && threadIdx.x == 0) {
    nedge[b] = grand;
    eoff[(int64_t)b * (cap_in + 1) + nf] = grand;
  }
  const int64_t j0 = chunk * kScanElems + threadIdx.x * 4;
  int c[4];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    c[i] = (j0 + i < nf) ? cnt[(int64_t)b * cap_in + j0 + i] : 0;
    sum += c[i];
  }
  int dummy;
  int at = base + block_excl_scan<256>(sum, s_red, &dummy);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t j = j0 + i;
    if (j >= nf) break;
    const int64_t row = (int64_t)b * cap_in + j;
    eoff[(int64_t)b * (cap_in + 1) + j] = at;
    const int32_t d = front[row];
    for (int r = 0; r < c[i]; ++r) {
      if (at < cap_e) {
        src[(int64_t)b * cap_e + at] = ell[row * F + r];
        dst[(int64_t)b * cap_e + at] = d;
      }
      ++at;
    }
  }
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" int rg_mark_seeds(const int32_t* d_seeds, const int32_t* d_nseeds, int32_t G,
                             int32_t seed_cap, uint32_t* d_bm, int64_t nwords, void* stream) {
  RG_REQUIRE(G >= 1 && G <= 65535 && seed_cap >= 1, "rg_mark_seeds: bad G=%d cap=%d", G,
             seed_cap);
  const int blocks = (int)std::min<int64_t>((seed_cap + 255) / 256, 64);
  mark_seeds_kernel<<<dim3(blocks, G), 256, 0, (cudaStream_t)stream>>>(d_seeds, d_nseeds,
                                                                       seed_cap, d_bm, nwords);
  return check_launch("mark_seeds");
}

extern "C" int rg_sample_level(const int64_t* d_indptr, const int32_t* d_indices, int64_t n,
                               int32_t G, const int32_t* d_front, int64_t cap_in,
                               const int32_t* d_nfront, int32_t fanout, int32_t level,
                               const uint64_t* d_rng_seed, int32_t* d_ell, int32_t* d_cnt,
                               uint32_t* d_bm, int64_t nwords, int32_t* d_slow,
                               int32_t* d_meta, int32_t sorted_rows, int32_t prng,
                               void* stream) {
  RG_REQUIRE(prng >= kSplitMix && prng <= kXoshiro256pp, "rg_sample_level: unknown prng %d", prng);
  RG_REQUIRE(G >= 1 && G <= 65535 && cap_in >= 1 && n >= 1, "rg_sample_level: bad sizes");
  RG_REQUIRE(fanout >= 1, "rg_sample_level: fanout must be >= 1");
  if (fanout > kSlowCap) {
    set_error("rg_sample_level: fanout %d above the supported %d", fanout, kSlowCap);
    return RG_ERR_UNSUPPORTED;
  }
  RG_REQUIRE(fanout <= 32 || d_slow != nullptr, "rg_sample_level: fanout > 32 needs d_slow");
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t level_mix = (uint64_t)(level + 1) * GOLDEN;  // sampler.py:143
  int32_t* slow = fanout > 32 ? d_slow : nullptr;
  if (slow && cudaMemsetAsync(slow, 0, sizeof(int32_t), s) != cudaSuccess)
    return check_launch("sample_level memset");
  RG_REQUIRE(d_meta != nullptr, "rg_sample_level: d_meta scratch is required");
  // headroom: every warp adds one claim past the end before it stops
  RG_REQUIRE((uint64_t)G * (uint64_t)cap_in < (1ull << 32) - (1ull << 24),
             "rg_sample_level: G * cap_in above the 32-bit work queue");
  int4* meta = reinterpret_cast<int4*>(d_meta);
  // launch-wide work queue: the extra record after the G*cap_in meta records
  unsigned* queue = reinterpret_cast<unsigned*>(meta + (int64_t)G * cap_in);
  if (cudaMemsetAsync(queue, 0, sizeof(unsigned), s) != cudaSuccess)
    return check_launch("sample_level queue");
  {
    const int bx = (int)std::min<int64_t>((cap_in + 255) / 256, std::max(1, kNumSMs * 16 / G));
    node_meta_kernel<<<dim3(bx, G), 256, 0, s>>>(d_indptr, d_front, cap_in, d_nfront, meta);
    if (int rc = check_launch("node_meta")) return rc;
  }
  static const unsigned claim_env = [] {
    const char* e = getenv("RG_SAMPLER_CLAIM");
    return e ? (unsigned)std::max(1, std::min(32, atoi(e))) : 0u;
  }();
  // larger claims amortise the queue atomic when every batch's frontier is
  // in the launch; small groups need the finer split (Products, same box:
  // G = 128 claim 16 14,184 vs 10 14,116 batches/s; G = 2 5,275 vs 5,475)
  const unsigned claim = claim_env ? claim_env : (G >= 64 ? kClaimLarge : kClaim);
  // one wave: 48 regs x 256 threads = 5 CTAs per SM (capping at 40 regs for
  // 6/SM measured 1-2 % slower; the PRNG variants at 4/SM: -1.2 %);
  // SplitMix64 keys (the reference) and the PRNG variants are separate
  // instantiations so the reference path keeps its register budget
  static const unsigned vclaim = [] {
    const char* e = getenv("RG_SAMPLER_VCLAIM");
    return e ? (unsigned)std::max(1, std::min(32, atoi(e))) : kVariantClaim;
  }();
  static const int vctas = [] {
    const char* e = getenv("RG_SAMPLER_VCTAS");
    return e ? std::max(1, std::min(5, atoi(e))) : 5;
  }();
  if (prng == kSplitMix)
    sample_level_kernel<false><<<kNumSMs * 5, kSampleWarps * 32, 0, s>>>(
        d_indptr, d_indices, G, d_front, meta, cap_in, d_nfront, fanout, level_mix, d_rng_seed,
        d_ell, d_cnt, d_bm, nwords, slow, sorted_rows, prng, queue, claim);
  else
    sample_level_kernel<true><<<kNumSMs * vctas, kSampleWarps * 32, 0, s>>>(
        d_indptr, d_indices, G, d_front, meta, cap_in, d_nfront, fanout, level_mix, d_rng_seed,
        d_ell, d_cnt, d_bm, nwords, slow, sorted_rows, prng, queue, vclaim);
  int rc = check_launch("sample_level");
  if (rc || !slow) return rc;
  sample_slow_kernel<<<kNumSMs, 256, 0, s>>>(d_indptr, d_indices, G, d_front, cap_in, fanout,
                                             level_mix, d_rng_seed, d_ell, d_bm, nwords, slow,
                                             prng);
  return check_launch("sample_slow");
}

extern "C" int64_t rg_bitmap_chunks(int64_t nwords) {
  return (nwords + kCompactWords - 1) / kCompactWords;
}

extern "C" int rg_bitmap_compact_launches(int64_t nwords) {
  return rg_bitmap_chunks(nwords) > kEmitScanMax ? 3 : 2;
}

extern "C" int rg_bitmap_compact(const uint32_t* d_bm, int64_t nwords, int32_t G,
                                 int32_t* d_chunk, int32_t* d_out, int64_t cap_out,
                                 int32_t* d_nout, int32_t* d_wpre, void* stream) {
  RG_REQUIRE(G >= 1 && G <= 65535 && nwords >= 1, "rg_bitmap_compact: bad sizes");
  const int64_t nchunks = rg_bitmap_chunks(nwords);
  RG_REQUIRE(nchunks < (1ll << 31), "rg_bitmap_compact: too many chunks");
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)nchunks, G);
  bitmap_count_kernel<<<grid, kCompactThreads, 0, s>>>(d_bm, nwords, nchunks, d_chunk);
  int rc = check_launch("bitmap_count");
  if (rc) return rc;
  const int prescanned = nchunks > kEmitScanMax;
  if (prescanned) {
    chunk_scan_kernel<<<G, kChunkScanThreads, 0, s>>>(d_chunk, nchunks, d_nout);
    if ((rc = check_launch("chunk_scan"))) return rc;
  }
  bitmap_emit_kernel<<<grid, kCompactThreads, 0, s>>>(d_bm, nwords, nchunks, d_chunk, d_out,
                                                      cap_out, d_nout, d_wpre, prescanned);
  return check_launch("bitmap_emit");
}

extern "C" int rg_bitmap_set(const int32_t* d_ids, const int32_t* d_n, uint32_t* d_bm,
                             void* stream) {
  bitmap_set_kernel<<<kNumSMs * 2, 256, 0, (cudaStream_t)stream>>>(d_ids, d_n, d_bm);
  return check_launch("bitmap_set");
}

extern "C" int64_t rg_scan_chunks(int64_t cap) { return (cap + kScanElems - 1) / kScanElems; }

extern "C" int rg_ell_to_edges(const int32_t* d_front, const int32_t* d_nfront, int64_t cap_in,
                               const int32_t* d_ell, const int32_t* d_cnt, int32_t fanout,
                               int32_t G, int32_t* d_chunk, int32_t* d_eoff, int32_t* d_src,
                               int32_t* d_dst, int64_t cap_e, int32_t* d_nedge, void* stream) {
  RG_REQUIRE(G >= 1 && G <= 65535 && cap_in >= 1 && fanout >= 1, "rg_ell_to_edges: bad sizes");
  const int64_t nchunks = rg_scan_chunks(cap_in);
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)nchunks, G);
  ell_count_kernel<<<grid, 256, 0, s>>>(d_nfront, cap_in, d_cnt, nchunks, d_chunk);
  int rc = check_launch("ell_count");
  if (rc) return rc;
  ell_emit_kernel<<<grid, 256, 0, s>>>(d_front, d_nfront, cap_in, d_ell, d_cnt, fanout, nchunks,
                                       d_chunk, d_eoff, d_src, d_dst, cap_e, d_nedge);
  return check_launch("ell_emit");
}
