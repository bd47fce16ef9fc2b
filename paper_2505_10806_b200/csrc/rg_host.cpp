// Host-side graph materialisation for the benchmark shapes.
//
// The hot path consumes a CSR graph and a partition owner array; producing
// them is outside the path, but the reference's
// generator is a Python loop (graph.py:157-174) and its LDG partitioner a
// Python BFS (partition.py:55-76) that take minutes at Products scale.  These
// are native restatements that reproduce the reference's outputs exactly:
//
//  * rg_synth_powerlaw_csr  == gnnpipe.graph.synth_powerlaw(n, m, ...) CSR
//    (graph.py:145-182).  The draw stream is numpy's Philox4x64-10 bit
//    generator (key taken from numpy's SeedSequence by the caller) feeding
//    Generator.integers(0, rep_len, size=m), i.e. numpy's buffered 32-bit
//    Lemire bounded draw.  Features/labels are not produced here.
//  * rg_partition_edgecut == gnnpipe.partition.partition_edgecut
//    (partition.py:37-77), same float64 scoring and tie-breaks.
//
// Both are pinned against hashes of the reference's own outputs in
// tests/golden (see tests/golden/make_golden.py).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <limits>
#include <vector>

#include "../../include/rapidgnn_b200.h"

namespace {

typedef unsigned __int128 u128;

struct Philox4x64 {
  uint64_t ctr[4] = {0, 0, 0, 0};
  uint64_t key[2];
  uint64_t buf[4] = {0, 0, 0, 0};
  int pos = 4;
  bool has32 = false;
  uint32_t hold32 = 0;

  static void block(const uint64_t c[4], const uint64_t k_in[2], uint64_t out[4]) {
    uint64_t k0 = k_in[0], k1 = k_in[1];
    uint64_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
    for (int r = 0; r < 10; ++r) {
      if (r) {
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
      }
      u128 p0 = (u128)0xD2E7470EE14C6C93ULL * x0;
      u128 p1 = (u128)0xCA5A826395121157ULL * x2;
      uint64_t y0 = (uint64_t)(p1 >> 64) ^ x1 ^ k0;
      uint64_t y1 = (uint64_t)p1;
      uint64_t y2 = (uint64_t)(p0 >> 64) ^ x3 ^ k1;
      uint64_t y3 = (uint64_t)p0;
      x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
  }

  uint64_t next64() {
    if (pos < 4) return buf[pos++];
    if (++ctr[0] == 0 && ++ctr[1] == 0 && ++ctr[2] == 0) ++ctr[3];
    block(ctr, key, buf);
    pos = 1;
    return buf[0];
  }

  uint32_t next32() {
    if (has32) {
      has32 = false;
      return hold32;
    }
    uint64_t v = next64();
    has32 = true;
    hold32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }

  // numpy random_bounded_uint64_fill, rng <= 0xFFFFFFFE, use_masked=False:
  // buffered_bounded_lemire_uint32 with rng_excl = rng + 1.
  uint32_t lemire32(uint32_t rng_excl) {
    uint64_t m = (uint64_t)next32() * rng_excl;
    uint32_t left = (uint32_t)m;
    if (left < rng_excl) {
      const uint32_t thresh = (uint32_t)(UINT32_MAX - (rng_excl - 1)) % rng_excl;
      while (left < thresh) {
        m = (uint64_t)next32() * rng_excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

}  // namespace

extern "C" int rg_philox_raw(uint64_t key0, uint64_t key1, int64_t count, uint64_t* out) {
  Philox4x64 g;
  g.key[0] = key0;
  g.key[1] = key1;
  for (int64_t i = 0; i < count; ++i) out[i] = g.next64();
  return 0;
}

extern "C" int rg_synth_powerlaw_csr(int64_t n, int64_t m, uint64_t key0, uint64_t key1,
                                     int64_t* indptr, int32_t* indices, uint64_t* state_out) {
  if (m < 1 || n <= m) return RG_ERR_INVALID;
  const int64_t n_new = n - m;
  if (2 * m * n_new >= (int64_t)UINT32_MAX) return RG_ERR_INVALID;
  if (n > (int64_t)INT32_MAX) return RG_ERR_INVALID;
  Philox4x64 g;
  g.key[0] = key0;
  g.key[1] = key1;

  // (new node v) -> its m sorted attachment targets, laid out v-major.
  std::vector<int32_t> tgt((size_t)(m * n_new));
  std::vector<int32_t> rep((size_t)(2 * m * n_new));
  std::vector<int32_t> stamp((size_t)n, -1);
  std::vector<uint32_t> draw((size_t)m);
  std::vector<int32_t> chosen;
  chosen.reserve((size_t)m);
  std::vector<int32_t> targets((size_t)m);
  for (int64_t i = 0; i < m; ++i) targets[i] = (int32_t)i;
  int64_t rep_len = 0;
  for (int64_t v = m; v < n; ++v) {
    int32_t* row = &tgt[(size_t)((v - m) * m)];
    for (int64_t i = 0; i < m; ++i) row[i] = targets[i];
    for (int64_t i = 0; i < m; ++i) rep[rep_len + i] = targets[i];
    for (int64_t i = 0; i < m; ++i) rep[rep_len + m + i] = (int32_t)v;
    rep_len += 2 * m;
    if (v == n - 1) break;
    chosen.clear();
    while ((int64_t)chosen.size() < m) {
      // one Generator.integers(0, rep_len, size=m) call consumes all m draws
      for (int64_t i = 0; i < m; ++i) draw[i] = g.lemire32((uint32_t)rep_len);
      for (int64_t i = 0; i < m; ++i) {
        int32_t t = rep[draw[i]];
        if (stamp[t] != (int32_t)v) {
          stamp[t] = (int32_t)v;
          chosen.push_back(t);
          if ((int64_t)chosen.size() == m) break;
        }
      }
    }
    std::sort(chosen.begin(), chosen.end());
    for (int64_t i = 0; i < m; ++i) targets[i] = chosen[i];
  }
  if (state_out) {  // numpy Philox state after the attachment loop
    for (int i = 0; i < 4; ++i) state_out[i] = g.ctr[i];
    state_out[4] = g.key[0];
    state_out[5] = g.key[1];
    for (int i = 0; i < 4; ++i) state_out[6 + i] = g.buf[i];
    state_out[10] = (uint64_t)g.pos;
    state_out[11] = g.has32 ? 1 : 0;
    state_out[12] = g.hold32;
  }

  // symmetric CSR, rows sorted ascending (graph.py:176-182)
  std::vector<int64_t> deg((size_t)n, 0);
  for (int64_t v = m; v < n; ++v) {
    deg[v] += m;
    const int32_t* row = &tgt[(size_t)((v - m) * m)];
    for (int64_t i = 0; i < m; ++i) deg[row[i]] += 1;
  }
  indptr[0] = 0;
  for (int64_t v = 0; v < n; ++v) indptr[v + 1] = indptr[v] + deg[v];
  std::vector<int64_t> fill(indptr, indptr + n);
  for (int64_t v = m; v < n; ++v) {
    const int32_t* row = &tgt[(size_t)((v - m) * m)];
    for (int64_t i = 0; i < m; ++i) {
      indices[fill[v]++] = row[i];
      indices[fill[row[i]]++] = (int32_t)v;
    }
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; ++v) std::sort(indices + indptr[v], indices + indptr[v + 1]);
  return 0;
}

extern "C" int rg_partition_edgecut(int64_t n, const int64_t* indptr, const int32_t* indices,
                                    int32_t k, int32_t* owner) {
  if (k < 1 || n < 0) return RG_ERR_INVALID;
  const int64_t capacity = (int64_t)std::ceil(1.05 * (double)n / (double)k);
  std::vector<int64_t> sizes((size_t)k, 0);
  std::vector<uint8_t> visited((size_t)n, 0);
  std::vector<int64_t> counts((size_t)k);
  std::vector<double> score((size_t)k);
  std::deque<int32_t> queue;
  for (int64_t i = 0; i < n; ++i) owner[i] = -1;
  int64_t next_start = 0;
  const double neg_inf = -std::numeric_limits<double>::infinity();
  for (int64_t it = 0; it < n; ++it) {
    if (queue.empty()) {
      while (visited[next_start]) ++next_start;
      queue.push_back((int32_t)next_start);
      visited[next_start] = 1;
    }
    const int32_t v = queue.front();
    queue.pop_front();
    std::fill(counts.begin(), counts.end(), 0);
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
      int32_t o = owner[indices[e]];
      if (o >= 0) counts[o] += 1;
    }
    double best = neg_inf;
    for (int32_t p = 0; p < k; ++p) {
      double s = (double)counts[p] * (1.0 - (double)sizes[p] / (double)capacity);
      if (sizes[p] >= capacity) s = neg_inf;
      score[p] = s;
      if (p == 0 || s > best) best = s;
    }
    int32_t pick = -1;
    for (int32_t p = 0; p < k; ++p) {
      if (score[p] == best && (pick < 0 || sizes[p] < sizes[pick])) pick = p;
    }
    owner[v] = pick;
    sizes[pick] += 1;
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
      int32_t u = indices[e];
      if (!visited[u]) {
        visited[u] = 1;
        queue.push_back(u);
      }
    }
  }
  return 0;
}
