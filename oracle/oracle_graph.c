/* CPU ORACLE — test infrastructure, not product code.
 *
 * Plain-C restatement of the reference's input generators, so the bench's
 * reference arm (bench.py --impl reference) and the CPU baseline can build
 * the Products-shape graph in seconds without loading the product library:
 *
 *   oracle_synth_powerlaw_csr  == gnnpipe.graph.synth_powerlaw's attachment
 *       loop and CSR (graph.py:145-182): numpy Generator(Philox(seed)),
 *       rng.integers(0, rep_len, size=m) per attempt (numpy's
 *       random_bounded_uint64_fill -> buffered_bounded_lemire_uint32 with the
 *       bit generator's persistent 32-bit half buffer), distinct targets
 *       accumulated in draw order, sorted; CSR rows sorted by (src, dst).
 *       The Philox state after the loop is returned so numpy continues the
 *       same stream for features (graph.py:184).
 *   oracle_partition_edgecut   == gnnpipe.partition.partition_edgecut
 *       (partition.py:37-77): BFS from the lowest unvisited node, LDG score
 *       count_p * (1 - size_p / capacity) in float64, full partitions
 *       excluded, ties -> least loaded -> lowest index.
 *
 * Pinned: tests/test_oracle_golden.py checks both against the content hashes
 * the reference itself produced (tests/golden/golden.json, "graphs").
 * Built by oracle/Makefile (gcc) into oracle/_build/liboracle_graph.so.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

typedef struct {
  uint64_t ctr[4], key[2], buf[4];
  int pos;          /* next buffered output; 4 = empty */
  int has32;        /* numpy bitgen has_uint32 */
  uint32_t half;    /* numpy bitgen uinteger */
} philox_t;

static void philox_block(philox_t* s) {
  uint64_t x[4] = {s->ctr[0], s->ctr[1], s->ctr[2], s->ctr[3]};
  uint64_t k0 = s->key[0], k1 = s->key[1];
  for (int r = 0; r < 10; ++r) {
    u128 a = (u128)0xD2E7470EE14C6C93ULL * x[0];
    u128 b = (u128)0xCA5A826395121157ULL * x[2];
    uint64_t y0 = (uint64_t)(b >> 64) ^ x[1] ^ k0;
    uint64_t y2 = (uint64_t)(a >> 64) ^ x[3] ^ k1;
    x[1] = (uint64_t)b;
    x[3] = (uint64_t)a;
    x[0] = y0;
    x[2] = y2;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  memcpy(s->buf, x, sizeof x);
}

static uint64_t philox_next64(philox_t* s) {
  if (s->pos < 4) return s->buf[s->pos++];
  for (int i = 0; i < 4; ++i)
    if (++s->ctr[i] != 0) break; /* counter carry */
  philox_block(s);
  s->pos = 1;
  return s->buf[0];
}

static uint32_t philox_next32(philox_t* s) {
  if (s->has32) {
    s->has32 = 0;
    return s->half;
  }
  uint64_t v = philox_next64(s);
  s->has32 = 1;
  s->half = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

/* uniform integer in [0, n) for 1 <= n <= 2^32 - 1: Lemire's method as numpy */
static uint32_t bounded32(philox_t* s, uint32_t n) {
  uint64_t m = (uint64_t)philox_next32(s) * n;
  uint32_t lo = (uint32_t)m;
  if (lo < n) {
    uint32_t t = (uint32_t)(-n) % n;
    while (lo < t) {
      m = (uint64_t)philox_next32(s) * n;
      lo = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* indptr[n+1], indices[2 m (n-m)]; state13 = ctr[4] key[2] buf[4] pos has32 half */
int oracle_synth_powerlaw_csr(int64_t n, int64_t m, uint64_t key0, uint64_t key1,
                              int64_t* indptr, int32_t* indices, uint64_t* state13) {
  if (m < 1 || n <= m || 2 * m * (n - m) >= 0x7FFFFFFFLL) return -1;
  philox_t s;
  memset(&s, 0, sizeof s);
  s.key[0] = key0;
  s.key[1] = key1;
  s.pos = 4;
  const int64_t nnew = n - m;
  int32_t* att = malloc(sizeof(int32_t) * m * nnew); /* att[(v-m)*m + i]: targets of v */
  int32_t* pool = malloc(sizeof(int32_t) * 2 * m * nnew);
  int32_t* last = malloc(sizeof(int32_t) * n); /* last new node that picked t */
  int32_t* tg = malloc(sizeof(int32_t) * m);
  if (!att || !pool || !last || !tg) return -2;
  for (int64_t i = 0; i < n; ++i) last[i] = -1;
  for (int64_t i = 0; i < m; ++i) tg[i] = (int32_t)i;
  int64_t plen = 0;
  for (int64_t v = m; v < n; ++v) {
    memcpy(att + (v - m) * m, tg, sizeof(int32_t) * m);
    memcpy(pool + plen, tg, sizeof(int32_t) * m);
    for (int64_t i = 0; i < m; ++i) pool[plen + m + i] = (int32_t)v;
    plen += 2 * m;
    if (v == n - 1) break;
    int64_t got = 0;
    while (got < m) {
      /* one rng.integers(0, plen, size=m) call draws all m values first */
      uint32_t draws[64];
      uint32_t* dr = m <= 64 ? draws : malloc(sizeof(uint32_t) * m);
      for (int64_t i = 0; i < m; ++i) dr[i] = bounded32(&s, (uint32_t)plen);
      for (int64_t i = 0; i < m && got < m; ++i) {
        int32_t t = pool[dr[i]];
        if (last[t] != (int32_t)v) {
          last[t] = (int32_t)v;
          tg[got++] = t;
        }
      }
      if (dr != draws) free(dr);
    }
    qsort(tg, (size_t)m, sizeof(int32_t), cmp_i32);
  }
  /* symmetric CSR: row u = {targets of u} U {new nodes that picked u},
   * ascending (np.lexsort((dst, src))) */
  int64_t* deg = calloc((size_t)n, sizeof(int64_t));
  for (int64_t v = m; v < n; ++v) {
    deg[v] += m;
    for (int64_t i = 0; i < m; ++i) deg[att[(v - m) * m + i]] += 1;
  }
  indptr[0] = 0;
  for (int64_t u = 0; u < n; ++u) indptr[u + 1] = indptr[u] + deg[u];
  int64_t* fillp = malloc(sizeof(int64_t) * n);
  for (int64_t u = 0; u < n; ++u) fillp[u] = indptr[u];
  for (int64_t v = m; v < n; ++v) /* u < v picked by v: appended in v order */
    for (int64_t i = 0; i < m; ++i) {
      int32_t u = att[(v - m) * m + i];
      indices[fillp[u]++] = (int32_t)v;
      indices[fillp[v]++] = u;
    }
  for (int64_t u = 0; u < n; ++u)
    qsort(indices + indptr[u], (size_t)(indptr[u + 1] - indptr[u]), sizeof(int32_t), cmp_i32);
  if (state13) {
    for (int i = 0; i < 4; ++i) state13[i] = s.ctr[i];
    state13[4] = s.key[0];
    state13[5] = s.key[1];
    for (int i = 0; i < 4; ++i) state13[6 + i] = s.buf[i];
    state13[10] = (uint64_t)s.pos;
    state13[11] = (uint64_t)s.has32;
    state13[12] = (uint64_t)s.half;
  }
  free(att);
  free(pool);
  free(last);
  free(tg);
  free(deg);
  free(fillp);
  return 0;
}

int oracle_partition_edgecut(int64_t n, const int64_t* indptr, const int32_t* indices, int32_t k,
                             int64_t* owner) {
  if (k < 1 || k > 4096) return -1;
  const double cap = ceil(1.05 * (double)n / (double)k);
  int64_t* sizes = calloc((size_t)k, sizeof(int64_t));
  int64_t* cnt = calloc((size_t)k, sizeof(int64_t));
  double* score = malloc(sizeof(double) * k);
  uint8_t* seen = calloc((size_t)n, 1);
  int64_t* q = malloc(sizeof(int64_t) * n);
  if (!sizes || !cnt || !score || !seen || !q) return -2;
  for (int64_t i = 0; i < n; ++i) owner[i] = -1;
  int64_t head = 0, tail = 0, next_start = 0;
  for (int64_t it = 0; it < n; ++it) {
    if (head == tail) {
      while (seen[next_start]) ++next_start;
      q[tail++] = next_start;
      seen[next_start] = 1;
    }
    const int64_t v = q[head++];
    memset(cnt, 0, sizeof(int64_t) * k);
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
      const int64_t o = owner[indices[e]];
      if (o >= 0) cnt[o] += 1;
    }
    double best = -INFINITY;
    for (int p = 0; p < k; ++p) {
      score[p] = (double)sizes[p] >= cap ? -INFINITY
                                         : (double)cnt[p] * (1.0 - (double)sizes[p] / cap);
      if (score[p] > best) best = score[p];
    }
    int pick = -1;
    for (int p = 0; p < k; ++p) /* first of the least-loaded among the maxima */
      if (score[p] == best && (pick < 0 || sizes[p] < sizes[pick])) pick = p;
    owner[v] = pick;
    sizes[pick] += 1;
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
      const int32_t u = indices[e];
      if (!seen[u]) {
        seen[u] = 1;
        q[tail++] = u;
      }
    }
  }
  free(sizes);
  free(cnt);
  free(score);
  free(seen);
  free(q);
  return 0;
}
