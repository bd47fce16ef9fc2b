/*
 * rapidgnn_b200.h — C ABI of the B200 hot path for RapidGNN's data path
 * (reference: gnnpipe, /root/reference/pkg/src/gnnpipe).
 *
 * The reference is pure Python/numpy and has no FFI of its own: its
 * boundary is the module API re-exported by gnnpipe/__init__.py:5-19.  Each
 * entry point below is the device kernel behind one of those functions;
 * paper_2505_10806_b200/ (Python, ctypes) mirrors the reference API on top
 * of it (see INTEGRATION.md for the binding a maintainer would add).
 *
 * Conventions
 *   - every function returns 0 (RG_OK) or a negative RG_ERR_* code and never
 *     throws; rg_last_error() returns a thread-local message for the last
 *     failure on the calling thread;
 *   - pointers named d_* are device pointers, h_* host pointers; all device
 *     buffers are caller-owned, nothing allocates behind the caller's back;
 *   - work is enqueued on the caller's stream (cudaStream_t passed as void*),
 *     no entry point synchronises the host, so every call is capturable in a
 *     CUDA graph;
 *   - node ids are int32 on device (every configured graph has n < 2^31),
 *     CSR row pointers int64;
 *   - "group" = G mini-batches processed by one launch; per-batch buffers are
 *     G fixed-capacity slots laid out back to back (slot b at b * cap).
 */
#ifndef RAPIDGNN_B200_H
#define RAPIDGNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RG_OK 0
#define RG_ERR_INVALID (-1)     /* bad argument (maps to ValueError)          */
#define RG_ERR_CUDA (-2)        /* CUDA runtime / launch failure              */
#define RG_ERR_UNSUPPORTED (-3) /* shape outside what the kernels support     */
#define RG_ERR_NOT_OWNED (-4)   /* pull for an id the shard does not own      */

/* route word of a node, one uint32 per node:
 *   bits 28..31 = source kind: partition id 0..14, or RG_KIND_CACHE
 *   bits  0..27 = row index inside that partition's shard / the cache   */
#define RG_KIND_SHIFT 28
#define RG_KIND_CACHE 15u
#define RG_ROW_MASK 0x0FFFFFFFu
#define RG_ROUTE_INVALID 0xFFFFFFFFu
#define RG_MAX_PARTS 15

/* per-batch bundle counters written by rg_gather_bundle (uint32 each)   */
#define RG_CNT_LOCAL 0
#define RG_CNT_HIT 1
#define RG_CNT_FALLBACK 2
#define RG_CNT_OWNER_MASK 3 /* bit q set <=> >=1 fallback row owned by q */
#define RG_CNT_BAD 4        /* rows whose route was RG_ROUTE_INVALID     */
#define RG_CNT_PEER 5       /* fallback rows read from a peer GPU's shard */
#define RG_NCOUNTERS 8

const char* rg_last_error(void);
int rg_abi_version(void);
/* 1 if the library was built for sm_100a and a device is usable, else 0 */
int rg_device_ok(void);

/* ---- L1 randomness (rng.py:28-62) ----------------------------------- */
/* out[i] = mix64(in[i])                              rng.py:28-44       */
int rg_mix64(const uint64_t* d_in, uint64_t* d_out, int64_t n, void* stream);
/* out[j] = mix64((j+1)*GOLDEN + master), j < count  rng.py:47-50       */
int rg_stream_keys(uint64_t master, int64_t count, uint64_t* d_out, void* stream);

/* ---- L2 sampling (sampler.py:86-152) -------------------------------- */
/* Seeds of batches i0..i0+G-1 of an epoch permutation (chunks of
 * batch_size, last one partial; sampler.py:57) into d_seeds (G x seed_cap)
 * / d_nseeds, and rng[b] = mix64(s0 ^ (epoch<<32 | i0+b)) (sampler.py:40).*/
int rg_fill_seeds(const int32_t* d_perm, int64_t n_perm, int32_t batch_size, int64_t i0,
                  int32_t G, int32_t* d_seeds, int32_t* d_nseeds, int32_t seed_cap, uint64_t s0,
                  int64_t epoch, uint64_t* d_rng, void* stream);

/* Level-0 frontier: mark the seeds of every batch in its bitmap.
 * d_seeds: G x seed_cap int32, d_nseeds: G int32; d_bm: G x nwords.
 * (np.unique(seeds), sampler.py:138, is the compaction that follows.)  */
int rg_mark_seeds(const int32_t* d_seeds, const int32_t* d_nseeds, int32_t G, int32_t seed_cap,
                  uint32_t* d_bm, int64_t nwords, void* stream);

/* One expansion step d for G batches (sampler.py:86-113 + 145-148).
 * For frontier node j of batch b (v = front[b*cap_in + j]):
 *   take = min(deg v, fanout); the take positions with the smallest
 *   SplitMix64 keys mix(nk + (p+1)G), nk = mix((v+1)G ^ s_d),
 *   s_d = mix(rng_seed[b] ^ (level+1)G), are selected; their neighbour ids,
 *   ascending, go to ell[b*cap_in*fanout + j*fanout + r], r < take, and
 *   cnt[b*cap_in + j] = take.  Each selected neighbour id is OR-ed into the
 *   batch bitmap, so after the step bm = F_d U src (sampler.py:148).
 * d_slow: scratch of 1 + G*cap_in int32, required only when fanout > 32
 * (rows with take > 32 go to a CTA-per-row path); fanout <= 4096.
 * d_meta: scratch of (G*cap_in + 1) x 16 B: a lane-parallel pass first
 * stores (row start, degree, id) of every frontier node (int4 per slot) so
 * the per-node warps skip the front -> indptr chain; the last record holds
 * the launch-wide work-queue counter.
 * sorted_rows != 0 promises every CSR row is ascending (true for the
 * reference's generator and from_edge_list): selected positions are then
 * emitted in position order without a sort.                            */
int rg_sample_level(const int64_t* d_indptr, const int32_t* d_indices, int64_t n,
                    int32_t G, const int32_t* d_front, int64_t cap_in, const int32_t* d_nfront,
                    int32_t fanout, int32_t level, const uint64_t* d_rng_seed, int32_t* d_ell,
                    int32_t* d_cnt, uint32_t* d_bm, int64_t nwords, int32_t* d_slow,
                    int32_t* d_meta, int32_t sorted_rows, int32_t prng, void* stream);

/* PRNG variants (not in the reference; semantics in rg_prng.cuh and
 * DESIGN.md §10): prng = 0 SplitMix64 keys (reference), 1 pcg32,
 * 2 sfc64, 3 xoshiro256++ (passed to rg_sample_level).  Host forms for
 * known-answer tests: raw stream seeded with (k0, k1), and the Floyd
 * position draw of one node (positions in draw order).                 */
#define RG_PRNG_SPLITMIX 0
#define RG_PRNG_PCG32 1
#define RG_PRNG_SFC64 2
#define RG_PRNG_XOSHIRO256PP 3
int rg_prng_raw(int32_t kind, uint64_t k0, uint64_t k1, int64_t count, uint64_t* h_out);
int rg_prng_select(int32_t kind, uint64_t nk, uint64_t sd, int32_t D, int32_t T, int32_t* h_pos);

/* Sorted-unique compaction of G bitmaps (np.unique / np.union1d).
 * Writes ascending ids of set bits to out[b*cap_out ...], count to
 * d_nout[b].  d_chunk: G x rg_bitmap_chunks(nwords) int32 scratch.
 * If d_wpre != NULL it also receives the exclusive popcount prefix per
 * word (G x nwords), i.e. rank(v) = wpre[v>>5] + popc(bm & lowmask). */
int64_t rg_bitmap_chunks(int64_t nwords);
/* kernel launches one rg_bitmap_compact call makes (2, or 3 when the chunk
 * totals get their own scan kernel: more than 256 chunks)               */
int rg_bitmap_compact_launches(int64_t nwords);
int rg_bitmap_compact(const uint32_t* d_bm, int64_t nwords, int32_t G, int32_t* d_chunk,
                      int32_t* d_out, int64_t cap_out, int32_t* d_nout, int32_t* d_wpre,
                      void* stream);
/* set bit v for every v in ids[0..n) (single bitmap)                   */
int rg_bitmap_set(const int32_t* d_ids, const int32_t* d_n, uint32_t* d_bm, void* stream);

/* ELL block level -> flat (src, dst) edge list in (dst, src) order, as
 * ComputationBlock.edges[d] (sampler.py:145-146).  d_eoff (G x (cap_in+1))
 * receives per-dst offsets, d_nedge[b] the edge count; src/dst written at
 * b*cap_e.  d_chunk: G x rg_scan_chunks(cap_in) scratch.            */
int64_t rg_scan_chunks(int64_t cap);
int rg_ell_to_edges(const int32_t* d_front, const int32_t* d_nfront, int64_t cap_in,
                    const int32_t* d_ell, const int32_t* d_cnt, int32_t fanout, int32_t G,
                    int32_t* d_chunk, int32_t* d_eoff, int32_t* d_src, int32_t* d_dst,
                    int64_t cap_e, int32_t* d_nedge, void* stream);

/* ---- L3 planning (plan.py:108-141) ---------------------------------- */
/* counts[v] += number of the G batch bitmaps holding v (one access per
 * batch appearance, plan.py:117-130 before the remote mask).          */
int rg_count_inputs(const uint32_t* d_bm, int64_t nwords, int32_t G, int64_t n,
                    uint32_t* d_counts, void* stream);
/* candidates: route kind != my_part and counts[v] > 0.
 * hist[c] += 1 for each candidate with count c (c clamped to max_count);
 * d_bm_cand receives the candidate bitmap.                            */
int rg_count_histogram(const uint32_t* d_counts, const uint8_t* d_owner, int32_t my_part,
                       int64_t n, uint32_t* d_hist, int32_t max_count, uint32_t* d_bm_cand,
                       void* stream);
/* threshold split for top_hot (plan.py:133-141): bm_gt = candidates with
 * count > c_star, bm_eq = candidates with count == c_star.             */
int rg_threshold_split(const uint32_t* d_counts, const uint32_t* d_bm_cand, int64_t n,
                       uint32_t c_star, uint32_t* d_bm_gt, uint32_t* d_bm_eq, void* stream);
/* synthetic feature rows for config X (the reference's numpy generator
 * does not scale to 1e8 nodes): row of node ids[i] -> out[i*stride],
 * value(v,c) = Box-Muller normal from mix64(seed ^ ((v*d+c+1)*GOLDEN)).  */
int rg_fill_features(const int32_t* d_ids, int64_t n, int32_t d, int32_t stride, uint64_t seed,
                     float* d_out, void* stream);
/* out[i] = counts[ids[i]] (FrequencyTable.counts)                      */
int rg_gather_counts(const uint32_t* d_counts, const int32_t* d_ids, const int32_t* d_n,
                     int64_t cap, uint32_t* d_out, void* stream);

/* ---- L4 feature path (cache.py, store.py, prefetch.py) -------------- */
/* route[v] = RG_KIND_CACHE<<28 | i for v = hot[i] (i < n_hot), copied from
 * base_route elsewhere: the slot map of FeatureCache (cache.py:54-78). */
int rg_route_with_cache(const uint32_t* d_base_route, int64_t n, const int32_t* d_hot,
                        int64_t n_hot, uint32_t* d_route, void* stream);

/* Feature bundle gather for G batches (prefetch.py:41-88, cache.py:54-78,
 * store.py:66-69,173-196).  Row j of batch b is copied bit-exactly from
 *   bases[kind] + (route[id] & RG_ROW_MASK) * src_stride
 * to out[(b*cap + j) * stride] (stride floats), kind = route >> 28
 * (partition shard or cache).  Classification per row: kind == my_part ->
 * local, kind == RG_KIND_CACHE -> cache hit, else fallback pull from shard
 * `kind`.  d_counters: G x RG_NCOUNTERS uint32, accumulated (caller zeroes).
 * h_bases: host array of 16 device pointers (peer pointers allowed);
 * peer_mask: bit q set if shard q lives on another GPU (RG_CNT_PEER).
 * stride, src_stride: floats, multiples of 4 (16-byte rows); src_stride >=
 * stride lets sources keep sector/line-aligned padded rows (NVLink reads
 * run at full rate on 128-byte-aligned rows) while the bundle stays dense. */
int rg_gather_bundle(const int32_t* d_ids, const int32_t* d_nids, int64_t cap, int32_t G,
                     const uint32_t* d_route, const float* const* h_bases, int32_t src_stride,
                     int32_t stride, int32_t my_part, uint32_t peer_mask, float* d_out,
                     uint32_t* d_counters, void* stream);

/* The same gather for a whole group, driven by the group's input bitmaps
 * instead of id lists: d_bm [G x nwords] (bit j of word w set <=> node
 * 32w+j is in batch b's input set, the sampler's level-L bitmaps) and d_wpre
 * [G x nwords] (rank of node 32w in batch b's sorted set, rg_bitmap_compact's
 * d_wpre); row r of batch b's bundle (the r-th smallest input node) goes to
 * d_out + (b*cap + r)*stride.  A CTA stages each present source row of a
 * 64-id window once in shared memory and writes every batch's run of the
 * window contiguously, so rows shared by the group's batches are read from
 * HBM once per group.  Same route / bases / counters contract as
 * rg_gather_bundle; G <= 128, rows up to ~1.5 K floats.                  */
int rg_gather_window(const uint32_t* d_bm, const int32_t* d_wpre, int64_t nwords, int32_t G,
                     int64_t cap, const uint32_t* d_route, const float* const* h_bases,
                     int32_t src_stride, int32_t stride, int32_t my_part, uint32_t peer_mask,
                     float* d_out, uint32_t* d_counters, void* stream);

/* Copy nbytes from d_src to d_dst on the stream's copy engine (either
 * address may be a peer GPU's IPC mapping): the whole-shard form of the
 * group prefetch for dense groups.                                       */
int rg_copy_bytes(void* d_dst, const void* d_src, int64_t nbytes, void* stream);

/* Cross-GPU group sequence counters for shared sampling (N > 1; DESIGN.md
 * §7).  Every worker samples every batch (train.py:291-311), so the ranks
 * split a group's batches and copy each other's sampled input sets over
 * NVLink.  rg_flag_signal: after the stream's earlier work, publish
 * *d_flag = value (system-scope release).  rg_flag_wait: the stream waits
 * until *d_flag >= value (d_flag may be a peer GPU's IPC mapping; acquire
 * loads); after timeout_ms it gives up and sets *d_status = 1 instead of
 * hanging.                                                                */
int rg_flag_signal(uint64_t* d_flag, uint64_t value, void* stream);
int rg_flag_wait(const uint64_t* d_flag, uint64_t value, int32_t timeout_ms, int32_t* d_status,
                 void* stream);

/* ---- group prefetch of peer rows (north_star item 4) ---
 * bits[w] bit j = the route kind of node 32w+j is in kind_mask.         */
int rg_route_kind_bits(const uint32_t* d_route, int64_t n, uint32_t kind_mask, uint32_t* d_bits,
                       void* stream);
/* out[w] = mask[w] & OR over b < G of bm[b*nwords + w]: the group's input
 * nodes (level-L bitmaps of rg_sample_level) that live on peer shards.  */
int rg_group_union(const uint32_t* d_bm, int64_t nwords, int32_t G, const uint32_t* d_mask,
                   uint32_t* d_out, void* stream);
/* for i < *nids: copy the row of ids[i] (kind/row from its route word)
 * from h_src[kind] to h_dst[kind] at the same row offset (src_stride
 * floats per row, ceil(d/4) 16-B vectors): peer shard -> local shadow.  */
int rg_prefetch_rows(const int32_t* d_ids, const int32_t* d_nids, int64_t cap,
                     const uint32_t* d_route, const float* const* h_src, float* const* h_dst,
                     int32_t src_stride, int32_t d, void* stream);

/* NCCL transport of the group prefetch: rows[i] (rows_stride floats apart,
 * received from its owner) is written to h_dst[kind] + row * dst_stride,
 * kind/row from the route word of ids[i]; ceil(d/4) 16-B vectors.       */
int rg_scatter_rows(const int32_t* d_ids, int64_t n, const uint32_t* d_route,
                    const float* d_rows, int32_t rows_stride, float* const* h_dst,
                    int32_t dst_stride, int32_t d, void* stream);

/* ---- L5 aggregation consumer (model.py:72-81, 126-135) -------------- */
#define RG_DTYPE_F32 0 /* RunConfig.precision "f32" (train.py:117)          */
#define RG_DTYPE_F64 1 /* RunConfig.precision "f64"                          */
/* Positions of one level (model.py:53-55, 74-75, the searchsorted of src
 * and dst into the sorted src frontier), resolved once and shared by the
 * forward and the backward: d_rank is an n_nodes int32 scratch table
 * (rank[src_front[j]] = j), d_epos[t*fanout + r] = position of the r-th
 * sampled neighbour of dst row t (-1 for r >= cnt[t]), d_self_pos[t] =
 * position of dst_front[t].  Frontiers are nested (dst ⊂ src) and every
 * ELL entry is a member of src_front (the sampler's contract).
 * Device counts: every aggregation entry point takes optional device words
 * d_n_src / d_n_dst (e.g. a sampler slot's nfront entries).  When given, the
 * host n_src / n_dst are capacities, the live counts are read on the device
 * (no host sync: the whole training step can be captured in a CUDA graph)
 * and rows past them are padding (no edges, zero outputs).  NULL: the host
 * sizes are the counts.                                                  */
int rg_sage_positions(const int32_t* d_src_front, int64_t n_src, const int32_t* d_dst_front,
                      int64_t n_dst, const int32_t* d_ell, const int32_t* d_cnt, int32_t fanout,
                      int64_t n_nodes, const int32_t* d_n_src, const int32_t* d_n_dst,
                      int32_t* d_rank, int32_t* d_epos, int32_t* d_self_pos, void* stream);
/* mean[t] = (in stored order, sum of h[epos[t, r]]) / max(cnt_t, 1) and
 * self[t] = h[self_pos[t]] (self may be NULL); h rows ldh elements apart,
 * outputs dense [n_dst, H].  dtype RG_DTYPE_F32 / F64; in-order, IEEE
 * divide: bit-exact with the reference's np.add.at / divide.            */
int rg_sage_mean_fwd(int32_t dtype, const void* d_h, int32_t H, int32_t ldh,
                     const int32_t* d_epos, const int32_t* d_self_pos, int64_t n_dst,
                     const int32_t* d_n_dst, const int32_t* d_cnt, int32_t fanout, void* d_mean,
                     void* d_self, void* stream);
/* Transposed edge index for the backward: edges grouped by src position,
 * ascending dst row inside a group (the reference's edge order for that
 * src), any group length.  d_toff n_src+1, d_tdst n_dst*fanout; scratch
 * of rg_sage_transpose_scratch(...) BYTES (-1: sizes out of range).     */
int64_t rg_sage_transpose_scratch(int64_t n_src, int64_t n_dst, int32_t fanout);
int rg_sage_transpose(const int32_t* d_epos, const int32_t* d_cnt, int64_t n_dst, int32_t fanout,
                      int64_t n_src, int32_t* d_toff, int32_t* d_tdst, void* d_scratch,
                      int64_t scratch_bytes, void* stream);
/* Backward scatter (model.py:126-135): dh = 0; dh[self_pos[t]] += dself[t];
 * then for each edge in (dst asc, src asc) order dh[pos(src)] +=
 * dmean[t] / max(cnt_t,1).  Dense [n, H] operands; d_self_of: n_src
 * int32 scratch.                                                        */
int rg_sage_mean_bwd(int32_t dtype, const void* d_dself, const void* d_dmean, int64_t n_dst,
                     int32_t H, const int32_t* d_cnt, const int32_t* d_self_pos,
                     const int32_t* d_toff, const int32_t* d_tdst, int64_t n_src,
                     const int32_t* d_n_src, const int32_t* d_n_dst, int32_t* d_self_of,
                     void* d_dh, void* stream);

/* ---- training-step head and update (model.py:107-146) ---------------
 * rg_softmax_xent: for the live rows r < min(*d_n, cap) of logits [cap, C]
 * (C <= 64, dtype as above): y = labels[front0[r]], nll_r = log(sum_j
 * exp(l_rj - m_r)) - (l_ry - m_r), d_dz[r, j] = (softmax_rj - [j == y]) / n;
 * padding rows get zero gradient; d_nll: cap-element scratch of the same
 * dtype (receives nll_r); *d_loss_acc += (sum_r nll_r) / n as a double,
 * summed in a fixed order (deterministic).
 * Replaces the mean softmax cross-entropy and its gradient of
 * loss_and_grad (model.py:107-124).                                      */
int rg_softmax_xent(int32_t dtype, const void* d_logits, int32_t C, int64_t cap,
                    const int32_t* d_n, const int64_t* d_labels, const int32_t* d_front0,
                    void* d_dz, void* d_nll, double* d_loss_acc, void* stream);
/* rg_sgd_apply: for t < n_tensors (<= 3): w_t[i] -= lr * sum_{c < chunks_t}
 * g_t[c * n_t + i].  The chunk partials are summed in a fixed order: S_k =
 * in-order sum over c = k, k + 8, ... (k < 8), then ((S0 + S1) + (S2 + S3))
 * + ((S4 + S5) + (S6 + S7)); then the reference's rounding: lr * g rounded,
 * then subtracted.  sgd_step, model.py:139-146.                           */
int rg_sgd_apply(int32_t dtype, int32_t n_tensors, void* const* h_w, const void* const* h_g,
                 const int64_t* h_n, const int32_t* h_chunks, double lr, void* stream);

/* ---- host-side graph materialisation (graph.py, partition.py) ------- */
int rg_philox_raw(uint64_t key0, uint64_t key1, int64_t count, uint64_t* h_out);
/* CSR of gnnpipe.graph.synth_powerlaw(n, m, ., ., seed) with the Philox
 * key numpy derives from seed; h_indptr n+1, h_indices 2*m*(n-m).
 * h_state13 (optional) receives the generator state after the attachment
 * loop: counter[4], key[2], buffer[4], buffer_pos, has_uint32, uinteger,
 * so the caller can continue the same numpy stream (features, masks).  */
int rg_synth_powerlaw_csr(int64_t n, int64_t m, uint64_t key0, uint64_t key1, int64_t* h_indptr,
                          int32_t* h_indices, uint64_t* h_state13);
/* gnnpipe.partition.partition_edgecut(g, k).owner                     */
int rg_partition_edgecut(int64_t n, const int64_t* h_indptr, const int32_t* h_indices, int32_t k,
                         int32_t* h_owner);

/* ---- multi-GPU plumbing: CUDA IPC for peer shard pointers ----------- */
/* handle of the allocation holding d_ptr, and d_ptr's offset inside it */
int rg_ipc_handle(const void* d_ptr, uint8_t* h_handle64, int64_t* h_offset);
int rg_ipc_open(const uint8_t* h_handle64, void** d_ptr_out);
int rg_ipc_close(void* d_ptr);
/* single process, several GPUs: current device may read `peer`'s memory  */
int rg_enable_peer(int32_t peer);

#ifdef __cplusplus
}
#endif
#endif /* RAPIDGNN_B200_H */
