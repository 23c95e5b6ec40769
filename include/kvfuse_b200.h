/*
 * kvfuse_b200.h -- C ABI of the B200 (sm_100a) KV-block fusion library.
 *
 * This is the drop-in boundary for the reference's fusion hot path
 * (/root/reference/pkg/src/kvfuse). The reference is pure Python/numpy; its
 * "FFI" for this path is the Python call surface
 *   fuse_batch  (fusion.py:360)   fuse_chunks (fusion.py:377)
 *   fast_fusion (fusion.py:339)   refold      (core.py:285)
 *   paged_attention (attention.py:58)
 * which paper_2601_03067_b200/ mirrors and implements on top of the entry
 * points below via ctypes (see INTEGRATION.md for the binding stub).
 *
 * Conventions
 *  - Every pointer named *_dev / pool / norms / table ... is a DEVICE pointer
 *    (cudaMalloc / torch CUDA storage). Host pointers are named *_host.
 *  - `stream` is a cudaStream_t passed as void*. All entry points are
 *    stream-ordered and asynchronous unless documented otherwise.
 *  - dtype codes: 0 = float64, 1 = float32, 2 = bfloat16. "Acc" buffers
 *    (norms, scales) are float64 for a float64 pool and float32 otherwise.
 *  - Pool layout: (L, NB, t, h, d) C-order; NB = B*p physical blocks per
 *    layer (reference cache (L, B, p, t, h, d), core.py:54-76). head_mode 0 =
 *    "folded" (unit = layer; block vector = t*h*d entries, core.py:128),
 *    1 = "per_head" (unit = layer*h + head; vector = t*d entries).
 *  - Status codes: KVF_OK, or an error whose message kvf_last_error()
 *    returns (thread-local). The Python layer maps them to the reference's
 *    exception classes (errors.py:4-50).
 */
#ifndef KVFUSE_B200_H
#define KVFUSE_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define KVF_OK 0
#define KVF_ERR_INVALID 1    /* -> ConfigError / InvalidCacheError */
#define KVF_ERR_ALIGNMENT 2  /* -> AlignmentError                  */
#define KVF_ERR_CORRUPTION 3 /* -> CorruptionError                 */
#define KVF_ERR_CUDA 4       /* CUDA runtime / launch failure      */

#define KVF_PATH_AUTO 0
#define KVF_PATH_SIMT 1  /* CUDA-core similarity (f64 / f32 / bf16)           */
#define KVF_PATH_TC 2    /* tcgen05 + TMEM + TMA similarity (bf16 pools only) */
#define KVF_PATH_TC_WIDE 3 /* tcgen05, 512 x 256 tile per CTA pair (one TMEM
                              accumulator; nsplit == 1, staged or direct rows) */
/* OR-ed into kvf_similarity_select's path (KVF_PATH_TC, bf16 pool, nsplit == 1, direct
 * rows; folded or per-head units): the launch computes the key norm of every row it streams
 * from the shared-memory stages (the tree's first level, where each block is an operand
 * row of exactly one tile) and writes knorm and fusable = (knorm > 0) itself -- replaces
 * the K pass of kvf_block_norms (core.py:115-119) with no extra HBM read. */
#define KVF_SIM_WRITE_NORMS 0x100
/* OR-ed into kvf_similarity_select's path (KVF_PATH_TC, direct rows): a level whose merges
 * all have <= 128 blocks per side runs two merges per tile on the diagonal of the CTA
 * pair's 256 x 256 product -- tile k = merges 2k (CTA 0) and 2k + 1 (CTA 1), tiles int32
 * [ceil(nm / 2)][3] = {2k, 0, 0}; the tile's 16 partials slots are merge 2k's first 8 and
 * merge 2k + 1's last 8 (kvf_level_stats tile offsets (m / 2) * 16 + (m % 2) * 8). Each CTA
 * streams only its own merge's rows: half the operand bytes of one merge per tile. */
#define KVF_SIM_PAIRED 0x200

/* Library identity and last error (thread-local). */
const char* kvf_last_error(void);
int kvf_version(void);

/* Validation of a cache (PagedKvCache.__post_init__, core.py:73-74):
 * adds the number of NaN/Inf entries of data[0:n] to *count_dev. */
int kvf_count_nonfinite(const void* data, int dtype, int64_t n,
                        unsigned long long* count_dev, void* stream);

/* K1 -- per-block L2 norms (replaces _split_norm_direction, core.py:115-119).
 * norms: Acc[U][NB], U = L (folded) or L*h (per_head). */
int kvf_block_norms(const void* pool, int dtype, int64_t L, int64_t NB, int t,
                    int h, int d, int head_mode, void* norms, void* stream);

/* Fusion state for U units (replaces _Engine.__init__, fusion.py:208-228, and
 * BlockTable.identity, core.py:191-201): fusable = knorm > 0, alive = 1,
 * absorber = NONE, table = identity, refcount = 1. knorm == NULL leaves fusable
 * to the level-1 similarity launch with KVF_SIM_WRITE_NORMS. */
int kvf_state_init(int dtype, int64_t U, int64_t NB, const void* knorm,
                   uint8_t* fusable, uint8_t* alive, int32_t* absorber,
                   int32_t* table, int32_t* refcount, void* stream);

/* Similarity tile shape used by a path (tiles passed to
 * kvf_similarity_select must be built with it) and the number of partials
 * slots each tile writes (the tcgen05 path runs one tile per CTA pair). */
int kvf_sim_tile_shape(int dtype, int head_mode, int path, int* tile_m,
                       int* tile_n, int* partials_per_tile);

/* K2 + K3 -- similarity + first-match selection for every merge of one tree
 * level (replaces fusion.py:244-265):
 *   sim(i, j) = <x_i, x_j> / (|x_i| |x_j|) over alive, fusable blocks,
 *   absorber[j] = min { i in left : sim(i, j) > thr }   (atomicMin).
 * merges : int32[nm][3] block ranges {left_begin, split, right_end};
 * tiles  : int32[nt][3] {merge, i0, j0} offsets inside the merge;
 * partials (out): double[nU][nt * partials_per_tile][5] = {count, sum,
 *   sumsq, min, max} of sim (kvf_level_stats takes the same scaled counts);
 * samples (optional, out): double, samples[(u-u0)*sample_stride +
 *   sample_off[m] + il*right_n + jl] = sim or NaN for masked pairs (compacted
 *   launches leave dead pairs untouched: pre-fill with NaN).
 * Compaction (tcgen05 path only): live/rank from kvf_alive_rank -- tiles
 * then index the merge's alive blocks only. With staged (kvf_stage_rows) the
 * operands stream from the staged dense rows; with staged == NULL (folded
 * units) they are gathered straight from the pool with TMA gather4.
 * Re-score (tcgen05 path): pairs with |sim - thr| <= rescore_band are queued
 * (int32[4 * (rescore_cap + 1)], entries then the count) and decided from a
 * float64 recomputation in the same call; NULL / 0 disables it.
 * filter (float32 pools): bf16 copy of the pool (kvf_convert_rows) that the
 *   tensor cores read; the re-score reads the float32 pool.
 * shadow / sidx (exact mode, kvf_merge_groups): the re-score reads a fused
 *   key from its fp32 shadow row instead of the rounded pool block.
 * nsplit > 1 (tcgen05 path): split-K over each tile's k-steps for levels with
 *   few, long-K tiles; split_part = float[nt * nU * nsplit * 65536] partials,
 *   split_count = int32[nt * nU * 2] zeroed once (left at zero on exit). */
int kvf_similarity_select(const void* pool_k, int dtype, int64_t L, int64_t NB,
                          int t, int h, int d, int head_mode, int64_t u0,
                          int64_t nU, const void* knorm, const uint8_t* fusable,
                          const uint8_t* alive, int32_t* absorber,
                          const int32_t* merges, int nm, const int32_t* tiles,
                          int nt, double thr, double* partials, double* samples,
                          const int64_t* sample_off, int64_t sample_stride,
                          const int32_t* live, const int32_t* rank,
                          const void* staged, int32_t* rescore_queue,
                          int64_t rescore_cap, double rescore_band,
                          const void* filter, const float* shadow,
                          const int32_t* sidx, int nsplit, float* split_part,
                          int32_t* split_count, int path, void* stream);

/* bf16 operand copy of a float32 pool for the tcgen05 similarity: every
 * vector (level_ws == NULL) or the key absorbers of the current level. */
int kvf_convert_rows(const void* src, int src_dtype, void* dst, int64_t L,
                     int64_t NB, int t, int h, int d, int head_mode,
                     int32_t* level_ws, void* stream);

/* Ascending alive list live[U][NB], exclusive rank[U][NB + 1] (number of
 * alive blocks before each id) and count[U] for units [u0, u0 + nU). */
int kvf_alive_rank(int64_t u0, int64_t nU, int64_t NB, const uint8_t* alive,
                   int32_t* live, int32_t* rank, int32_t* count, void* stream);

/* Staged copy of the alive K rows: staged[(u - u0) * NB + k][0:r] =
 * vector(u, live[u][k]) for k < count[u] (bf16 pools). */
int kvf_stage_rows(const void* pool, int dtype, int64_t L, int64_t NB, int t,
                   int h, int d, int head_mode, int64_t u0, int64_t nU,
                   const int32_t* live, const int32_t* count, void* staged,
                   void* stream);

/* Level workspace: int32[kvf_level_ws_ints(U * NB)], zero-filled once before
 * the first level (kvf_remap restores the zero invariant for the next one).
 * Holds member counts / segments / ids per absorber and the absorber list. */
int64_t kvf_level_ws_ints(int64_t n_total);

/* Per-merge statistics of one level + member lists (MergeRecord,
 * fusion.py:93-110, 273-281). stats: double[nU][nm][8] = {left_blocks,
 * right_blocks, fused_count, n, sum, sumsq, min, max}. For every absorber l
 * of the level, the ascending ids j with absorber[j] == l (the `rids` of
 * fusion.py:256-259) are written to the level workspace. */
int kvf_level_stats(int64_t u0, int64_t nU, int64_t U, int64_t NB,
                    const uint8_t* fusable, const uint8_t* alive,
                    const int32_t* absorber, const int32_t* merges, int nm,
                    const int32_t* tile_off, int nt, const double* partials,
                    double* stats, int32_t* level_ws, void* stream);

/* K4 -- in-place block merge (replaces fusion.py:259-261, _unit 285-287):
 * for each absorber l, dir = unit(dir_l + sum_{j: absorber[j]=l} dir_j) for K
 * and the same indices for V (members summed in ascending order); written
 * back as s_home * dir with s_home the home slot's original norm (1 if
 * zero); stored norm recomputed from the rounded values. which: 1 = K only,
 * 2 = V only, 3 = both.
 * Exact-decision mode (bf16 pools; shadow != NULL): the key directions follow
 * the reference's float64 ones -- members fused earlier are read from their
 * fp32 unit shadow row shadow[sidx[j]] (original blocks as x / |x|), and each
 * key absorber's new unit direction is written to its row (taken from
 * *shadow_count on its first fusion, up to shadow_cap; overflowing absorbers
 * keep sidx = -1 and the count exceeds the cap); the pool still receives
 * bf16(s_home * dir). r <= 16384. which | KVF_MERGE_LAST_LEVEL: the tree's last
 * level -- shadow rows are still read but no longer written (nothing reads them
 * after the last merge). */
#define KVF_MERGE_LAST_LEVEL 0x10
int kvf_merge_groups(void* pool_k, void* pool_v, int dtype, int64_t L,
                     int64_t NB, int t, int h, int d, int head_mode, void* knorm,
                     void* vnorm, const void* orig_knorm, const void* orig_vnorm,
                     int32_t* level_ws, int which, float* shadow,
                     int64_t shadow_cap, int32_t* sidx, int32_t* shadow_count,
                     void* stream);

/* K5 -- block-table remap + refcounts (replaces BlockTable.redirect,
 * core.py:217-227, and alive[rid] = False, fusion.py:262-264); resets the
 * level workspace counters. */
int kvf_remap(int64_t u0, int64_t nU, int64_t U, int64_t NB,
              const int32_t* absorber, int32_t* table, int32_t* refcount,
              uint8_t* alive, int32_t* level_ws, void* stream);

/* Finalize: per-slot scales k_scale[s] = orig_knorm[s] / knorm[table[s]]
 * (same for V; refold semantics core.py:303-304), ascending live list
 * (FusedLayer.phys_ids, fusion.py:316) and ascending free list per unit.
 * live_ids == NULL: scales only (after a BlockTable mutation). */
int kvf_finalize(int dtype, int64_t u0, int64_t nU, int64_t NB,
                 const void* orig_knorm, const void* orig_vnorm,
                 const void* knorm, const void* vnorm, const int32_t* table,
                 const uint8_t* alive, void* k_scale, void* v_scale,
                 int32_t* live_ids, int32_t* live_count, int32_t* free_ids,
                 int32_t* free_count, void* stream);

/* Device audit (BlockTable.audit, core.py:232-241): *bad_dev (int32, zeroed
 * here) becomes nonzero if refcount != histogram(table), a slot points at a
 * dead or out-of-range block, or a live block has refcount 0.
 * scratch: int32[U*NB]. */
int kvf_table_audit(int64_t U, int64_t NB, const int32_t* table,
                    const int32_t* refcount, const uint8_t* alive,
                    int32_t* scratch, int32_t* bad_dev, void* stream);

/* BlockTable.redirect (core.py:217-227) for one unit; *bad_dev set when
 * from/to is dangling. */
int kvf_table_redirect(int64_t NB, int32_t* table, int32_t* refcount,
                       uint8_t* alive, int32_t from_phys, int32_t to_phys,
                       int32_t* bad_dev, void* stream);

/* Gather vectors of unit u: out[k][:] = c_k * x_{ids[k]} (Acc dtype) with
 * c_k = (norms ? 1/norms[u][ids[k]] : 1) * (scales ? scales[k] : 1).
 * norms -> FusedLayer.directions (core.py:244-258); ids = table row and
 * scales = k_scale row -> refold of one unit (core.py:298-304). */
int kvf_gather_vectors(const void* pool, int dtype, int64_t L, int64_t NB,
                       int t, int h, int d, int head_mode, int64_t u,
                       const int32_t* ids, int64_t n, const void* norms,
                       const void* scales, void* out, void* stream);

/* refold (core.py:285-305) of one layer: out[s][tok][hh][:] =
 * scale[u][s] * pool[layer][table[u][s]][tok][hh][:] with u = layer (folded)
 * or layer*h + hh (per_head). out: Acc[NB][t][h][d]. */
int kvf_refold(const void* pool, int dtype, int64_t L, int64_t NB, int t,
               int h, int d, int head_mode, int64_t layer,
               const int32_t* table, const void* scale, void* out,
               void* stream);

/* K6 -- paged decode attention over the fused cache (attention.py:58-80
 * generalised to a batch, GQA and per-slot norm scales):
 *   for request b, query head qh (kv head qh / (Hq/h)):
 *   out = softmax(sm_scale * K q) V with K/V rows read through table/scales.
 * q: Acc-or-bf16 [B][Hq][d] (q_dtype), out: float32 [B][Hq][d] (float64
 * when dtype == 0), lse: same dtype [B][Hq], probs (optional, small
 * problems): [B][Hq][p*t]. seq_blocks (optional) int32[B] valid blocks per
 * request. workspace: kvf_decode_workspace_size() bytes. */
int64_t kvf_decode_workspace_size(int dtype, int64_t B, int Hq, int d,
                                  int64_t p_blocks, int t);
int kvf_paged_decode(const void* q, int q_dtype, const void* pool_k,
                     const void* pool_v, int dtype, int64_t L, int64_t NB,
                     int t, int h, int d, int head_mode, int64_t layer,
                     const int32_t* table, const void* k_scale,
                     const void* v_scale, int64_t B, int64_t p_blocks,
                     const int32_t* seq_blocks, int Hq, double sm_scale,
                     void* out, void* lse, void* probs, void* workspace,
                     int64_t workspace_bytes, void* stream);

/* Chunked-prefill attention over a CFF-fused context with computation reuse
 * (PAPER.md:57-59, 130-131): the queries of chunk `chunk`
 * (bf16 [B][chunk_blocks*t][Hq][d]) attend to the logical keys of chunks
 * 0..chunk-1 (all visible) and causally to the chunk's own keys, every slot
 * read through table / k_scale / v_scale (core.py:303-304). order: int32
 * [B][p_blocks] each request's positions sorted by physical block (the decode
 * schedule's `order`). dedup = 1: S = Q K_P^T and P V_P once per physical
 * block P with the slots' scales folded in; dedup = 0: once per slot.
 * out: float32 [B][chunk_blocks*t][Hq][d]. bf16, folded, t = 16, Hq/h | 8.
 * path: 0 auto (tcgen05 when d = 128), 1 mma.sync kernel, 2 tcgen05 kernel
 * (S and P V on the tensor cores, accumulators in TMEM, two query tiles per
 * CTA, 4 units = 64 keys per softmax step). */
int kvf_chunk_prefill(const void* q, const void* pool_k, const void* pool_v,
                      int dtype, int64_t L, int64_t NB, int t, int h, int d,
                      int head_mode, int64_t layer, const int32_t* table,
                      const void* k_scale, const void* v_scale,
                      const int32_t* order, int64_t B, int64_t p_blocks,
                      int chunk_blocks, int chunk, int Hq, double sm_scale,
                      int dedup, int path, void* out, void* stream);

/* Percentile mode of the threshold controller on the device (fusion.py:418-437,
 * SURVEY §8f rank 3): *out = np.quantile(x, q) (numpy's default 'linear'
 * method) over the non-NaN entries of nparts float64 device segments
 * parts[i][0:lens[i]] (host arrays of device pointers / lengths; e.g. the
 * per-level sample rows of a fusion run, masked pairs are NaN). NaN when no
 * sample is valid. Exact: 8-pass radix select on order-preserving keys.
 * workspace: kvf_quantile_ws_bytes() device bytes. */
int64_t kvf_quantile_ws_bytes(void);
int kvf_quantile(const void* const* parts, const int64_t* lens, int nparts,
                 double q, double* out, void* workspace,
                 int64_t workspace_bytes, void* stream);

/* Compaction of a fused layer (the reference's FusedCache storage: live
 * blocks only, ascending physical id, core.py:246-270 / fusion.py:318-327):
 * kvf_alive_rank gives the ascending live ids and the exclusive alive rank of
 * every block, kvf_stage_rows copies the live rows densely (bf16, folded), and
 * kvf_remap_ids maps slot tables and decode-schedule ids to dense rows:
 * out[i] = map[ids[i]] for 0 <= ids[i] < map_len, else -1. */
int kvf_remap_ids(const int32_t* ids, int64_t n, const int32_t* map,
                  int64_t map_len, int32_t* out, void* stream);

/* Sharing-aware decode schedule (PAPER.md:56, 130-131:
 * a fused block shared by several requests should be fetched once). For
 * serving batches it replaces the request-major loop of attention.py:58-80;
 * results equal kvf_paged_decode up to fp32 summation order (softmax is
 * permutation invariant). Per layer and head unit hu (nh = h units when
 * head_mode == 1, else 1), with nit = ceil(p_blocks / item_blocks):
 *   order int32 [nh][B][p_blocks]  request b's positions sorted by physical
 *                                  block (-1 past seq_blocks[b])
 *   meta  int32 [nh][B*nit]        b*nit + k of each item, items ascending by
 *                                  first physical block; n_items[hu] valid
 *   phys  int32 [nh][B*nit][item_blocks] physical block of each item slot
 *                                  (-1 = padding); ks / vs float, same shape:
 *                                  the slots' K / V scales
 * n_repeats (optional, int32[1]): slots that repeat the previous slot's block
 * inside an item (runs of a block the request references several times, e.g.
 * after CFF); nonzero -> pass dedup = 1 to kvf_paged_decode_sched.
 * item_blocks: 8 or 16 (kvf_decode_schedule_item_blocks() = tuned default).
 * workspace: kvf_decode_schedule_ws_ints() int32 words. Rebuild the schedule
 * after any change of the layer's table or scales. */
int kvf_decode_schedule_item_blocks(void);
int64_t kvf_decode_schedule_ws_ints(int head_mode, int h, int64_t NB, int64_t B,
                                    int64_t p_blocks, int item_blocks);
int kvf_decode_schedule(const int32_t* table, const void* k_scale,
                        const void* v_scale, int64_t L, int64_t NB, int t,
                        int h, int d, int head_mode, int64_t layer, int64_t B,
                        int64_t p_blocks, const int32_t* seq_blocks,
                        int item_blocks, int32_t* order, int32_t* meta,
                        int32_t* phys, float* ks, float* vs, int32_t* n_items,
                        int32_t* n_repeats, int32_t* workspace,
                        int64_t workspace_ints, void* stream);
/* K6 over a schedule: persistent warps sweep the items head by head, so
 * requests sharing a fused block read it within one L2 window; with dedup, a
 * run of slots on one block is loaded once, S = K q^T is computed once and
 * reused with each slot's scale, and P V runs once on the scale-weighted sum
 * of the run's probabilities (computation reuse). bf16 pools,
 * d in {64, 128}, t | 32. Same q / out / lse contract as kvf_paged_decode
 * (no probability output); workspace >= B*Hq*nit*(d+2)*4 bytes. */
int kvf_paged_decode_sched(const void* q, int q_dtype, const void* pool_k,
                           const void* pool_v, int dtype, int64_t L,
                           int64_t NB, int t, int h, int d, int head_mode,
                           int64_t layer, const int32_t* table,
                           const void* k_scale, const void* v_scale, int64_t B,
                           int64_t p_blocks, const int32_t* seq_blocks, int Hq,
                           double sm_scale, void* out, void* lse,
                           int item_blocks, const int32_t* meta,
                           const int32_t* phys, const float* ks,
                           const float* vs, const int32_t* n_items, int dedup,
                           void* workspace, int64_t workspace_bytes,
                           void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* KVFUSE_B200_H */
