// Internal launch interface between the C ABI (kvf_abi.cu) and the kernel
// translation units. Every launcher returns cudaGetLastError() of its launch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"

namespace kvf {

cudaError_t launch_count_nonfinite(const void* data, int dtype, int64_t n,
                                   unsigned long long* count, cudaStream_t s);
cudaError_t launch_block_norms(const void* pool, int dtype, const Geom& g,
                               void* norms, cudaStream_t s);
cudaError_t launch_state_init(int dtype, int64_t U, int64_t NB, const void* knorm,
                              uint8_t* fusable, uint8_t* alive, int32_t* absorber,
                              int32_t* table, int32_t* refcount, cudaStream_t s);

struct SimArgs {
  const void* pool;
  int dtype;
  Geom g;
  int64_t u0, nU;
  const void* knorm;
  const uint8_t* fusable;
  const uint8_t* alive;
  int32_t* absorber;
  const int32_t* merges;
  int nm;
  const int32_t* tiles;
  int nt;
  double thr;
  double* partials;
  double* samples;
  const int64_t* sample_off;
  int64_t sample_stride;
  // compaction (tcgen05 path): ascending alive ids / exclusive alive rank
  // [U][NB + 1] / staged K rows [nU][NB][r] (bf16); all null = direct mode
  const int32_t* live = nullptr;
  const int32_t* rank = nullptr;
  const void* staged = nullptr;
  // near-threshold re-score queue (tcgen05 path): int4 {u, i, j, merge}
  int32_t* resc = nullptr;
  int32_t* resc_count = nullptr;
  int64_t resc_cap = 0;
  double resc_band = 0.0;
  // float32 pools: `pool` is the hi/lo bf16 split copy (2 * L * NB rows, kvf_convert_rows)
  int split3 = 0;
  // split-K over the k-steps of each tile (nsplit > 1): fp32 partials
  // [nt * nU][nsplit][2][256][128] and per-(tile, CTA) arrival counters [nt * nU][2]
  // (zero-initialised once; the kernel leaves them at zero)
  int nsplit = 1;
  float* split_part = nullptr;
  int32_t* split_count = nullptr;
  // wide tile (KVF_PATH_TC_WIDE): 512 x 256 per CTA pair (tiles of kTcTileMWide rows)
  int wide = 0;
  // level 1 only: the launch computes the key norm of every streamed row (knorm written,
  // fusable = knorm > 0) instead of reading them (KVF_SIM_WRITE_NORMS)
  int write_norms = 0;
  // paired small merges (KVF_SIM_PAIRED): tile k holds merges 2k (CTA 0) and 2k + 1 (CTA 1)
  int paired = 0;
};

struct RescoreArgs {
  const void* pool;
  int dtype;
  Geom g;
  int64_t u0;
  const int32_t* resc;
  const int32_t* resc_count;
  int64_t resc_cap;
  double thr;
  int32_t* absorber;
  const int32_t* merges;
  double* samples;
  const int64_t* sample_off;
  int64_t sample_stride;
  const float* shadow = nullptr;  // exact mode: fp32 unit directions of fused keys
  const int32_t* sidx = nullptr;  // [U][NB] shadow slot or -1
};
cudaError_t launch_rescore(const RescoreArgs& a, cudaStream_t s);

constexpr int kSimtTile = 64;
cudaError_t launch_sim_simt(const SimArgs& a, cudaStream_t s);

// tcgen05 path (bf16 only): one 256 x 256 tile per CTA pair (cta_group::2),
// similarity partials written per CTA (2 slots per tile)
constexpr int kMergeLastLevel = 0x10;  // = KVF_MERGE_LAST_LEVEL (include/kvfuse_b200.h)
constexpr int kTcTileM = 256;
constexpr int kTcTileMWide = 512;
constexpr int kTcTileN = 256;
constexpr int kTcPartialsPerTile = 16;  // one moment slot per epilogue warp of the CTA pair
bool tc_supported(const SimArgs& a, const char** why);
cudaError_t launch_sim_tc(const SimArgs& a, cudaStream_t s);

// Per-level workspace shared by level_stats / merge / remap (int32 words):
//   mcnt[n] member count per absorber   mfill[n] scatter cursor per absorber
//   mstart[n] member segment start      members[n] member ids (ascending per absorber)
//   list[n] absorber global ids          count (absorbers), cursor (members)
// n = U * NB (all units). remap re-zeroes mcnt / mfill for the next level.
struct LevelWs {
  int32_t *mcnt, *mfill, *mstart, *members, *list, *count, *cursor, *fetch;
  __host__ __device__ LevelWs(int32_t* ws, int64_t n)
      : mcnt(ws), mfill(ws + n), mstart(ws + 2 * n), members(ws + 3 * n), list(ws + 4 * n),
        count(ws + 5 * n), cursor(ws + 5 * n + 1), fetch(ws + 5 * n + 2) {}
  static int64_t ints(int64_t n) { return 5 * n + 64; }
};

cudaError_t launch_level_stats(int64_t u0, int64_t nU, int64_t NB, int64_t n_total,
                               const uint8_t* fusable, const uint8_t* alive,
                               const int32_t* absorber, const int32_t* merges, int nm,
                               const int32_t* tile_off, int nt, const double* partials,
                               double* stats, int32_t* level_ws, cudaStream_t s);
cudaError_t launch_merge_groups(void* pool_k, void* pool_v, int dtype, const Geom& g,
                                void* knorm, void* vnorm, const void* oknorm,
                                const void* ovnorm, int32_t* level_ws, int which, float* shadow,
                                int64_t shadow_cap, int32_t* sidx, int32_t* scount, cudaStream_t s);
// exact-decision mode (kern_exact.cu)
cudaError_t launch_exact_merge_keys(void* pool_k, const Geom& g, float* knorm, const float* oknorm,
                                    float* shadow, int64_t cap, int32_t* sidx, int32_t* scount,
                                    int32_t* level_ws, cudaStream_t s);
cudaError_t launch_convert_rows(const void* src, void* dst, const Geom& g, int32_t* level_ws,
                                cudaStream_t s);
cudaError_t launch_alive_rank(int64_t u0, int64_t nU, int64_t NB, const uint8_t* alive,
                              int32_t* live, int32_t* rank, int32_t* count, cudaStream_t s);
cudaError_t launch_stage_rows(const void* pool, int dtype, const Geom& g, int64_t u0, int64_t nU,
                              const int32_t* live, const int32_t* count, void* staged,
                              cudaStream_t s);
cudaError_t launch_remap(int64_t u0, int64_t nU, int64_t NB, int64_t n_total,
                         const int32_t* absorber, int32_t* table, int32_t* refcount,
                         uint8_t* alive, int32_t* level_ws, cudaStream_t s);
cudaError_t launch_finalize(int dtype, int64_t u0, int64_t nU, int64_t NB, const void* okn,
                            const void* ovn, const void* kn, const void* vn,
                            const int32_t* table, const uint8_t* alive, void* ks, void* vs,
                            int32_t* live_ids, int32_t* live_count, int32_t* free_ids,
                            int32_t* free_count, cudaStream_t s);
cudaError_t launch_table_audit(int64_t U, int64_t NB, const int32_t* table,
                               const int32_t* refcount, const uint8_t* alive,
                               int32_t* scratch, int32_t* bad, cudaStream_t s);
cudaError_t launch_table_redirect(int64_t NB, int32_t* table, int32_t* refcount,
                                  uint8_t* alive, int32_t from, int32_t to, int32_t* bad,
                                  cudaStream_t s);
cudaError_t launch_gather_vectors(const void* pool, int dtype, const Geom& g, int64_t u,
                                  const int32_t* ids, int64_t n, const void* norms,
                                  const void* scales, void* out, cudaStream_t s);
cudaError_t launch_refold(const void* pool, int dtype, const Geom& g, int64_t layer,
                          const int32_t* table, const void* scale, void* out,
                          cudaStream_t s);

struct SchedView;
// exact np.quantile (linear) of the non-NaN entries of float64 device segments
int64_t quantile_ws_bytes();
cudaError_t launch_quantile(const void* const* parts, const int64_t* lens, int nseg, double q,
                            double* out, void* ws, cudaStream_t s);

int64_t decode_workspace_size(int dtype, int64_t B, int Hq, int d, int64_t p_blocks, int t);
struct DecodeArgs {
  const void* q;
  int q_dtype;
  const void* pool_k;
  const void* pool_v;
  int dtype;
  Geom g;
  int64_t layer;
  const int32_t* table;
  const void* k_scale;
  const void* v_scale;
  int64_t B, p_blocks;
  const int32_t* seq_blocks;
  int Hq;
  double sm_scale;
  void* out;
  void* lse;
  void* probs;
  void* ws;
  int64_t ws_bytes;
  // sharing-aware schedule (kvf_decode_schedule); null = request-major path
  const struct SchedView* sched = nullptr;
};
cudaError_t launch_paged_decode(const DecodeArgs& a, cudaStream_t s);
// TMA + mma.sync decode path (kern_decode_tma.cu) and the shared split combine
bool decode_tma_supported(const DecodeArgs& a);
cudaError_t launch_decode_tma(const DecodeArgs& a, cudaStream_t s);
// sharing-aware decode (kern_decode_sched.cu). A schedule lists, per head
// unit hu (h units in per_head mode, else 1), `n_items` items of `ib` slots:
//   meta[hu][i]          = b * nit + k  (request b, k-th item of b), items in
//                          ascending order of their middle slot's physical block
//   phys/ks/vs[hu][i][j] = physical block / K scale / V scale of the item's
//                          j-th slot (slots of a request in ascending phys
//                          order); phys = -1 marks padding past seq_blocks
// cap = B * nit is the per-unit stride of meta (x ib for the slot arrays).
struct SchedView {
  const int32_t* meta;
  const int32_t* phys;
  const float* ks;
  const float* vs;
  const int32_t* n_items;
  int64_t cap;
  int ib;
  int dedup;  // runs of repeated blocks inside items (decode them once)
};
bool decode_sched_item_blocks_ok(int ib);
bool decode_sched_shape_ok(int t, int d);  // one block per warp tile: t in {16, 32}
int64_t decode_schedule_ws_ints(int64_t nh, int64_t NB, int64_t B, int64_t p_blocks, int ib);
cudaError_t launch_decode_schedule(const int32_t* table, const float* k_scale, const float* v_scale,
                                   const Geom& g, int64_t layer, int64_t B, int64_t p_blocks,
                                   const int32_t* seq_blocks, int ib, int32_t* order,
                                   int32_t* meta, int32_t* phys, float* ks, float* vs,
                                   int32_t* n_items, int32_t* n_repeats, int32_t* ws,
                                   cudaStream_t s);
cudaError_t launch_decode_sched(const DecodeArgs& a, cudaStream_t s);
// chunked-prefill attention over a CFF-fused context with computation reuse
// (kern_prefill.cu): queries of chunk `chunk` of every request against the
// earlier chunks' keys (all visible) and the chunk's own keys (causal)
struct ChunkPrefillArgs {
  const void* q;  // bf16 [B][chunk_blocks * t][Hq][d]
  const void* pool_k;
  const void* pool_v;
  Geom g;
  int64_t layer;
  const int32_t* table;
  const float* k_scale;
  const float* v_scale;
  const int32_t* order;  // [B][p_blocks] positions sorted by physical block (-1 = none)
  int64_t B, p_blocks;
  int chunk_blocks, chunk, Hq;
  double sm_scale;
  int dedup;
  float* out;  // [B][chunk_blocks * t][Hq][d]
};
bool chunk_prefill_supported(const ChunkPrefillArgs& a, const char** why);
cudaError_t launch_chunk_prefill(const ChunkPrefillArgs& a, cudaStream_t s);
bool chunk_prefill_tc_supported(const ChunkPrefillArgs& a);  // kern_prefill_tc.cu
cudaError_t launch_chunk_prefill_tc(const ChunkPrefillArgs& a, cudaStream_t s);

// out[i] = map[ids[i]] for 0 <= ids[i] < map_len, else -1 (compaction: slot
// tables / schedule ids -> dense rows of a compacted pool)
cudaError_t launch_remap_ids(const int32_t* ids, int64_t n, const int32_t* map, int64_t map_len,
                             int32_t* out, cudaStream_t s);
cudaError_t launch_decode_combine(const DecodeArgs& a, int64_t nsplit, int cbs, cudaStream_t s);

}  // namespace kvf
