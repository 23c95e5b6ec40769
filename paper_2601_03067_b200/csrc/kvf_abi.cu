// extern "C" boundary of libkvfuse_b200.so (declared in include/kvfuse_b200.h).
// Validates arguments, dispatches to the kernel launchers, and maps failures
// to status codes + a thread-local message (kvf_last_error).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include "../../include/kvfuse_b200.h"
#include "kernels.h"

using namespace kvf;


namespace {
thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return KVF_OK;
  return fail(KVF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool valid_dtype(int dt) { return dt == F64 || dt == F32 || dt == BF16; }

int check_geom(int64_t L, int64_t NB, int t, int h, int d, int head_mode, Geom* g) {
  if (L < 1 || NB < 1 || t < 1 || h < 1 || d < 1)
    return fail(KVF_ERR_INVALID, "dimensions must be positive (L=%lld NB=%lld t=%d h=%d d=%d)",
                (long long)L, (long long)NB, t, h, d);
  if (head_mode != 0 && head_mode != 1)
    return fail(KVF_ERR_INVALID, "head_mode must be 0 (folded) or 1 (per_head)");
  if (NB >= (int64_t)INT32_MAX / 2)
    return fail(KVF_ERR_INVALID, "too many blocks per layer (%lld)", (long long)NB);
  g->L = L;
  g->NB = NB;
  g->t = t;
  g->h = h;
  g->d = d;
  g->head_mode = head_mode;
  if (g->units() * NB >= (int64_t)INT32_MAX)
    return fail(KVF_ERR_INVALID, "units*blocks exceeds int32 ids");
  return KVF_OK;
}
}  // namespace

extern "C" {

const char* kvf_last_error(void) { return g_last_error.c_str(); }
int kvf_version(void) { return 10000; }

int kvf_count_nonfinite(const void* data, int dtype, int64_t n, unsigned long long* count_dev,
                        void* stream) {
  if (!valid_dtype(dtype)) return fail(KVF_ERR_INVALID, "bad dtype %d", dtype);
  if (n > 0 && (!data || !count_dev)) return fail(KVF_ERR_INVALID, "null pointer");
  return cuda_status(launch_count_nonfinite(data, dtype, n, count_dev, (cudaStream_t)stream),
                     "kvf_count_nonfinite");
}

int kvf_block_norms(const void* pool, int dtype, int64_t L, int64_t NB, int t, int h, int d,
                    int head_mode, void* norms, void* stream) {
  Geom g;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &g)) return rc;
  if (!valid_dtype(dtype)) return fail(KVF_ERR_INVALID, "bad dtype %d", dtype);
  if (!pool || !norms) return fail(KVF_ERR_INVALID, "null pointer");
  return cuda_status(launch_block_norms(pool, dtype, g, norms, (cudaStream_t)stream),
                     "kvf_block_norms");
}

int kvf_state_init(int dtype, int64_t U, int64_t NB, const void* knorm, uint8_t* fusable,
                   uint8_t* alive, int32_t* absorber, int32_t* table, int32_t* refcount,
                   void* stream) {
  if (!valid_dtype(dtype)) return fail(KVF_ERR_INVALID, "bad dtype %d", dtype);
  if (U < 0 || NB < 0) return fail(KVF_ERR_INVALID, "negative sizes");
  return cuda_status(launch_state_init(dtype, U, NB, knorm, fusable, alive, absorber, table,
                                       refcount, (cudaStream_t)stream),
                     "kvf_state_init");
}

int kvf_sim_tile_shape(int dtype, int head_mode, int path, int* tile_m, int* tile_n,
                       int* partials_per_tile) {
  if (!tile_m || !tile_n || !partials_per_tile) return fail(KVF_ERR_INVALID, "null pointer");
  if (path == KVF_PATH_AUTO) path = dtype == BF16 ? KVF_PATH_TC : KVF_PATH_SIMT;
  if (path == KVF_PATH_TC || path == KVF_PATH_TC_WIDE) {
    // float32 pools run it on a bf16 operand copy (kvf_convert_rows)
    if (dtype != BF16 && dtype != F32)
      return fail(KVF_ERR_INVALID, "tcgen05 path requires a bf16 or float32 pool");
    *tile_m = path == KVF_PATH_TC_WIDE ? kTcTileMWide : kTcTileM;
    *tile_n = kTcTileN;
    *partials_per_tile = kTcPartialsPerTile;
    return KVF_OK;
  }
  if (path != KVF_PATH_SIMT) return fail(KVF_ERR_INVALID, "unknown path %d", path);
  *tile_m = kSimtTile;
  *tile_n = kSimtTile;
  *partials_per_tile = 1;
  return KVF_OK;
}

int kvf_similarity_select(const void* pool_k, int dtype, int64_t L, int64_t NB, int t, int h,
                          int d, int head_mode, int64_t u0, int64_t nU, const void* knorm,
                          const uint8_t* fusable, const uint8_t* alive, int32_t* absorber,
                          const int32_t* merges, int nm, const int32_t* tiles, int nt,
                          double thr, double* partials, double* samples,
                          const int64_t* sample_off, int64_t sample_stride,
                          const int32_t* live, const int32_t* rank, const void* staged,
                          int32_t* rescore_queue, int64_t rescore_cap, double rescore_band,
                          const void* filter, const float* shadow, const int32_t* sidx,
                          int nsplit, float* split_part, int32_t* split_count,
                          int path, void* stream) {
  SimArgs a;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &a.g)) return rc;
  if (!valid_dtype(dtype)) return fail(KVF_ERR_INVALID, "bad dtype %d", dtype);
  if (!(thr > -1.0 && thr < 1.0))
    return fail(KVF_ERR_INVALID, "threshold must lie strictly inside (-1, 1), got %g", thr);
  if (u0 < 0 || nU < 0 || u0 + nU > a.g.units())
    return fail(KVF_ERR_INVALID, "unit range [%lld, %lld) out of bounds", (long long)u0,
                (long long)(u0 + nU));
  if (nt > 0 && (!pool_k || !knorm || !fusable || !alive || !absorber || !merges || !tiles ||
                 !partials))
    return fail(KVF_ERR_INVALID, "null pointer");
  if (samples && !sample_off) return fail(KVF_ERR_INVALID, "samples need sample_off");
  a.pool = pool_k;
  a.dtype = dtype;
  a.u0 = u0;
  a.nU = nU;
  a.knorm = knorm;
  a.fusable = fusable;
  a.alive = alive;
  a.absorber = absorber;
  a.merges = merges;
  a.nm = nm;
  a.tiles = tiles;
  a.nt = nt;
  a.thr = thr;
  a.partials = partials;
  a.samples = samples;
  a.sample_off = sample_off;
  a.sample_stride = sample_stride;
  a.live = live;
  a.rank = rank;
  a.staged = staged;
  if ((live != nullptr) != (rank != nullptr))
    return fail(KVF_ERR_INVALID, "compaction needs live and rank together");
  if (live && !staged && head_mode)
    return fail(KVF_ERR_INVALID, "gathered compaction (no staged rows) needs head_mode 0");
  if ((shadow != nullptr) != (sidx != nullptr))
    return fail(KVF_ERR_INVALID, "shadow rows and shadow index go together");
  if (nsplit < 1 || nsplit > 64) return fail(KVF_ERR_INVALID, "nsplit must lie in [1, 64]");
  if (nsplit > 1 && (!split_part || !split_count))
    return fail(KVF_ERR_INVALID, "split-K needs the partials buffer and the arrival counters");
  a.nsplit = nsplit;
  a.split_part = split_part;
  a.split_count = split_count;
  if (filter && dtype != F32)
    return fail(KVF_ERR_INVALID, "a bf16 operand copy (filter) is for float32 pools");
  const int sim_flags = path & (KVF_SIM_PAIRED | KVF_SIM_WRITE_NORMS);
  path &= ~(KVF_SIM_PAIRED | KVF_SIM_WRITE_NORMS);
  if (sim_flags & KVF_SIM_PAIRED) {
    if (path != KVF_PATH_TC || live)
      return fail(KVF_ERR_INVALID, "KVF_SIM_PAIRED needs the narrow tcgen05 tile and direct rows");
    a.paired = 1;
  }
  if (sim_flags & KVF_SIM_WRITE_NORMS) {
    if (path != KVF_PATH_TC || dtype != BF16 || nsplit != 1 || live || filter)
      return fail(KVF_ERR_INVALID,
                  "KVF_SIM_WRITE_NORMS needs the narrow tcgen05 tile, a bf16 pool, nsplit == 1 "
                  "and direct rows");
    a.write_norms = 1;
  }
  if (path == KVF_PATH_AUTO) path = (dtype == BF16 || filter) ? KVF_PATH_TC : KVF_PATH_SIMT;
  if (path == KVF_PATH_TC_WIDE) {
    if (nsplit != 1) return fail(KVF_ERR_INVALID, "the wide tcgen05 tile takes nsplit == 1");
    if (live && !staged)
      return fail(KVF_ERR_INVALID, "the wide tcgen05 tile takes staged (not gathered) compaction");
    a.wide = 1;
    path = KVF_PATH_TC;
  }
  if (filter) {  // the tensor cores read the bf16 copy; re-scores read the fp32 pool
    if (path != KVF_PATH_TC) return fail(KVF_ERR_INVALID, "a filter copy needs the tcgen05 path");
    a.pool = filter;
    a.dtype = BF16;
    a.split3 = 1;
    if (live) return fail(KVF_ERR_INVALID, "compaction is not available with a float32 split copy");
  }
  if (live && path != KVF_PATH_TC)
    return fail(KVF_ERR_INVALID, "compacted similarity requires the tcgen05 path");
  if (path == KVF_PATH_TC) {
    const char* why = "";
    if (!tc_supported(a, &why))
      return fail(KVF_ERR_INVALID, "tcgen05 similarity path unavailable: %s", why);
    cudaStream_t st = (cudaStream_t)stream;
    const bool resc = rescore_queue != nullptr && rescore_cap > 0 && rescore_band > 0.0;
    if (resc) {
      if (rescore_cap > INT32_MAX / 4) return fail(KVF_ERR_INVALID, "rescore queue too large");
      a.resc = rescore_queue;
      a.resc_count = rescore_queue + 4 * rescore_cap;
      a.resc_cap = rescore_cap;
      a.resc_band = rescore_band;
      cudaError_t e = cudaMemsetAsync(a.resc_count, 0, sizeof(int32_t), st);
      if (e != cudaSuccess) return cuda_status(e, "kvf_similarity_select[tc]");
    }
    if (int rc = cuda_status(launch_sim_tc(a, st), "kvf_similarity_select[tc]")) return rc;
    if (!resc) return KVF_OK;
    RescoreArgs r{pool_k, dtype, a.g, u0, a.resc, a.resc_count, rescore_cap, thr, absorber,
                  merges, samples, sample_off, sample_stride, shadow, sidx};
    return cuda_status(launch_rescore(r, st), "kvf_similarity_select[rescore]");
  }
  if (path != KVF_PATH_SIMT) return fail(KVF_ERR_INVALID, "unknown path %d", path);
  return cuda_status(launch_sim_simt(a, (cudaStream_t)stream), "kvf_similarity_select[simt]");
}

int64_t kvf_level_ws_ints(int64_t n_total) { return LevelWs::ints(n_total); }

int kvf_level_stats(int64_t u0, int64_t nU, int64_t U, int64_t NB, const uint8_t* fusable,
                    const uint8_t* alive, const int32_t* absorber, const int32_t* merges, int nm,
                    const int32_t* tile_off, int nt, const double* partials, double* stats,
                    int32_t* level_ws, void* stream) {
  if (!level_ws) return fail(KVF_ERR_INVALID, "null level workspace");
  if (u0 < 0 || nU < 0 || u0 + nU > U) return fail(KVF_ERR_INVALID, "bad unit range");
  if (nm > 0 && nU > 0 && (!fusable || !alive || !absorber || !merges || !tile_off || !stats))
    return fail(KVF_ERR_INVALID, "null pointer");
  return cuda_status(launch_level_stats(u0, nU, NB, U * NB, fusable, alive, absorber, merges, nm,
                                        tile_off, nt, partials, stats, level_ws,
                                        (cudaStream_t)stream),
                     "kvf_level_stats");
}

int kvf_merge_groups(void* pool_k, void* pool_v, int dtype, int64_t L, int64_t NB, int t, int h,
                     int d, int head_mode, void* knorm, void* vnorm, const void* orig_knorm,
                     const void* orig_vnorm, int32_t* level_ws, int which, float* shadow,
                     int64_t shadow_cap, int32_t* sidx, int32_t* shadow_count, void* stream) {
  Geom g;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &g)) return rc;
  if (!valid_dtype(dtype)) return fail(KVF_ERR_INVALID, "bad dtype %d", dtype);
  if (!pool_k || !pool_v || !knorm || !vnorm || !orig_knorm || !orig_vnorm || !level_ws)
    return fail(KVF_ERR_INVALID, "null pointer");
  if (shadow && g.r() > 16384)
    return fail(KVF_ERR_INVALID, "exact mode supports block vectors up to 16384 elements, got %lld",
                (long long)g.r());
  const int which_sel = which & ~KVF_MERGE_LAST_LEVEL;
  if (which_sel < 1 || which_sel > 3)
    return fail(KVF_ERR_INVALID, "which must be 1 (K), 2 (V) or 3 (K and V)");
  if (shadow) {
    if (dtype != BF16) return fail(KVF_ERR_INVALID, "exact mode (shadow rows) is for bfloat16 pools");
    if (!sidx || !shadow_count) return fail(KVF_ERR_INVALID, "shadow rows need sidx and shadow_count");
    if (d % 8 != 0 || (reinterpret_cast<uintptr_t>(pool_k) & 15) ||
        (reinterpret_cast<uintptr_t>(shadow) & 15))
      return fail(KVF_ERR_INVALID, "exact mode needs d %% 8 == 0 and 16-byte aligned buffers");
  }
  cudaError_t e = launch_merge_groups(pool_k, pool_v, dtype, g, knorm, vnorm, orig_knorm,
                                      orig_vnorm, level_ws, which, shadow, shadow_cap, sidx,
                                      shadow_count, (cudaStream_t)stream);
  return cuda_status(e, "kvf_merge_groups");
}

int kvf_convert_rows(const void* src, int src_dtype, void* dst, int64_t L, int64_t NB, int t,
                     int h, int d, int head_mode, int32_t* level_ws, void* stream) {
  Geom g;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &g)) return rc;
  if (src_dtype != F32) return fail(KVF_ERR_INVALID, "convert_rows reads float32 pools");
  if (!src || !dst) return fail(KVF_ERR_INVALID, "null pointer");
  if (d % 8 != 0 || (reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
    return fail(KVF_ERR_INVALID, "convert_rows needs d %% 8 == 0 and 16-byte aligned buffers");
  return cuda_status(launch_convert_rows(src, dst, g, level_ws, (cudaStream_t)stream),
                     "kvf_convert_rows");
}

int kvf_alive_rank(int64_t u0, int64_t nU, int64_t NB, const uint8_t* alive, int32_t* live,
                   int32_t* rank, int32_t* count, void* stream) {
  if (!alive || !live || !rank || !count) return fail(KVF_ERR_INVALID, "null pointer");
  return cuda_status(launch_alive_rank(u0, nU, NB, alive, live, rank, count, (cudaStream_t)stream),
                     "kvf_alive_rank");
}

int kvf_stage_rows(const void* pool, int dtype, int64_t L, int64_t NB, int t, int h, int d,
                   int head_mode, int64_t u0, int64_t nU, const int32_t* live,
                   const int32_t* count, void* staged, void* stream) {
  Geom g;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &g)) return rc;
  if (dtype != BF16 || d % 8 != 0)
    return fail(KVF_ERR_INVALID, "row staging needs a bf16 pool with d %% 8 == 0");
  if (u0 < 0 || nU < 0 || u0 + nU > g.units()) return fail(KVF_ERR_INVALID, "bad unit range");
  return cuda_status(
      launch_stage_rows(pool, dtype, g, u0, nU, live, count, staged, (cudaStream_t)stream),
      "kvf_stage_rows");
}

int kvf_remap(int64_t u0, int64_t nU, int64_t U, int64_t NB, const int32_t* absorber,
              int32_t* table, int32_t* refcount, uint8_t* alive, int32_t* level_ws,
              void* stream) {
  if (!absorber || !table || !refcount || !alive || !level_ws)
    return fail(KVF_ERR_INVALID, "null pointer");
  if (u0 < 0 || nU < 0 || u0 + nU > U) return fail(KVF_ERR_INVALID, "bad unit range");
  return cuda_status(launch_remap(u0, nU, NB, U * NB, absorber, table, refcount, alive, level_ws,
                                  (cudaStream_t)stream),
                     "kvf_remap");
}

int kvf_finalize(int dtype, int64_t u0, int64_t nU, int64_t NB, const void* orig_knorm,
                 const void* orig_vnorm, const void* knorm, const void* vnorm,
                 const int32_t* table, const uint8_t* alive, void* k_scale, void* v_scale,
                 int32_t* live_ids, int32_t* live_count, int32_t* free_ids, int32_t* free_count,
                 void* stream) {
  if (!valid_dtype(dtype)) return fail(KVF_ERR_INVALID, "bad dtype %d", dtype);
  return cuda_status(launch_finalize(dtype, u0, nU, NB, orig_knorm, orig_vnorm, knorm, vnorm,
                                     table, alive, k_scale, v_scale, live_ids, live_count,
                                     free_ids, free_count, (cudaStream_t)stream),
                     "kvf_finalize");
}

int kvf_table_audit(int64_t U, int64_t NB, const int32_t* table, const int32_t* refcount,
                    const uint8_t* alive, int32_t* scratch, int32_t* bad_dev, void* stream) {
  if (!bad_dev) return fail(KVF_ERR_INVALID, "null pointer");
  return cuda_status(launch_table_audit(U, NB, table, refcount, alive, scratch, bad_dev,
                                        (cudaStream_t)stream),
                     "kvf_table_audit");
}

int kvf_table_redirect(int64_t NB, int32_t* table, int32_t* refcount, uint8_t* alive,
                       int32_t from_phys, int32_t to_phys, int32_t* bad_dev, void* stream) {
  if (!table || !refcount || !alive || !bad_dev) return fail(KVF_ERR_INVALID, "null pointer");
  return cuda_status(launch_table_redirect(NB, table, refcount, alive, from_phys, to_phys,
                                           bad_dev, (cudaStream_t)stream),
                     "kvf_table_redirect");
}

int kvf_gather_vectors(const void* pool, int dtype, int64_t L, int64_t NB, int t, int h, int d,
                       int head_mode, int64_t u, const int32_t* ids, int64_t n,
                       const void* norms, const void* scales, void* out, void* stream) {
  Geom g;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &g)) return rc;
  if (!valid_dtype(dtype)) return fail(KVF_ERR_INVALID, "bad dtype %d", dtype);
  if (u < 0 || u >= g.units()) return fail(KVF_ERR_INVALID, "unit %lld out of range", (long long)u);
  return cuda_status(
      launch_gather_vectors(pool, dtype, g, u, ids, n, norms, scales, out, (cudaStream_t)stream),
      "kvf_gather_vectors");
}

int kvf_refold(const void* pool, int dtype, int64_t L, int64_t NB, int t, int h, int d,
               int head_mode, int64_t layer, const int32_t* table, const void* scale, void* out,
               void* stream) {
  Geom g;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &g)) return rc;
  if (!valid_dtype(dtype)) return fail(KVF_ERR_INVALID, "bad dtype %d", dtype);
  if (layer < 0 || layer >= L)
    return fail(KVF_ERR_INVALID, "layer %lld out of range [0, %lld)", (long long)layer,
                (long long)L);
  return cuda_status(launch_refold(pool, dtype, g, layer, table, scale, out, (cudaStream_t)stream),
                     "kvf_refold");
}

int64_t kvf_decode_workspace_size(int dtype, int64_t B, int Hq, int d, int64_t p_blocks, int t) {
  return decode_workspace_size(dtype, B, Hq, d, p_blocks, t);
}

static int paged_decode_impl(const void* q, int q_dtype, const void* pool_k, const void* pool_v,
                     int dtype, int64_t L, int64_t NB, int t, int h, int d, int head_mode,
                     int64_t layer, const int32_t* table, const void* k_scale,
                     const void* v_scale, int64_t B, int64_t p_blocks,
                     const int32_t* seq_blocks, int Hq, double sm_scale, void* out, void* lse,
                     void* probs, void* workspace, int64_t workspace_bytes, void* stream,
                             const SchedView* sched) {
  DecodeArgs a;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &a.g)) return rc;
  if (!valid_dtype(dtype) || !valid_dtype(q_dtype)) return fail(KVF_ERR_INVALID, "bad dtype");
  if (layer < 0 || layer >= L) return fail(KVF_ERR_INVALID, "layer out of range");
  if (Hq < 1 || Hq % h != 0)
    return fail(KVF_ERR_INVALID, "query heads %d must be a positive multiple of kv heads %d", Hq, h);
  if (Hq / h > 8 || d > 128 || t > 32)
    return fail(KVF_ERR_INVALID, "decode kernel limits: Hq/h <= 8, d <= 128, t <= 32");
  // the request-major path reads table[unit][b * p_blocks + j]; the scheduled
  // path reads only the schedule's physical ids (< NB), so a compacted pool
  // (NB = live blocks < slots) is allowed there
  if (B < 0 || p_blocks < 1 || (!sched && B * p_blocks > NB))
    return fail(KVF_ERR_INVALID, "B*p_blocks (%lld) exceeds blocks per layer (%lld)",
                (long long)(B * p_blocks), (long long)NB);
  a.q = q;
  a.q_dtype = q_dtype;
  a.pool_k = pool_k;
  a.pool_v = pool_v;
  a.dtype = dtype;
  a.layer = layer;
  a.table = table;
  a.k_scale = k_scale;
  a.v_scale = v_scale;
  a.B = B;
  a.p_blocks = p_blocks;
  a.seq_blocks = seq_blocks;
  a.Hq = Hq;
  a.sm_scale = sm_scale;
  a.out = out;
  a.lse = lse;
  a.probs = probs;
  a.ws = workspace;
  a.ws_bytes = workspace_bytes;
  a.sched = sched;
  if (sched) {
    if (!sched->meta || !sched->phys || !sched->ks || !sched->vs || !sched->n_items)
      return fail(KVF_ERR_INVALID, "schedule arrays must all be given");
    if (!decode_sched_item_blocks_ok(sched->ib))
      return fail(KVF_ERR_INVALID, "item_blocks must be 8 or 16, got %d", sched->ib);
    if (!decode_sched_shape_ok(t, d))
      return fail(KVF_ERR_INVALID, "scheduled decode needs t in {16, 32} and d in {64, 128}");
    if (!decode_tma_supported(a))
      return fail(KVF_ERR_INVALID, "scheduled decode needs bf16 pools, d in {64,128}, t | 32");
  }
  if (!sched && workspace_bytes < decode_workspace_size(dtype, B, Hq, d, p_blocks, t))
    return fail(KVF_ERR_INVALID, "decode workspace too small");
  return cuda_status(launch_paged_decode(a, (cudaStream_t)stream), "kvf_paged_decode");
}

int kvf_paged_decode(const void* q, int q_dtype, const void* pool_k, const void* pool_v,
                     int dtype, int64_t L, int64_t NB, int t, int h, int d, int head_mode,
                     int64_t layer, const int32_t* table, const void* k_scale,
                     const void* v_scale, int64_t B, int64_t p_blocks,
                     const int32_t* seq_blocks, int Hq, double sm_scale, void* out, void* lse,
                     void* probs, void* workspace, int64_t workspace_bytes, void* stream) {
  return paged_decode_impl(q, q_dtype, pool_k, pool_v, dtype, L, NB, t, h, d, head_mode, layer,
                           table, k_scale, v_scale, B, p_blocks, seq_blocks, Hq, sm_scale, out,
                           lse, probs, workspace, workspace_bytes, stream, nullptr);
}

int kvf_remap_ids(const int32_t* ids, int64_t n, const int32_t* map, int64_t map_len, int32_t* out,
                  void* stream) {
  if (n < 0 || map_len < 0) return fail(KVF_ERR_INVALID, "negative length");
  if (n > 0 && (!ids || !map || !out)) return fail(KVF_ERR_INVALID, "null pointer");
  return cuda_status(launch_remap_ids(ids, n, map, map_len, out, (cudaStream_t)stream),
                     "kvf_remap_ids");
}

int64_t kvf_quantile_ws_bytes(void) { return quantile_ws_bytes(); }

int kvf_quantile(const void* const* parts, const int64_t* lens, int nparts, double q, double* out,
                 void* workspace, int64_t workspace_bytes, void* stream) {
  if (!(q >= 0.0 && q <= 1.0)) return fail(KVF_ERR_INVALID, "quantile q must lie in [0, 1], got %g", q);
  if (nparts < 0 || (nparts > 0 && (!parts || !lens))) return fail(KVF_ERR_INVALID, "bad segment list");
  if (!out || !workspace) return fail(KVF_ERR_INVALID, "null pointer");
  if (workspace_bytes < quantile_ws_bytes()) return fail(KVF_ERR_INVALID, "quantile workspace too small");
  for (int i = 0; i < nparts; ++i)
    if (lens[i] < 0 || (lens[i] > 0 && !parts[i])) return fail(KVF_ERR_INVALID, "bad segment %d", i);
  return cuda_status(launch_quantile(parts, lens, nparts, q, out, workspace, (cudaStream_t)stream),
                     "kvf_quantile");
}

int kvf_chunk_prefill(const void* q, const void* pool_k, const void* pool_v, int dtype, int64_t L,
                      int64_t NB, int t, int h, int d, int head_mode, int64_t layer,
                      const int32_t* table, const void* k_scale, const void* v_scale,
                      const int32_t* order, int64_t B, int64_t p_blocks, int chunk_blocks,
                      int chunk, int Hq, double sm_scale, int dedup, int path, void* out,
                      void* stream) {
  ChunkPrefillArgs a;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &a.g)) return rc;
  if (dtype != BF16) return fail(KVF_ERR_INVALID, "chunked prefill needs bf16 pools");
  if (layer < 0 || layer >= L) return fail(KVF_ERR_INVALID, "layer out of range");
  if (B < 0 || p_blocks < 1 || B * p_blocks > NB || chunk_blocks < 1 || Hq < 1 || Hq % h)
    return fail(KVF_ERR_INVALID, "bad batch / chunk / head shape");
  if (B > 0 && (!q || !pool_k || !pool_v || !table || !k_scale || !v_scale || !order || !out))
    return fail(KVF_ERR_INVALID, "null pointer");
  a.q = q;
  a.pool_k = pool_k;
  a.pool_v = pool_v;
  a.layer = layer;
  a.table = table;
  a.k_scale = (const float*)k_scale;
  a.v_scale = (const float*)v_scale;
  a.order = order;
  a.B = B;
  a.p_blocks = p_blocks;
  a.chunk_blocks = chunk_blocks;
  a.chunk = chunk;
  a.Hq = Hq;
  a.sm_scale = sm_scale;
  a.dedup = dedup ? 1 : 0;
  a.out = (float*)out;
  const char* why = "";
  if (!chunk_prefill_supported(a, &why)) return fail(KVF_ERR_INVALID, "chunked prefill: %s", why);
  // path: 0 auto (tcgen05 when the shape allows: 3.7 vs 9.7 ms mma.sync on the last
  // chunk of 4 x 16K), 1 mma.sync, 2 tcgen05
  const bool tc_ok = chunk_prefill_tc_supported(a);
  if (path == 2 && !tc_ok)
    return fail(KVF_ERR_INVALID,
                "tcgen05 chunked prefill needs d = 128, t = 16, folded units, 128 %% G == 0, "
                "chunk tokens a multiple of 256 / G and p <= 1024 (path = auto falls back to mma.sync)");
  if (path != 1 && tc_ok)
    return cuda_status(launch_chunk_prefill_tc(a, (cudaStream_t)stream), "kvf_chunk_prefill[tc]");
  return cuda_status(launch_chunk_prefill(a, (cudaStream_t)stream), "kvf_chunk_prefill");
}

int kvf_decode_schedule_item_blocks(void) { return 16; }

int64_t kvf_decode_schedule_ws_ints(int head_mode, int h, int64_t NB, int64_t B, int64_t p_blocks,
                                    int item_blocks) {
  if (!decode_sched_item_blocks_ok(item_blocks)) return -1;
  return decode_schedule_ws_ints(head_mode ? h : 1, NB, B, p_blocks, item_blocks);
}

int kvf_decode_schedule(const int32_t* table, const void* k_scale, const void* v_scale, int64_t L,
                        int64_t NB, int t, int h, int d, int head_mode, int64_t layer, int64_t B,
                        int64_t p_blocks, const int32_t* seq_blocks, int item_blocks,
                        int32_t* order, int32_t* meta, int32_t* phys, float* ks, float* vs,
                        int32_t* n_items, int32_t* n_repeats, int32_t* workspace,
                        int64_t workspace_ints, void* stream) {
  Geom g;
  if (int rc = check_geom(L, NB, t, h, d, head_mode, &g)) return rc;
  if (layer < 0 || layer >= L) return fail(KVF_ERR_INVALID, "layer out of range");
  if (B < 0 || p_blocks < 1 || B * p_blocks > NB)
    return fail(KVF_ERR_INVALID, "B*p_blocks (%lld) exceeds blocks per layer (%lld)",
                (long long)(B * p_blocks), (long long)NB);
  if (p_blocks > 16384) return fail(KVF_ERR_INVALID, "p_blocks > 16384 per request");
  if (!decode_sched_item_blocks_ok(item_blocks))
    return fail(KVF_ERR_INVALID, "item_blocks must be 8 or 16, got %d", item_blocks);
  if (!table || !k_scale || !v_scale || !order || !meta || !phys || !ks || !vs || !n_items ||
      !workspace)
    return fail(KVF_ERR_INVALID, "null pointer");
  if (workspace_ints < decode_schedule_ws_ints(head_mode ? h : 1, NB, B, p_blocks, item_blocks))
    return fail(KVF_ERR_INVALID, "schedule workspace too small");
  return cuda_status(launch_decode_schedule(table, (const float*)k_scale, (const float*)v_scale, g,
                                            layer, B, p_blocks, seq_blocks, item_blocks, order,
                                            meta, phys, ks, vs, n_items, n_repeats, workspace,
                                            (cudaStream_t)stream),
                     "kvf_decode_schedule");
}

int kvf_paged_decode_sched(const void* q, int q_dtype, const void* pool_k, const void* pool_v,
                           int dtype, int64_t L, int64_t NB, int t, int h, int d, int head_mode,
                           int64_t layer, const int32_t* table, const void* k_scale,
                           const void* v_scale, int64_t B, int64_t p_blocks,
                           const int32_t* seq_blocks, int Hq, double sm_scale, void* out,
                           void* lse, int item_blocks, const int32_t* meta, const int32_t* phys,
                           const float* ks, const float* vs, const int32_t* n_items, int dedup,
                           void* workspace, int64_t workspace_bytes, void* stream) {
  const int64_t nit = item_blocks > 0 ? (p_blocks + item_blocks - 1) / item_blocks : 0;
  SchedView v{meta, phys, ks, vs, n_items, B * nit, item_blocks, dedup ? 1 : 0};
  if (workspace_bytes < B * Hq * nit * (int64_t)(d + 2) * 4)
    return fail(KVF_ERR_INVALID, "decode workspace too small");
  return paged_decode_impl(q, q_dtype, pool_k, pool_v, dtype, L, NB, t, h, d, head_mode, layer,
                           table, k_scale, v_scale, B, p_blocks, seq_blocks, Hq, sm_scale, out,
                           lse, nullptr, workspace, workspace_bytes, stream, &v);
}

}  // extern "C"
