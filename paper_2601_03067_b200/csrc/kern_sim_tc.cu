// K2 + K3 on the 5th-gen tensor cores (sm_100a): block-similarity GEMM with
// the first-match selection fused into the epilogue. Replaces fusion.py:244-265
// (sim = kdir[left] @ kdir[right].T, then the per-left-row candidate loop).
//
// A CTA pair (cluster of 2, tcgen05 cta_group::2) computes a 256 (left
// blocks) x 256 (right blocks) similarity tile of one merge of one unit,
// K = the block vector length r (t*h*d folded, t*d per head), bf16 inputs,
// fp32 accumulation in TMEM. Each CTA stages its 128 A rows and its 128-row
// half of B; the leader issues M256 N256 K16 MMAs over both CTAs' smem:
//   warp 0      TMA producer (both CTAs): 4-D tensor map over the pool
//               (d, h, t, rows) or over the staged alive rows, box
//               {64, 1, 1, 128}, 128B swizzle, 6-stage ring of 32 KB; both
//               CTAs' bytes complete on the leader's full barrier
//   warp 1      MMA issuer (leader): 4 x tcgen05.mma.cta_group::2.kind::f16
//               per 64-wide k-step; tcgen05.commit multicasts the stage
//               release to both CTAs
//   warp 2      TMEM allocator (2 x 256 columns, cta_group::2)
//   warps 4..11 epilogue (two warps per TMEM lane quarter, one per column
//               half): per-tile column metadata, tcgen05.ld 32x32b.x32
//               -> sim = acc / (|x_i||x_j|), alive/fusable masks, strict
//               '> thr' (pairs within resc_band deferred to the exact
//               re-score), per-column min row via redux.sync + smem atomicMin
//               -> one global atomicMin per column; similarity moments per CTA.
// Raw pool rows are fed to the MMA (no normalised copy): norms are applied in
// the epilogue, so level-1 similarities are exact-input bf16 products.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include "kernels.h"

namespace kvf {

namespace {
constexpr int BM = 128;               // A rows per CTA (M = 256 per pair)
constexpr int BN = kTcTileN;          // 256 right blocks per pair (N)
constexpr int BNH = BN / 2;           // B rows staged per CTA
constexpr int BK = 64;                // bf16 elements per k-step (128 B rows)
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BNH * BK * 2;  // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;  // two 256-column accumulators
constexpr int EPI_WARPS = 8;  // 2 per TMEM lane quarter, each half of the columns
static_assert(kTcPartialsPerTile == 2 * EPI_WARPS, "one moment slot per epilogue warp of the pair");
constexpr int NTHREADS = 128 + 32 * EPI_WARPS;
constexpr int META_BYTES = 12288;  // barriers, work records, epilogue / norm metadata
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + META_BYTES;
// wide tile (256 A rows per CTA): 4 stages of 48 KB
constexpr int SMEM_BYTES_WIDE = 4 * (2 * A_BYTES + B_BYTES) + 1024 + META_BYTES;
static_assert(SMEM_BYTES_WIDE <= 227 * 1024, "wide ring exceeds shared memory");
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // cluster smem address of CTA 0

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 2-SM TMA: the bytes complete on the leader CTA's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_4d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1),
      "r"(c2), "r"(c3)
      : "memory");
}
// 2-SM TMA gather4: rows r[0..3] x 64 columns of a 2-D map into 4 consecutive
// 128 B smem rows (the 128B swizzle follows the smem address, so 32 gathers at
// 512 B steps lay out exactly like one 128-row box)
__device__ __forceinline__ void tma_gather4_2sm(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int col, const int (&r)[4]) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerMask), "r"(col), "r"(r[0]),
      "r"(r[1]), "r"(r[2]), "r"(r[3])
      : "memory");
}
// K-major, 128B-swizzled UMMA shared-memory descriptor: SBO = 1024 B (8 rows
// x 128 B), LBO unused (1), version 1 (sm_100), layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t desc = 0;
  desc |= (uint64_t)((saddr >> 4) & 0x3FFF);
  desc |= (uint64_t)1 << 16;
  desc |= (uint64_t)(1024 >> 4) << 32;
  desc |= (uint64_t)1 << 46;
  desc |= (uint64_t)2 << 61;
  return desc;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N = 256,
// M = 256 (pair).
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)((2 * BM) >> 4) << 24);

__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accum));
}
// completion of all prior MMAs arrives on the barrier at this offset in both CTAs
__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
}  // namespace

struct TileInfo {
  bool active;
  int64_t ul, u;
  int m, i0, j0, lb, mid, re, pl, pm, pr;
};

// Work item w (unit-major: clusters running together share a unit's operand
// rows in L2) -> tile geometry.
__device__ __forceinline__ TileInfo tile_info(int w, int nt, int64_t u0, const Geom& g,
                                              const int32_t* __restrict__ merges,
                                              const int32_t* __restrict__ tiles,
                                              const int32_t* __restrict__ rank, bool staged) {
  TileInfo t;
  t.ul = w / nt;
  const int tile = w - (int)t.ul * nt;
  t.u = u0 + t.ul;
  t.m = tiles[3 * tile];
  t.i0 = tiles[3 * tile + 1];
  t.j0 = tiles[3 * tile + 2];
  t.lb = merges[3 * t.m];
  t.mid = merges[3 * t.m + 1];
  t.re = merges[3 * t.m + 2];
  t.pl = t.lb;
  t.pm = t.mid;
  t.pr = t.re;
  if (staged) {  // compacted mode: rows are positions in the unit's alive list
    const int32_t* rk = rank + t.u * (g.NB + 1);
    t.pl = rk[t.lb];
    t.pm = rk[t.mid];
    t.pr = rk[t.re];
  }
  t.active = t.i0 < t.pm - t.pl && t.j0 < t.pr - t.pm;
  return t;
}

// A published work item: w and the tile geometry (the scheduler warp computes it once,
// consumers read it from shared memory instead of re-walking tiles / merges / rank)
constexpr int kRec = 12;
__device__ __forceinline__ TileInfo rec_info(const int32_t* r, int nt, int64_t u0) {
  TileInfo t;
  const int w = r[0];
  t.ul = w / nt;
  t.u = u0 + t.ul;
  t.m = r[1];
  t.i0 = r[2];
  t.j0 = r[3];
  t.lb = r[4];
  t.mid = r[5];
  t.re = r[6];
  t.pl = r[7];
  t.pm = r[8];
  t.pr = r[9];
  t.active = true;
  return t;
}

// Paired small merges (every merge side of the level <= 128 blocks): a tile holds merge m on
// CTA 0 and merge m + 1 on CTA 1, i.e. on the diagonal of the pair's 256 x 256 product --
// CTA c streams its own merge's left blocks as A and its right blocks as its B half, and
// only its own quadrant counts. The view shifts i0 / j0 so the shared address and index
// arithmetic lands on merge m + c; `dead` marks the odd level's missing partner merge.
__device__ __forceinline__ void pair_view(TileInfo& t, uint32_t crank, const int32_t* __restrict__ merges,
                                          int nm, bool& dead) {
  const int mc = t.m + (int)crank;
  dead = mc >= nm;
  const int mm = dead ? nm - 1 : mc;  // addresses of a real merge; its rows are masked
  t.m = mm;
  t.lb = t.pl = merges[3 * mm];
  t.mid = t.pm = merges[3 * mm + 1];
  t.re = t.pr = merges[3 * mm + 2];
  t.i0 = -(int)crank * BM;
  t.j0 = -(int)crank * BNH;
}

// 16-byte global -> shared copy on the LSU path (L2 only), completion tracked by an
// mbarrier arrive-on (noinc: the barrier's expected count covers the arriving lanes)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_addr(const void* p, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(cta));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   cluster_addr(bar, cta))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_cluster_s32(const void* p, uint32_t cta, int32_t v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cluster_addr(p, cta)), "r"(v) : "memory");
}

constexpr int SCHED_DEPTH = 4;
// sched_empty arrivals per slot: producers of both CTAs + leader MMA warp + the
// epilogue warps of both CTAs
// warps in each CTA
constexpr uint32_t kSchedConsumers = 3 + 2 * EPI_WARPS;

// Persistent: P CTA pairs pull work items from a global counter (the leader's
// producer thread fetches, skips tiles beyond the alive blocks, and broadcasts
// the item to both CTAs' roles through a 4-deep shared-memory ring). TMEM
// holds two 256-column accumulators, so the epilogue of tile k overlaps the
// MMAs of tile k + 1 (tmem_full / tmem_empty barrier pair per buffer).
template <int BMC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
sim_tc_kernel(const __grid_constant__ CUtensorMap tmap, Geom g, int64_t u0, int64_t nU,
              float* __restrict__ knorm, uint8_t* __restrict__ fusable,
              const uint8_t* __restrict__ alive, int32_t* __restrict__ absorber,
              const int32_t* __restrict__ merges, const int32_t* __restrict__ tiles, int nt,
              float thr, double* __restrict__ partials, double* __restrict__ samples,
              const int64_t* __restrict__ sample_off, int64_t sample_stride,
              const int32_t* __restrict__ live, const int32_t* __restrict__ rank,
              int32_t* __restrict__ resc, int32_t* __restrict__ resc_count, int resc_cap,
              float resc_band, int32_t* __restrict__ work_counter, int gathered, int split3,
              int nsplit, float* __restrict__ spart, int32_t* __restrict__ scnt,
              const __nv_bfloat16* __restrict__ pool, int fnorm, int nm, int paired) {
  // BMC = A rows per CTA: 128 (pair tile 256 x 256, two TMEM accumulators, the epilogue of
  // tile k overlaps the MMAs of tile k + 1) or 256 ("wide": pair tile 512 x 256, one
  // accumulator filling TMEM; per k-step a CTA loads 32 KB of A + 16 KB of B for twice the
  // MMAs, 171 instead of 128 FLOP per L2->SM byte -- the crossbar rate bounds the narrow tile)
  constexpr bool WIDE = BMC == 256;
  constexpr int STG = WIDE ? 4 : 6;            // ring stages (48 KB / 32 KB each)
  constexpr int ABY = BMC * BK * 2;
  constexpr int SBY = ABY + B_BYTES;
  constexpr uint32_t NACC = WIDE ? 1 : 2;       // TMEM accumulators
  if (WIDE) gathered = 0;  // gathered operands and split-K run on the narrow tile only
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ int split_last_sh;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* meta = smem + STG * SBY;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(meta);
  uint64_t* empty_bar = full_bar + STG;
  uint64_t* tmem_full = empty_bar + STG;           // [2]
  uint64_t* tmem_empty = tmem_full + 2;               // [2], used on the leader
  uint64_t* sched_full = tmem_empty + 2;              // [SCHED_DEPTH]
  uint64_t* sched_empty = sched_full + SCHED_DEPTH;   // [SCHED_DEPTH], used on the leader
  int32_t* sched_rec = reinterpret_cast<int32_t*>(sched_empty + SCHED_DEPTH);  // [SCHED_DEPTH][kRec]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched_rec + SCHED_DEPTH * kRec);
  // gathered rows on the LSU path (gathered == 2): per-CTA completion of a stage's
  // cp.async copies (both producer warps' lanes arrive on it)
  uint64_t* full_loc = reinterpret_cast<uint64_t*>(meta + 448);  // [STG]
  // epilogue column metadata, double-buffered by tile parity: [2][BN] each
  float* inv_j_b = reinterpret_cast<float*>(meta + 512);
  int32_t* colmin_b = reinterpret_cast<int32_t*>(meta + 512 + 8 * BN);
  int32_t* colid_b = reinterpret_cast<int32_t*>(meta + 512 + 16 * BN);  // block ids
  uint8_t* ok_j_b = meta + 512 + 24 * BN;
  // fused key norms (fnorm, level 1): per-stage "MMA done" barriers in both CTAs (the norm
  // warps copy a stage's rows to registers after the MMAs read it -- the MMA commit is the
  // one completion signal the peer CTA receives for its own rows -- and release it next to
  // the commit; relaying the leader's full barrier to the peer instead measured slower:
  // cluster-scope acquires invalidate L1 on every stage), norms-ready barriers by tile
  // parity, and the tile's row / column norms ([2][BM] A rows, [2][BN] B rows of the pair)
  uint64_t* mma_done = reinterpret_cast<uint64_t*>(meta + 7168);  // [STG]
  uint64_t* norm_ready = mma_done + 8;                              // [2]
  float* anorm_b = reinterpret_cast<float*>(meta + 8192);
  float* bnorm_b = anorm_b + 2 * BM;
  if (WIDE) fnorm = paired = 0;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cta_rank();
  const bool leader = crank == 0;
  const bool staged = live != nullptr;  // tiles index alive positions (staged or gathered rows)
  // split-K (few, long-K tiles: cfg1 / CFF levels): work item = (tile, k-split); each
  // split's fp32 accumulator goes to spart, the CTA arriving last per (tile, CTA rank)
  // sums the nsplit partials in split order (deterministic) and runs the epilogue
  const int nwork = (int)(nt * nU) * nsplit;
  const int P = (int)(gridDim.x >> 1);
  const int layer_div = g.head_mode ? g.h : 1;
  const int dpc = g.d / BK;
  const int nk = g.head_mode ? g.t * dpc : g.t * g.h * dpc;
  // split3 (float32 pools): the operand copy holds hi = bf16(x) in rows [0, L*NB) and
  // lo = bf16(x - hi) in rows [L*NB, 2*L*NB); three passes over K accumulate
  // hi.hi + hi.lo + lo.hi (the dropped lo.lo term is ~2^-16 relative)
  const int nk_run = split3 ? 3 * nk : nk;
  const int lo_rows = (int)(g.L * g.NB);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STG; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], fnorm ? 1 + EPI_WARPS : 1);  // MMA commit (+ the norm warps)
      mbar_init(&mma_done[s], 1);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&norm_ready[b], 2 * EPI_WARPS);  // both CTAs
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 2 * EPI_WARPS);  // epilogue warps x 2 CTAs
    }
    for (int s = 0; s < STG; ++s) mbar_init(&full_loc[s], 64);
    for (int c = 0; c < 2 * BN; ++c) colmin_b[c] = kNone;
    for (int b = 0; b < SCHED_DEPTH; ++b) {
      mbar_init(&sched_full[b], 1);
      // + in LSU-gather mode: warp 2 of both CTAs (second producer) and the peer's relay
      mbar_init(&sched_empty[b], kSchedConsumers + (gathered == 2 ? 3 : 0));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 || (gathered == 2 && warp == 2)) {
    // producer warp: lane 0 runs the tile scheduler; operand rows are loaded by
    // lane 0 (tiled boxes over the pool or the staged rows) or, in gathered
    // mode, by all 32 lanes with TMA gather4 (4 alive rows per lane per operand)
    if (lane == 0)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    uint32_t kk = 0;  // global k-step counter (ring position)
    for (uint32_t it = 0;; ++it) {
      const int sl = it % SCHED_DEPTH;
      const uint32_t sph = (it / SCHED_DEPTH) & 1;
      int w = 0;
      if (lane == 0) {
        mbar_wait_cluster(&sched_full[sl], sph);
        w = sched_rec[sl * kRec];
      }
      w = __shfl_sync(0xffffffffu, w, 0);
      if (w < 0) {
        if (lane == 0) mbar_arrive_cluster(&sched_empty[sl], 0);
        break;
      }
      TileInfo t = rec_info(sched_rec + sl * kRec, nt, u0);
      if (paired) {
        bool dead;
        pair_view(t, crank, merges, nm, dead);
      }
      const int sk = sched_rec[sl * kRec + 10];
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&sched_empty[sl], 0);
      const int kr0 = (int)((int64_t)sk * nk_run / nsplit), kr1 = (int)((int64_t)(sk + 1) * nk_run / nsplit);
      const int layer = (int)(t.u / layer_div);
      const int head = g.head_mode ? (int)(t.u % g.h) : 0;
      const int mi0 = t.i0 + (int)crank * BMC;
      if (gathered == 2) {
        // LSU gather: warp 0 copies this CTA's 128 A rows, warp 2 its 128 B rows; a warp
        // instruction moves 4 rows x 128 B (lane = row (lane >> 3), 16-B chunk (lane & 7)),
        // stored at the 128B-swizzled position TMA would use; positions past the merge's
        // alive blocks repeat its last alive block (the epilogue masks them)
        const int pw = warp == 0 ? 0 : 1;
        const int sub = lane >> 3, ch = lane & 7;
        const int64_t gb = t.u * g.NB;
        const int nrow = pw == 0 ? t.pm - t.pl : t.pr - t.pm;
        const int p0 = pw == 0 ? mi0 : t.j0 + (int)crank * BNH;
        const int32_t* lv = live + gb + (pw == 0 ? t.pl : t.pm);
        const char* base[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int id = lv[min(p0 + 4 * i + sub, nrow - 1)];
          base[i] = reinterpret_cast<const char*>(pool) +
                    ((int64_t)layer * g.NB + id) * g.E() * 2 + ch * 16;
        }
        const uint32_t o0 = (uint32_t)(sub * 128 + ((ch ^ sub) * 16));
        const uint32_t o1 = (uint32_t)((sub + 4) * 128 + ((ch ^ (sub + 4)) * 16));
        for (int ks = 0; ks < nk; ++ks, ++kk) {
          const int s = kk % STG;
          const uint32_t ph = (kk / STG) & 1;
          if (lane == 0) mbar_wait(&empty_bar[s], ph ^ 1);
          __syncwarp();
          const uint32_t tile = smem_u32(smem + s * SBY + pw * ABY);
#pragma unroll
          for (int i = 0; i < 32; ++i)  // rows 4i + sub: 8-row swizzle atoms at i/2 * 1024 B
            cp_async16(tile + (uint32_t)(i >> 1) * 1024u + ((i & 1) ? o1 : o0), base[i] + ks * 128);
          cp_async_arrive_noinc(&full_loc[s]);
        }
        continue;
      }
      if (gathered) {
        // rows 4*lane .. 4*lane+3 of this CTA's A (left) and B (right) operand;
        // positions past the merge's alive blocks repeat its last alive block
        // (the epilogue masks them)
        const int64_t gb = t.u * g.NB;
        const int na = t.pm - t.pl, nb = t.pr - t.pm;
        int ra[4], rb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int pa = min(mi0 + 4 * lane + q, na - 1);
          const int pb = min(t.j0 + (int)crank * BNH + 4 * lane + q, nb - 1);
          ra[q] = layer * (int)g.NB + live[gb + t.pl + pa];
          rb[q] = layer * (int)g.NB + live[gb + t.pm + pb];
        }
        for (int ks = 0; ks < nk; ++ks, ++kk) {
          const int s = kk % STG;
          const uint32_t ph = (kk / STG) & 1;
          if (lane == 0) {
            mbar_wait(&empty_bar[s], ph ^ 1);
            if (leader) mbar_expect_tx(&full_bar[s], 2 * SBY);
          }
          __syncwarp();
          uint8_t* sa = smem + s * SBY;
          uint8_t* sb = sa + ABY;
          tma_gather4_2sm(sa + lane * 4 * BK * 2, &tmap, &full_bar[s], ks * BK, ra);
          tma_gather4_2sm(sb + lane * 4 * BK * 2, &tmap, &full_bar[s], ks * BK, rb);
        }
        continue;
      }
      if (lane != 0) continue;
      const int rowA = staged ? (int)(t.ul * g.NB) + t.pl + mi0 : layer * g.NB + t.lb + mi0;
      const int rowB =
          (staged ? (int)(t.ul * g.NB) + t.pm + t.j0 : layer * g.NB + t.mid + t.j0) +
          (int)crank * BNH;
      for (int kr = kr0; kr < kr1; ++kr, ++kk) {
        const int s = kk % STG;
        const uint32_t ph = (kk / STG) & 1;
        mbar_wait(&empty_bar[s], ph ^ 1);
        const int part = kr / nk;  // split3 pass: 0 hi.hi, 1 hi.lo, 2 lo.hi
        const int ks = kr - part * nk;
        const int dc = ks % dpc;
        const int rest = ks / dpc;
        const int hh = g.head_mode ? head : rest % g.h;
        const int tok = g.head_mode ? rest : rest / g.h;
        // pool map: (d, h, t, rows); staged map: (64, r/64, 1, rows)
        const int c0 = staged ? 0 : dc * BK, c1 = staged ? ks : hh, c2 = staged ? 0 : tok;
        uint8_t* sa = smem + s * SBY;
        uint8_t* sb = sa + ABY;
        if (leader) mbar_expect_tx(&full_bar[s], 2 * SBY);
        tma_load_4d_2sm(sa, &tmap, &full_bar[s], c0, c1, c2, rowA + (part == 2 ? lo_rows : 0));
        if (WIDE)
          tma_load_4d_2sm(sa + A_BYTES, &tmap, &full_bar[s], c0, c1, c2,
                          rowA + BM + (part == 2 ? lo_rows : 0));
        tma_load_4d_2sm(sb, &tmap, &full_bar[s], c0, c1, c2, rowB + (part == 1 ? lo_rows : 0));
      }
    }
  } else if (warp == 3 && !leader && gathered == 2) {
    // LSU-gather relay (peer CTA): a stage's cp.async copies complete on this CTA's
    // full_loc barrier; make them visible to the async proxy and tell the leader's MMA
    if (lane == 0) {
      uint32_t kk = 0;
      for (uint32_t it = 0;; ++it) {
        const int sl = it % SCHED_DEPTH;
        mbar_wait_cluster(&sched_full[sl], (it / SCHED_DEPTH) & 1);
        const int w = sched_rec[sl * kRec];
        mbar_arrive_cluster(&sched_empty[sl], 0);
        if (w < 0) break;
        for (int ks = 0; ks < nk; ++ks, ++kk) {
          const int s = kk % STG;
          mbar_wait(&full_loc[s], (kk / STG) & 1);
          fence_proxy_async_smem();
          mbar_arrive_cluster(&full_bar[s], 0);
        }
      }
    }
  } else if (warp == 3) {
    // tile scheduler (leader CTA): fetch the next work item with alive blocks,
    // resolve its geometry, publish the record to both CTAs, SCHED_DEPTH ahead
    if (leader && lane == 0) {
      for (uint32_t it = 0;; ++it) {
        const int sl = it % SCHED_DEPTH;
        mbar_wait_cluster(&sched_empty[sl], ((it / SCHED_DEPTH) & 1) ^ 1);
        int w;
        TileInfo t0;
        for (;;) {
          w = atomicAdd(work_counter, 1);
          if (w >= nwork) {
            if (w == nwork + P - 1) atomicExch(work_counter, 0);  // last fetch of the launch
            w = -1;
            break;
          }
          t0 = tile_info(w / nsplit, nt, u0, g, merges, tiles, rank, staged);
          if (t0.active) break;
          const int tile = w / nsplit - (int)t0.ul * nt;  // tile fully beyond the alive blocks
          double* pp = partials + ((int64_t)t0.ul * nt + tile) * kTcPartialsPerTile * 5;
          for (int q = 0; q < kTcPartialsPerTile; ++q) {
            pp[5 * q + 0] = pp[5 * q + 1] = pp[5 * q + 2] = 0.0;
            pp[5 * q + 3] = INFINITY;
            pp[5 * q + 4] = -INFINITY;
          }
        }
        // r[0] = tile work id (w / nsplit), r[10] = k-split
        int32_t r[kRec] = {w < 0 ? -1 : w / nsplit, 0, 0, 0, 0, 0, 0, 0, 0, 0, w < 0 ? 0 : w % nsplit, 0};
        if (w >= 0) {
          r[1] = t0.m; r[2] = t0.i0; r[3] = t0.j0; r[4] = t0.lb; r[5] = t0.mid; r[6] = t0.re;
          r[7] = t0.pl; r[8] = t0.pm; r[9] = t0.pr;
        }
        int32_t* dst = sched_rec + sl * kRec;
#pragma unroll
        for (int q = 0; q < 11; ++q) {
          dst[q] = r[q];
          st_cluster_s32(dst + q, 1, r[q]);
        }
        mbar_arrive_cluster(&sched_full[sl], 0);
        mbar_arrive_cluster(&sched_full[sl], 1);
        if (w < 0) break;
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      uint32_t kk = 0, tc = 0;
      for (uint32_t it = 0;; ++it) {
        const int sl = it % SCHED_DEPTH;
        mbar_wait_cluster(&sched_full[sl], (it / SCHED_DEPTH) & 1);
        const int w = sched_rec[sl * kRec];
        const int sk = sched_rec[sl * kRec + 10];
        mbar_arrive_cluster(&sched_empty[sl], 0);
        if (w < 0) break;
        const int nks = (int)((int64_t)(sk + 1) * nk_run / nsplit) - (int)((int64_t)sk * nk_run / nsplit);
        const uint32_t acc = tc % NACC;
        mbar_wait_cluster(&tmem_empty[acc], ((tc / NACC) & 1) ^ 1);  // epilogue drained it
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dst = tmem_base + acc * BN;  // wide: rows half h at columns h * BN
        for (int ks = 0; ks < nks; ++ks, ++kk) {
          const int s = kk % STG;
          const uint32_t ph = (kk / STG) & 1;
          mbar_wait(&full_bar[s], ph);
          if (gathered == 2) {  // LSU gather: the peer's rows (relay above), then our own
            mbar_wait(&full_loc[s], ph);
            fence_proxy_async_smem();
          }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * SBY);
          const uint32_t sb = sa + ABY;
#pragma unroll
          for (int hh = 0; hh < (WIDE ? 2 : 1); ++hh)
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_2sm(dst + hh * BN, sw128_desc(sa + hh * A_BYTES + k * 32),
                            sw128_desc(sb + k * 32), (ks | k) != 0);
          umma_commit_2sm(&empty_bar[s]);
          if (fnorm) umma_commit_2sm(&mma_done[s]);  // the stage is readable by the norm warps
        }
        umma_commit_2sm(&tmem_full[acc]);
        ++tc;
      }
    }
  } else if (warp >= 4) {
    // Epilogue. Column metadata (inverse norms, masks, block ids) and the per-column
    // first-match minima are double-buffered by tile parity, so a tile needs one
    // barrier (its metadata is written); the minima of tile k are flushed to the
    // global absorbers after tile k+1's barrier (every warp is past tile k then),
    // and each warp writes its own moment slot (reduced in fixed order by
    // level_stats), so no warp waits for another at the end of a tile.
    const int ew = warp - 4;
    const int quarter = ew & 3;           // TMEM lanes [32*quarter, 32*quarter + 32)
    // narrow: two warps per lane quarter split the 256 columns; wide: they take the two
    // 128-row halves of the CTA's 256 rows (TMEM columns [h * BN, h * BN + BN)), all columns
    const int rh = WIDE ? (ew >> 2) : 0;
    const int col0 = WIDE ? 0 : (ew >> 2) * (BN / 2);
    const int col1 = WIDE ? BN : col0 + BN / 2;
    const int row = rh * BM + quarter * 32 + lane;
    const int et = threadIdx.x - 128;
    constexpr int ET = 32 * EPI_WARPS;
    static_assert(ET >= BN, "one epilogue thread per column for the flush");
    uint32_t tc = 0;
    uint32_t kn = 0;  // fnorm: ring position of the norm pass (the MMA warp's k-step sequence)
    int64_t prev_gb = -1;  // unit base of the tile whose minima are pending
    auto flush = [&](int buf) {  // thread et owns column et of buffer buf
      if (et < BN && prev_gb >= 0) {
        int32_t* cmin = colmin_b + buf * BN;
        const int32_t cm = cmin[et];
        if (cm != kNone) atomicMin(&absorber[prev_gb + colid_b[buf * BN + et]], cm);
        cmin[et] = kNone;
      }
    };
    for (uint32_t it = 0;; ++it) {
      const int sl = it % SCHED_DEPTH;
      mbar_wait_cluster(&sched_full[sl], (it / SCHED_DEPTH) & 1);
      const int w = sched_rec[sl * kRec];
      const int sk = sched_rec[sl * kRec + 10];
      TileInfo t = rec_info(sched_rec + sl * kRec, nt, u0);
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&sched_empty[sl], 0);
      if (w < 0) break;
      bool dead = false;
      if (paired) pair_view(t, crank, merges, nm, dead);
      const int cbeg = paired ? (int)crank * BNH : 0;  // first column of this CTA's merge
      const int mb = (int)(tc & 1);  // metadata buffer of this tile
      float* inv_j = inv_j_b + mb * BN;
      int32_t* colmin = colmin_b + mb * BN;
      uint8_t* ok_j = ok_j_b + mb * BN;
      int32_t* colid = colid_b + mb * BN;
      const int tile = w - (int)t.ul * nt;
      double* pp = partials + (((int64_t)t.ul * nt + tile) * kTcPartialsPerTile + crank * EPI_WARPS + ew) * 5;
      const int64_t gb = t.u * g.NB;
      const int32_t* lv = live + gb;
      const int mi0 = t.i0 + (int)crank * BMC;
      const int ni = dead ? 0 : max(0, min(BMC, t.pm - t.pl - mi0));  // valid rows of this CTA
      const int nj = dead ? cbeg : min(BN, t.pr - t.pm - t.j0);        // columns [cbeg, nj)
      if (fnorm) {
        // Key norms of the rows this CTA streams (level 1: every block is an operand row of
        // exactly one tile), read from the ring after the MMAs: thread et takes A row et
        // or B row et - BM; 8-element fp32 partials of exact bf16 squares summed in float64,
        // as block_norms_flat_kernel does. The stage is released to the producer by the MMA
        // commit plus one arrival per norm warp.
        const int nrow = et & (BM - 1);
        const bool isA = et < BM;
        const uint32_t roff = (isA ? 0u : (uint32_t)A_BYTES) + (uint32_t)nrow * 128u;
        double nacc8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // one chain per chunk slot
        for (int ks = 0; ks < nk_run; ++ks, ++kn) {
          const int s = kn % STG;
          if (lane == 0) mbar_wait(&mma_done[s], (kn / STG) & 1);  // one poller per warp
          __syncwarp();
          const uint32_t rp = smem_u32(smem + s * SBY) + roff;
          uint4 q[8];
#pragma unroll
          for (int c = 0; c < 8; ++c)  // 16-B chunk c of the row sits at chunk c ^ (row % 8)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(q[c].x), "=r"(q[c].y), "=r"(q[c].z), "=r"(q[c].w)
                         : "r"(rp + ((uint32_t)(c ^ (nrow & 7)) << 4))
                         : "memory");
          __syncwarp();  // the row is in registers: release the stage before the math
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty_bar[s])) : "memory");
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&q[c]);
            float a = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(p2[e]);
              a = fmaf(f.x, f.x, a);
              a = fmaf(f.y, f.y, a);
            }
            nacc8[c] += a;  // independent float64 chains (the sum is exact in practice)
          }
        }
        const double nacc = ((nacc8[0] + nacc8[1]) + (nacc8[2] + nacc8[3])) +
                            ((nacc8[4] + nacc8[5]) + (nacc8[6] + nacc8[7]));
        const float nv = (float)sqrt(nacc);
        if (isA) {
          anorm_b[mb * BM + nrow] = nv;
          if (nrow < ni) {
            knorm[gb + t.lb + mi0 + nrow] = nv;
            fusable[gb + t.lb + mi0 + nrow] = nv > 0.f ? 1 : 0;
          }
        } else {
          const int cg = (int)crank * BNH + nrow;  // column of the pair tile
          bnorm_b[mb * BN + cg] = nv;
          asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(cluster_addr(&bnorm_b[mb * BN + cg], crank ^ 1)),
                       "f"(nv)
                       : "memory");
          if (cg < nj) {
            knorm[gb + t.mid + t.j0 + cg] = nv;
            fusable[gb + t.mid + t.j0 + cg] = nv > 0.f ? 1 : 0;
          }
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(&norm_ready[mb], 0);
          mbar_arrive_cluster(&norm_ready[mb], 1);
        }
        mbar_wait_cluster(&norm_ready[mb], (tc >> 1) & 1);  // both CTAs' norms of this tile
      }
      for (int c = et; c < BN; c += ET) {  // column metadata
        const bool inc = c >= cbeg && c < nj;
        const int64_t bj = gb + (inc ? (staged ? lv[t.pm + t.j0 + c] : t.mid + t.j0 + c) : 0);
        // independent loads (one round trip), combined afterwards
        const uint8_t al = alive[bj];
        const float nk = fnorm ? bnorm_b[mb * BN + c] : knorm[bj];
        const uint8_t fu = fnorm ? (nk > 0.f ? 1 : 0) : fusable[bj];
        const bool ok = inc && al && fu;
        colid[c] = (int32_t)(bj - gb);
        const float nv = ok ? nk : 0.f;
        ok_j[c] = ok;
        inv_j[c] = nv > 0.f ? 1.f / nv : 0.f;
      }
      const int32_t my_id = row < ni ? (staged ? lv[t.pl + mi0 + row] : t.lb + mi0 + row) : 0;
      const int64_t bi = gb + my_id;
      const uint8_t al_i = alive[bi];
      const float nk_i = fnorm ? anorm_b[mb * BM + row] : knorm[bi];
      const uint8_t fu_i = fnorm ? (nk_i > 0.f ? 1 : 0) : fusable[bi];
      const bool ok_i = row < ni && al_i && fu_i;
      const float ni_v = ok_i ? nk_i : 0.f;
      const float inv_i = ni_v > 0.f ? 1.f / ni_v : 0.f;
      float s1 = 0.f, s2 = 0.f, mn = INFINITY, mx = -INFINITY;
      int cnt = 0;
      double* samp = samples ? samples + t.ul * sample_stride + sample_off[t.m] : nullptr;
      asm volatile("bar.sync 1, %0;" ::"n"(ET) : "memory");  // column metadata visible
      if (nsplit > 1) {  // the previous tile's first matches (every warp is past it)
        flush(mb ^ 1);
        prev_gb = gb;
      }

      const uint32_t acc = tc % NACC;
      mbar_wait(&tmem_full[acc], (tc / NACC) & 1);
      const uint32_t tcol = WIDE ? rh * BN : acc * BN;  // this warp's accumulator columns
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (nsplit > 1) {
        // this split's partial accumulator -> spart[(tile, split, CTA)][col][row]
        // (column-major: a warp's 32 rows are one 128-B line per column)
        float* mine = spart + (((int64_t)w * nsplit + sk) * 2 + crank) * (int64_t)(BMC * BN);
        for (int c0 = col0; c0 < col1; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + tcol + c0, v);
#pragma unroll
          for (int c = 0; c < 32; ++c) mine[(int64_t)(c0 + c) * BMC + row] = __uint_as_float(v[c]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tmem_empty[acc], 0);  // accumulator free already
        __threadfence();
        asm volatile("bar.sync 2, %0;" ::"n"(ET) : "memory");
        if (et == 0) {
          int32_t* cp = scnt + (int64_t)w * 2 + crank;
          const int old = atomicAdd(cp, 1);
          split_last_sh = old == nsplit - 1;
          if (old == nsplit - 1) *cp = 0;  // reset for the next launch
        }
        asm volatile("bar.sync 2, %0;" ::"n"(ET) : "memory");
        const bool last = split_last_sh != 0;
        __threadfence();
        if (!last) {  // another split of this tile finishes it; no moments, no decisions
          ++tc;
          continue;
        }
      }
      // accumulator chunk c0 of this thread's row: TMEM, or the sum of the tile's
      // split partials in split order (bitwise reproducible)
      auto load_acc = [&](int c0, uint32_t (&v)[32]) {
        if (nsplit == 1) {
          tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + tcol + c0, v);
          return;
        }
        const float* p0 = spart + ((int64_t)w * nsplit * 2 + crank) * (int64_t)(BMC * BN) +
                          (int64_t)c0 * BMC + row;
        float a[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) a[c] = 0.f;
        for (int s = 0; s < nsplit; ++s) {  // 32 independent L2 loads in flight per split
          const float* ps = p0 + (int64_t)s * 2 * BMC * BN;
          float x[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) x[c] = __ldcg(ps + (int64_t)c * BMC);
#pragma unroll
          for (int c = 0; c < 32; ++c) a[c] += x[c];
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(a[c]);
      };
      // pairs with s > tlo take the slow path: threshold decision, or deferral
      // of near-threshold pairs to the exact float64 re-score (the tensor-core
      // fp32 accumulation over r/16 steps can be off by ~1e-4 relative)
      const float tlo = resc != nullptr ? thr - resc_band : thr;
      // fast path in row-scaled space: t = acc * inv_j, s = inv_i * t (inv_i >= 0), so the
      // row's sum / sum of squares / min / max of s follow from those of t; a column is a
      // candidate when t clears a slightly lowered row threshold, and only candidate
      // columns re-evaluate s exactly as below (bitwise the same decisions)
      const float tcand = ok_i && inv_i > 0.f ? (tlo - 1e-5f) / inv_i : INFINITY;
      float r1 = 0.f, r2 = 0.f, rmn = INFINITY, rmx = -INFINITY;
      // exact decisions for this thread's candidate columns (bit c of `cols`): no warp
      // collectives; a match lowers the column's first matching row in shared memory
      auto exact_cols = [&](const uint32_t (&v)[32], int c0, unsigned okm, unsigned cols) {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          if (!((cols >> c) & 1u)) continue;  // static c keeps v in registers
          const int col = c0 + c;
          if (!(ok_i && ((okm >> c) & 1u))) continue;
          const float sv = __uint_as_float(v[c]) * inv_i * inv_j[col];
          if (!(sv > tlo)) continue;
          bool hit = sv > thr;
          if (resc != nullptr && fabsf(sv - thr) <= resc_band) {
            const int pos = atomicAdd(resc_count, 1);
            if (pos < resc_cap) {
              int4 e;
              e.x = (int)t.u;
              e.y = my_id;
              e.z = colid[col];
              e.w = t.m;
              reinterpret_cast<int4*>(resc)[pos] = e;
              hit = false;  // decided by the re-score
            }
          }
          if (hit) atomicMin(&colmin[col], my_id);
        }
      };
      for (int c0 = col0; c0 < col1; c0 += 32) {
        uint32_t v[32];
        load_acc(c0, v);
        // columns of this chunk that take part (alive, fusable, inside the merge)
        const unsigned okm = __ballot_sync(0xffffffffu, ok_j[c0 + lane] != 0);
        if (ok_i) cnt += __popc(okm);
        if (samp) {  // small runs that keep every sample: per-element reference path
          for (int c = 0; c < 32; ++c) {
            const int col = c0 + c;
            const bool ok = ok_i && ((okm >> c) & 1u);
            const float sv = __uint_as_float(v[c]) * inv_i * inv_j[col];
            if (ok) {
              s1 += sv;
              s2 = fmaf(sv, sv, s2);
              mn = fminf(mn, sv);
              mx = fmaxf(mx, sv);
            }
            if (row < ni && col >= cbeg && col < nj)
              samp[(int64_t)(my_id - t.lb) * (t.re - t.mid) + (colid[col] - t.mid)] =
                  ok ? (double)sv : (double)NAN;
          }
          exact_cols(v, c0, okm, 0xffffffffu);
          continue;
        }
        unsigned cand = 0;
        if (okm == 0xffffffffu) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float tv = __uint_as_float(v[c]) * inv_j[c0 + c];
            r1 += tv;
            r2 = fmaf(tv, tv, r2);
            rmn = fminf(rmn, tv);
            rmx = fmaxf(rmx, tv);
            cand |= (tv > tcand ? 1u : 0u) << c;
          }
        } else if (okm) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            if (!((okm >> c) & 1u)) continue;  // warp-uniform
            const float tv = __uint_as_float(v[c]) * inv_j[c0 + c];
            r1 += tv;
            r2 = fmaf(tv, tv, r2);
            rmn = fminf(rmn, tv);
            rmx = fmaxf(rmx, tv);
            cand |= (tv > tcand ? 1u : 0u) << c;
          }
        }
        if (cand) exact_cols(v, c0, okm, cand);
      }
      if (ok_i && !samp) {  // row moments back to similarity space
        s1 += inv_i * r1;
        s2 = fmaf(inv_i * inv_i, r2, s2);
        if (rmn <= rmx) {
          mn = fminf(mn, inv_i * rmn);
          mx = fmaxf(mx, inv_i * rmx);
        }
      }
      // accumulator drained: hand the buffer back to the MMA warp (split tiles did above)
      if (nsplit == 1) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tmem_empty[acc], 0);
        // the previous tile's first matches, flushed only now: the cluster-scope release
        // of the arrive above waits for this thread's outstanding global atomics, so the
        // flush no longer delays the MMA warp's next accumulator (short per-head tiles)
        flush(mb ^ 1);
        prev_gb = gb;
      }
      ++tc;
      // this warp's similarity moments -> its own slot (fp32 warp tree, fixed order)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (lane == 0) {
        pp[0] = (double)cnt;
        pp[1] = (double)s1;
        pp[2] = (double)s2;
        pp[3] = (double)mn;
        pp[4] = (double)mx;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(ET) : "memory");  // every warp past the last tile
    flush((int)((tc & 1) ^ 1));
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();  // both CTAs done with TMEM and smem before teardown
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
// Tile-scheduler counter of the persistent kernel, one per stream (the kernel
// leaves it at zero when it exits).
int32_t* work_counter(cudaStream_t s) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, int32_t*> counters;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(s) << 8) ^ (uint64_t)dev;
  std::lock_guard<std::mutex> lk(mu);
  auto it = counters.find(key);
  if (it != counters.end()) return it->second;
  int32_t* p = nullptr;
  if (cudaMalloc(&p, sizeof(int32_t)) != cudaSuccess || cudaMemset(p, 0, sizeof(int32_t)) != cudaSuccess)
    return nullptr;
  counters.emplace(key, p);
  return p;
}
}  // namespace

bool tc_supported(const SimArgs& a, const char** why) {
  if (a.dtype != BF16) {
    *why = "pool dtype is not bfloat16";
    return false;
  }
  if (a.g.d % BK != 0) {
    *why = "head dim must be a multiple of 64";
    return false;
  }
  if ((reinterpret_cast<uintptr_t>(a.pool) & 15) != 0) {
    *why = "pool pointer must be 16-byte aligned";
    return false;
  }
  if (a.g.L * a.g.NB * (a.split3 ? 2 : 1) >= (int64_t)INT32_MAX - 512) {
    *why = "too many pool rows for int32 TMA coordinates";
    return false;
  }
  int dev = 0, major = 0, minor = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) {
    *why = "tcgen05 kernels are built for sm_100a (B200)";
    return false;
  }
  if (!get_encode()) {
    *why = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  return true;
}

cudaError_t launch_sim_tc(const SimArgs& a, cudaStream_t s) {
  if (a.nt == 0 || a.nU == 0) return cudaSuccess;
  CUtensorMap tmap;
  const Geom& g = a.g;
  const bool compact = a.live != nullptr;
  const bool gathered = compact && a.staged == nullptr;  // alive rows straight from the pool
  // gathered rows: LSU cp.async (default) or TMA gather4 (KVF_GATHER4=1, A/B)
  static const int gmode = getenv("KVF_GATHER4") ? 1 : 2;
  const bool staged = compact && !gathered;
  if (gathered && g.head_mode) return cudaErrorInvalidValue;
  const cuuint64_t r = (cuuint64_t)g.r();
  const bool split3 = a.split3 != 0;
  if (split3 && compact) return cudaErrorInvalidValue;
  cuuint64_t dims[4] = {(cuuint64_t)g.d, (cuuint64_t)g.h, (cuuint64_t)g.t,
                        (cuuint64_t)(g.L * g.NB * (split3 ? 2 : 1))};
  cuuint64_t strides[3] = {(cuuint64_t)g.d * 2, (cuuint64_t)g.h * g.d * 2,
                           (cuuint64_t)g.t * g.h * g.d * 2};
  if (staged) {  // staged rows: [nU * NB][r] -> (64, r/64, 1, rows)
    dims[0] = BK;
    dims[1] = r / BK;
    dims[2] = 1;
    dims[3] = (cuuint64_t)(a.nU * g.NB);
    strides[0] = BK * 2;
    strides[1] = r * 2;
    strides[2] = r * 2;
  }
  cuuint32_t box[4] = {(cuuint32_t)BK, 1, 1, (cuuint32_t)BM};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult res;
  if (gathered) {  // folded pool as 2-D (E, rows); gather4 boxes are {64, 1}
    cuuint64_t d2[2] = {(cuuint64_t)g.E(), (cuuint64_t)(g.L * g.NB)};
    cuuint64_t s2[1] = {(cuuint64_t)g.E() * 2};
    cuuint32_t b2[2] = {(cuuint32_t)BK, 1};
    res = get_encode()(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.pool), d2, s2,
                       b2, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    res = get_encode()(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                       const_cast<void*>(staged ? a.staged : a.pool), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (res != CUDA_SUCCESS) return cudaErrorInvalidValue;
  const bool wide = a.wide != 0;
  if (wide && (gathered || a.nsplit > 1)) return cudaErrorInvalidValue;
  if (a.write_norms && (wide || compact || a.nsplit > 1 || split3))
    return cudaErrorInvalidValue;
  if (a.paired && (wide || compact)) return cudaErrorInvalidValue;
  auto kern = wide ? sim_tc_kernel<2 * BM> : sim_tc_kernel<BM>;
  const int smem_bytes = wide ? SMEM_BYTES_WIDE : SMEM_BYTES;
  static bool attr_set[2] = {false, false};
  if (!attr_set[wide]) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return e;
    attr_set[wide] = true;
  }
  float thr = (float)a.thr;
  if ((double)thr > a.thr) thr = nextafterf(thr, -INFINITY);  // (float)s > thr_f <=> s > thr
  static int max_clusters_v[2] = {0, 0};
  int& max_clusters = max_clusters_v[wide];
  if (max_clusters == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2, 1, 1);
    cfg.blockDim = dim3(NTHREADS, 1, 1);
    cfg.dynamicSmemBytes = smem_bytes;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      n = sms / 2;
    }
    max_clusters = n;
  }
  const int nsplit = a.nsplit > 1 && !gathered ? a.nsplit : 1;
  if (nsplit > 1 && (!a.split_part || !a.split_count)) return cudaErrorInvalidValue;
  const int64_t nwork = (int64_t)a.nt * a.nU * nsplit;
  if (nwork + max_clusters >= INT32_MAX) return cudaErrorInvalidValue;
  int32_t* counter = work_counter(s);
  if (counter == nullptr) return cudaErrorMemoryAllocation;
  dim3 grid(2 * (unsigned)std::min<int64_t>(nwork, max_clusters), 1);
  kern<<<grid, NTHREADS, smem_bytes, s>>>(
      tmap, g, a.u0, a.nU, (float*)const_cast<void*>(a.knorm), const_cast<uint8_t*>(a.fusable), a.alive,
      a.absorber, a.merges, a.tiles,
      a.nt, thr, a.partials, a.samples, a.sample_off, a.sample_stride, a.live, a.rank, a.resc,
      a.resc_count, (int)a.resc_cap, (float)a.resc_band, counter, gathered ? gmode : 0, split3 ? 1 : 0,
      nsplit, a.split_part, a.split_count, (const __nv_bfloat16*)a.pool, a.write_norms && !wide ? 1 : 0,
      a.nm, a.paired);
  return cudaGetLastError();
}

}  // namespace kvf
