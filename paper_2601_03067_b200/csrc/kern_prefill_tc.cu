// Chunked-prefill attention with computation reuse on the 5th-gen tensor cores
// (the tcgen05 counterpart of kern_prefill.cu; same semantics, same unit list).
//
// CTA = 128 query rows = (128 / G) chunk tokens x the G query heads of one KV
// head (row r = token * G + head), one request. Per unit (a distinct physical
// block of the earlier chunks, or one own-chunk block):
//   S  = Q K_P^T          tcgen05.mma M128 N16 K128 -> TMEM (double-buffered)
//   softmax warpgroup     thread = TMEM lane = query row: logits = k_scale[s] S
//                         for every slot s on P (causal mask on own-chunk keys),
//                         running max / sum in registers, P_eff = sum_s
//                         v_scale[s] exp(.) -> bf16 into smem (UMMA A layout);
//                         O rescaled in TMEM only when a row's max moved
//   O += P_eff V_P        tcgen05.mma M128 N=d K16 (V read MN-major) -> TMEM
// Roles: warp 0 TMA producer (Q once, K/V ring), warp 1 MMA issuer, warps 2-5
// and 6-9 the softmax / epilogue warpgroups of two query tiles that share every
// K/V stage (ping-pong: one tile's softmax overlaps the other's MMAs). Reference: attention.py:58-80 generalised to chunked
// causal prefill over the refolded fused view (core.py:285-305).
#include "kernels.h"
#include "tma_util.cuh"
#include "umma_util.cuh"

namespace kvf {

using namespace tma;
using namespace umma_util;
namespace {
constexpr int PT_STAGES = 8;  // >= 2 groups: group g+1's loads reuse group g-1's stages
constexpr int PT_TILES = 2;     // query tiles per CTA (ping-pong softmax warpgroups)
constexpr int PT_THREADS = 64 + PT_TILES * 128;
constexpr int PT_MAXSLOTS = 1024;
constexpr int PT_ROWS = 128;    // rows per query tile

}  // namespace

template <int D>
__global__ void __launch_bounds__(PT_THREADS, 1)
chunk_prefill_tc_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                        const __grid_constant__ CUtensorMap qmap, Geom g, int64_t layer,
                        const int32_t* __restrict__ table, const float* __restrict__ k_scale,
                        const float* __restrict__ v_scale, const int32_t* __restrict__ order,
                        int64_t p_blocks, int chunk_blocks, int chunk, int Hq, float sm_scale,
                        int dedup, float* __restrict__ out) {
  constexpr int T = 16;
  constexpr int HALVES = D / 64;
  constexpr int BOX = T * 128;            // one (block, d half) box: 16 rows x 128 B
  constexpr int STAGE = 2 * HALVES * BOX;  // bytes one unit's K + V bring in
  // K and V live in per-half rings (unit u, half h at ring_h + (u % STAGES) BOX):
  // the UG consecutive units of a group are then contiguous 16-row slabs, i.e.
  // one 64-row UMMA operand (S: N = 64; P V: K = 64)
  constexpr int RING = PT_STAGES * BOX;
  constexpr int QBYTES = PT_ROWS * D * 2;  // Q tile, SW128 K-major, HALVES x 16 KB
  constexpr int UG = 4;                     // units per group (64 keys per softmax step)
  static_assert(PT_STAGES >= 2 * UG, "the MMA issuer waits a whole group's K/V before releasing the previous one");
  constexpr int PBYTES = PT_ROWS * UG * 16 * 2;  // P of a group: 128 rows x 64 keys bf16
  constexpr int PSBO = UG * 16 * 2 * 8;          // 8-row group stride of the P tile (1 KB)
  // TMEM: O of tile t at [t D, (t+1) D); S buffers of tile t at 2D + t (2 UG 16) + b (UG 16)
  constexpr int SCOL = PT_TILES * D;
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* dsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = dsm;                                  // [PT_TILES] Q tiles
  uint8_t* sK = sQ + PT_TILES * QBYTES;               // [HALVES] rings
  uint8_t* sV = sK + HALVES * RING;                   // [HALVES] rings
  uint8_t* sP = sV + HALVES * RING;                   // [PT_TILES][2] P buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + PT_TILES * 2 * PBYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + PT_STAGES;
  uint64_t* s_full = k_empty + PT_STAGES;  // [PT_TILES][2]
  uint64_t* s_empty = s_full + 2 * PT_TILES;
  uint64_t* p_full = s_empty + 2 * PT_TILES;
  uint64_t* p_empty = p_full + 2 * PT_TILES;
  uint64_t* pv_done = p_empty + 2 * PT_TILES;  // [PT_TILES]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + PT_TILES);
  int32_t* u_phys = reinterpret_cast<int32_t*>(tmem_slot + 2);
  int32_t* u_beg = u_phys + PT_MAXSLOTS;
  int32_t* u_kbase = u_beg + PT_MAXSLOTS + 1;
  float* s_ks = reinterpret_cast<float*>(u_kbase + PT_MAXSLOTS);
  float* s_vs = s_ks + PT_MAXSLOTS;
  int32_t* s_pos = reinterpret_cast<int32_t*>(s_vs + PT_MAXSLOTS);
  __shared__ int n_units;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = Hq / g.h;
  const int tok_per_tile = PT_ROWS / G;
  const int tok_per_cta = PT_TILES * tok_per_tile;
  const int kvh = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int q0 = blockIdx.x * tok_per_cta;
  const int prev_blocks = chunk * chunk_blocks;
  const int64_t slot0 = layer * g.NB + b * p_blocks;
  const int64_t Tq = (int64_t)chunk_blocks * T;
  // logits kept in base 2 (k_scale * sm_scale * log2 e): p = 2^(S ks - m) is one FFMA + EX2
  const float sm_scale2 = sm_scale * 1.4426950408889634f;

  // ---- unit list (as kern_prefill.cu) ----
  if (warp == 2) {
    int n = 0;
    for (int j0 = 0; j0 < p_blocks; j0 += 32) {
      const int j = j0 + lane;
      const int pos = j < p_blocks ? order[b * p_blocks + j] : -1;
      const bool keep = pos >= 0 && pos < prev_blocks;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) s_pos[n + __popc(m & ((1u << lane) - 1u))] = pos;
      n += __popc(m);
    }
    __syncwarp();
    int nu = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      int32_t ph = -1, prv = -1;
      if (j < n) {
        ph = table[slot0 + s_pos[j]];
        if (j > 0) prv = table[slot0 + s_pos[j - 1]];
        s_ks[j] = k_scale[slot0 + s_pos[j]] * sm_scale2;
        s_vs[j] = v_scale[slot0 + s_pos[j]];
      }
      const bool start = j < n && (!dedup || j == 0 || ph != prv);
      const unsigned m = __ballot_sync(0xffffffffu, start);
      if (start) {
        const int ui = nu + __popc(m & ((1u << lane) - 1u));
        u_phys[ui] = ph;
        u_beg[ui] = j;
        u_kbase[ui] = -1;
      }
      nu += __popc(m);
    }
    const int last_q = q0 + tok_per_cta - 1;
    const int n_own = min(chunk_blocks, last_q / T + 1);
    for (int i = lane; i < n_own; i += 32) {
      const int64_t sl = slot0 + prev_blocks + i;
      u_phys[nu + i] = table[sl];
      u_beg[nu + i] = n + i;
      u_kbase[nu + i] = i * T;
      s_ks[n + i] = k_scale[sl] * sm_scale2;
      s_vs[n + i] = v_scale[sl];
    }
    if (lane == 0) {
      u_beg[nu + n_own] = n + n_own;
      n_units = nu + n_own;
      mbar_init(q_full, 1);
      for (int s = 0; s < PT_STAGES; ++s) {
        mbar_init(&k_full[s], 1);
        mbar_init(&k_empty[s], 1);
      }
      for (int i = 0; i < 2 * PT_TILES; ++i) {
        mbar_init(&s_full[i], 1);
        mbar_init(&s_empty[i], 4);
        mbar_init(&p_full[i], 4);
        mbar_init(&p_empty[i], 1);
      }
      for (int t = 0; t < PT_TILES; ++t) mbar_init(&pv_done[t], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int nu = n_units;
  const int rowbase = (int)(layer * g.NB);

  if (warp == 0) {  // ---- TMA producer ----
    if (lane == 0) {
      mbar_expect_tx(q_full, (uint32_t)(PT_TILES * QBYTES));
      for (int t = 0; t < PT_TILES; ++t)
        for (int hf = 0; hf < HALVES; ++hf)
          tma4(sQ + t * QBYTES + hf * (QBYTES / HALVES), &qmap, q_full, hf * 64, kvh * G,
               q0 + t * tok_per_tile, (int)b);
      for (int u = 0; u < nu; ++u) {
        const int s = u % PT_STAGES;
        mbar_wait(&k_empty[s], ((u / PT_STAGES) & 1) ^ 1);
        const int row = rowbase + u_phys[u];
        mbar_expect_tx(&k_full[s], (uint32_t)STAGE);
#pragma unroll
        for (int hf = 0; hf < HALVES; ++hf) {
          tma4(sK + hf * RING + s * BOX, &kmap, &k_full[s], hf * 64, kvh, 0, row);
          tma4(sV + hf * RING + s * BOX, &vmap, &k_full[s], hf * 64, kvh, 0, row);
        }
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer ----
    if (lane == 0) {
      mbar_wait(q_full, 0);
      const int ngroups = (nu + UG - 1) / UG;
      for (int gi = 0; gi <= ngroups; ++gi) {
        if (gi < ngroups) {  // S of the group's units, both query tiles
          const int sb = gi & 1;
          const int u0 = gi * UG, ng = min(UG, nu - u0);
          for (int i = 0; i < ng; ++i) {
            const int u = u0 + i;
            const int s = u % PT_STAGES;
            mbar_wait(&k_full[s], (u / PT_STAGES) & 1);
          }
          const int s0 = u0 % PT_STAGES;  // the group's first slab (groups never wrap)
          for (int t = 0; t < PT_TILES; ++t) {
            mbar_wait(&s_empty[t * 2 + sb], ((gi >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t qa = su32(sQ + t * QBYTES);
#pragma unroll
            for (int hf = 0; hf < HALVES; ++hf)
#pragma unroll
              for (int k = 0; k < 4; ++k)
                umma(tmem + SCOL + t * 2 * UG * 16 + UG * 16 * sb,
                     desc_k128(qa + hf * (QBYTES / HALVES) + k * 32),
                     desc_k128(su32(sK + hf * RING + s0 * BOX) + k * 32), idesc(PT_ROWS, 16 * ng, false),
                     (hf | k) != 0);
            umma_commit(&s_full[t * 2 + sb]);
          }
        }
        if (gi >= 1) {  // O_t += P_t V over the previous group's 16 ng keys (K = 16 per MMA)
          const int gv = gi - 1;
          const int pb = gv & 1;
          const int u0 = gv * UG, ng = min(UG, nu - u0);
          const int s0 = u0 % PT_STAGES;
          for (int t = 0; t < PT_TILES; ++t) {
            mbar_wait(&p_full[t * 2 + pb], (gv >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t pa = su32(sP + (t * 2 + pb) * PBYTES);
            for (int i = 0; i < ng; ++i)
              umma(tmem + t * D, desc_interleave(pa + i * 256, 128, PSBO),
                   desc_mn128(su32(sV + (s0 + i) * BOX), RING, 1024), idesc(PT_ROWS, D, true),
                   (u0 + i) > 0);
            umma_commit(&p_empty[t * 2 + pb]);
            umma_commit(&pv_done[t]);
          }
          for (int i = 0; i < ng; ++i) umma_commit(&k_empty[s0 + i]);  // both tiles done
        }
      }
    }
  } else {  // ---- softmax / epilogue: thread = TMEM lane = query row of tile t ----
    const int t = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t ocol = t * D;
    const int tok = t * tok_per_tile + r / G;
    const int qi = q0 + tok;  // chunk-local query token
    float m_run = -INFINITY, l_run = 0.f;
    const int ngroups = (nu + UG - 1) / UG;
    for (int gi = 0; gi < ngroups; ++gi) {
      const int sb = gi & 1;
      const int u0 = gi * UG, ng = min(UG, nu - u0);
      mbar_wait(&s_full[t * 2 + sb], (gi >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float sv[UG][16];
#pragma unroll
      for (int i = 0; i < UG; ++i)
        if (i < ng) tld16(trow + SCOL + t * 2 * UG * 16 + 16 * (UG * sb + i), sv[i]);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive1(&s_empty[t * 2 + sb]);
      // group max over every slot of every unit (own-chunk units: causal). Slot
      // scales are >= 0 (norm ratios), so max_k(S_k ks) = ks max_k(S_k): one
      // max per unit, one multiply per slot
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < UG; ++i) {
        if (i >= ng) break;
        const int u = u0 + i;
        const int kbase = u_kbase[u];
        const int nvis = kbase < 0 ? 16 : max(0, min(16, qi - kbase + 1));
        float smax = -INFINITY;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < nvis) smax = fmaxf(smax, sv[i][k]);
        if (smax != -INFINITY)
          for (int sl = u_beg[u]; sl < u_beg[u + 1]; ++sl) mx = fmaxf(mx, smax * s_ks[sl]);
      }
      const float m_new = fmaxf(m_run, mx);
      const float alpha = m_new == -INFINITY ? 1.f : ex2(m_run - m_new);
      l_run *= alpha;
      m_run = m_new;
      // PV of the previous group has landed (waited every group, so the
      // barrier's phase never runs two ahead of this parity wait); O in TMEM is
      // rescaled only when a row's max moved
      if (gi > 0) {
        mbar_wait(&pv_done[t], (gi - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < D; c += 16) tld_st16(trow + ocol + c, alpha);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
      if (gi >= 2) mbar_wait(&p_empty[t * 2 + sb], ((gi >> 1) & 1) ^ 1);
#pragma unroll
      for (int i = 0; i < UG; ++i) {
        if (i >= ng) break;
        const int u = u0 + i;
        const int kbase = u_kbase[u];
        const int nvis = kbase < 0 ? 16 : max(0, min(16, qi - kbase + 1));
        float pe[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) pe[k] = 0.f;
        if (nvis == 16 && m_new != -INFINITY) {  // fully visible unit (earlier chunks)
          for (int sl = u_beg[u]; sl < u_beg[u + 1]; ++sl) {
            const float ks = s_ks[sl], vs = s_vs[sl];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const float p = ex2(fmaf(sv[i][k], ks, -m_new));
              l_run += p;
              pe[k] = fmaf(p, vs, pe[k]);
            }
          }
        } else if (nvis > 0 && m_new != -INFINITY) {  // causal own-chunk block
          for (int sl = u_beg[u]; sl < u_beg[u + 1]; ++sl) {
            const float ks = s_ks[sl], vs = s_vs[sl];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const float p = k < nvis ? ex2(fmaf(sv[i][k], ks, -m_new)) : 0.f;
              l_run += p;
              pe[k] = fmaf(p, vs, pe[k]);
            }
          }
        }
        // P_eff (bf16) into the UMMA A tile: 8 x 16 B core matrices, K chunks 128 B apart
        uint8_t* pt = sP + (t * 2 + sb) * PBYTES + (r >> 3) * PSBO + (r & 7) * 16 + i * 256;
        uint4 c0, c1;
        c0.x = pack_bf16(pe[0], pe[1]);
        c0.y = pack_bf16(pe[2], pe[3]);
        c0.z = pack_bf16(pe[4], pe[5]);
        c0.w = pack_bf16(pe[6], pe[7]);
        c1.x = pack_bf16(pe[8], pe[9]);
        c1.y = pack_bf16(pe[10], pe[11]);
        c1.z = pack_bf16(pe[12], pe[13]);
        c1.w = pack_bf16(pe[14], pe[15]);
        *reinterpret_cast<uint4*>(pt) = c0;
        *reinterpret_cast<uint4*>(pt + 128) = c1;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive1(&p_full[t * 2 + sb]);
    }
    if (ngroups > 0) mbar_wait(&pv_done[t], (ngroups - 1) & 1);
    // ---- epilogue: O / l -> out[b][q0 + tok][kvh * G + head][:] ----
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    float* op = out + ((b * Tq + qi) * Hq + kvh * G + (r % G)) * D;
#pragma unroll
    for (int c = 0; c < D; c += 16) {
      float v[16];
      tld16(trow + ocol + c, v);
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        *reinterpret_cast<float4*>(op + c + i) = make_float4(v[i] * inv, v[i + 1] * inv, v[i + 2] * inv, v[i + 3] * inv);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

namespace {
bool make_qmap(CUtensorMap* m, const void* q, int64_t B, int64_t Tq, int Hq, int d, int G) {
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)Hq, (cuuint64_t)Tq, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)Hq * d * 2, (cuuint64_t)Tq * Hq * d * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)G, (cuuint32_t)(PT_ROWS / G), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(q), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
cudaError_t prefill_tc_t(const ChunkPrefillArgs& a, cudaStream_t s) {
  const int G = a.Hq / a.g.h;
  const int64_t Tq = (int64_t)a.chunk_blocks * a.g.t;
  CUtensorMap km, vm, qm;
  if (!make_map(&km, a.pool_k, a.g) || !make_map(&vm, a.pool_v, a.g) ||
      !make_qmap(&qm, a.q, a.B, Tq, a.Hq, D, G))
    return cudaErrorInvalidValue;
  constexpr int STAGE = 2 * (D / 64) * 16 * 128;
  const int smem = 1024 + PT_TILES * PT_ROWS * D * 2 + PT_STAGES * STAGE + PT_TILES * 2 * 4 * PT_ROWS * 32 + 64 * 8 +
                   PT_MAXSLOTS * 4 * 6 + 64;
  auto kern = chunk_prefill_tc_kernel<D>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((unsigned)(Tq / (PT_TILES * PT_ROWS / G)), (unsigned)a.g.h, (unsigned)a.B);
  kern<<<grid, PT_THREADS, smem, s>>>(km, vm, qm, a.g, a.layer, a.table, a.k_scale, a.v_scale,
                                      a.order, a.p_blocks, a.chunk_blocks, a.chunk, a.Hq,
                                      (float)a.sm_scale, a.dedup, a.out);
  return cudaGetLastError();
}
}  // namespace

bool chunk_prefill_tc_supported(const ChunkPrefillArgs& a) {
  const int G = a.g.h > 0 ? a.Hq / a.g.h : 0;
  if (a.g.d != 128 || a.g.t != 16 || a.g.head_mode) return false;
  if (G < 1 || PT_ROWS % G || a.Hq % a.g.h) return false;
  if (((int64_t)a.chunk_blocks * a.g.t) % (PT_TILES * PT_ROWS / G)) return false;
  if ((reinterpret_cast<uintptr_t>(a.q) & 15) != 0) return false;
  return a.p_blocks <= PT_MAXSLOTS;
}

cudaError_t launch_chunk_prefill_tc(const ChunkPrefillArgs& a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  return prefill_tc_t<128>(a, s);
}

}  // namespace kvf
