// Chunked-prefill attention over a CFF-fused context with computation reuse
// ("any SA computation that
// involves a fused block can be reused in later chunks that comprise an
// instance of this block ... merging the SA of the fused components with that
// of the unique components (and rescaling)").
//
// Queries of chunk c of request b attend to the logical keys of chunks 0..c-1
// (all visible) and, causally, to chunk c's own keys. After CFF the earlier
// chunks' slots map to fused physical blocks, many of them several times:
// K_slot = k_scale[slot] * pool[phys], V_slot = v_scale[slot] * pool[phys]
// (core.py:303-304). Per physical block P the kernel computes S = Q K_P^T once;
// each slot s on P contributes logits k_scale[s] * S to the online softmax and
// v_scale[s] * exp(.) to one summed probability tile, so P V_P also runs once
// per block. Without dedup (`dedup = 0`) every slot is its own unit: the same
// kernel, used as the measured baseline.
//
// CTA = (query tile, kv head, request): 8 consumer warps (the GQA group's query
// heads x 16-token row tiles) + 1 TMA producer warp streaming the units' K/V
// head slices through a 12-stage ring. The unit list (runs of equal physical
// ids over the request's phys-sorted positions -- the decode schedule's
// `order`) is built in shared memory at CTA start. mma.sync m16n8k16, bf16 in,
// fp32 accumulate; query rows on M (the standard flash-attention layout).
#include "kernels.h"
#include "tma_util.cuh"

namespace kvf {

using namespace tma;
namespace {
constexpr int PF_CONS = 8;                 // consumer warps
constexpr int PF_THREADS = 32 * (PF_CONS + 1);
constexpr int PF_STAGES = 12;
constexpr int PF_MAXSLOTS = 2048;          // context blocks per request

__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
}  // namespace

template <int D, int T>
__global__ void __launch_bounds__(PF_THREADS, 1)
chunk_prefill_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                     const __nv_bfloat16* __restrict__ q, Geom g, int64_t layer,
                     const int32_t* __restrict__ table, const float* __restrict__ k_scale,
                     const float* __restrict__ v_scale, const int32_t* __restrict__ order,
                     int64_t p_blocks, int chunk_blocks, int chunk, int Hq, float sm_scale,
                     int dedup, float* __restrict__ out) {
  constexpr int HALVES = D / 64;
  constexpr int KS = D / 16;
  constexpr int NE = D / 8;
  constexpr int BOX = T * 128;
  constexpr int TENS = HALVES * BOX;
  constexpr int STAGE = 2 * TENS;
  static_assert(T == 16, "16-token blocks");
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* dsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + PF_STAGES * STAGE);
  uint64_t* empty = full + PF_STAGES;
  int32_t* u_phys = reinterpret_cast<int32_t*>(empty + PF_STAGES);  // [PF_MAXSLOTS]
  int32_t* u_beg = u_phys + PF_MAXSLOTS;                             // [PF_MAXSLOTS + 1]
  int32_t* u_kbase = u_beg + PF_MAXSLOTS + 1;                        // [PF_MAXSLOTS] causal key base, -1 = all visible
  float* s_ks = reinterpret_cast<float*>(u_kbase + PF_MAXSLOTS);     // [PF_MAXSLOTS]
  float* s_vs = s_ks + PF_MAXSLOTS;                                  // [PF_MAXSLOTS]
  int32_t* s_pos = reinterpret_cast<int32_t*>(s_vs + PF_MAXSLOTS);   // [PF_MAXSLOTS] scratch
  __shared__ int n_units, n_slots;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = Hq / g.h;
  const int rows_per_head = 16 * (PF_CONS / G);  // query tokens per CTA
  const int kvh = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int q0 = blockIdx.x * rows_per_head;     // chunk-local query token of the tile
  const int64_t unit = layer;                    // folded tables
  const int prev_blocks = chunk * chunk_blocks;  // blocks of the earlier chunks
  const int64_t slot0 = unit * g.NB + b * p_blocks;

  // ---- unit list: runs of equal phys over the request's sorted earlier-chunk positions ----
  if (warp == 0) {
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
        s_ks[j] = k_scale[slot0 + s_pos[j]] * sm_scale;
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
    // own chunk: block i holds chunk-local keys [16 i, 16 i + 16); only blocks
    // starting at or before the tile's last query token are visible
    const int last_q = q0 + rows_per_head - 1;
    const int n_own = min(chunk_blocks, last_q / T + 1);
    for (int i = lane; i < n_own; i += 32) {
      const int64_t sl = slot0 + prev_blocks + i;
      u_phys[nu + i] = table[sl];
      u_beg[nu + i] = n + i;
      u_kbase[nu + i] = i * T;
      s_ks[n + i] = k_scale[sl] * sm_scale;
      s_vs[n + i] = v_scale[sl];
    }
    if (lane == 0) {
      u_beg[nu + n_own] = n + n_own;
      n_units = nu + n_own;
      n_slots = n + n_own;
      for (int s = 0; s < PF_STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], PF_CONS);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const int nu = n_units;
  const int rowbase = (int)(layer * g.NB);

  if (warp == PF_CONS) {  // ---- TMA producer ----
    if (lane == 0) {
      for (int u = 0; u < nu; ++u) {
        const int s = u % PF_STAGES;
        mbar_wait(&empty[s], ((u / PF_STAGES) & 1) ^ 1);
        uint8_t* st = dsm + (size_t)s * STAGE;
        const int row = rowbase + u_phys[u];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[s], (uint32_t)STAGE);
#pragma unroll
        for (int hf = 0; hf < HALVES; ++hf) {
          tma4(st + hf * BOX, &kmap, &full[s], hf * 64, kvh, 0, row);
          tma4(st + TENS + hf * BOX, &vmap, &full[s], hf * 64, kvh, 0, row);
        }
      }
    }
    return;
  }

  // ---- consumers: warp = (query head of the group, 16-token row tile) ----
  const int tiles_per_head = PF_CONS / G;
  const int gq = warp / tiles_per_head;
  const int tsub = warp % tiles_per_head;
  const int qh = kvh * G + gq;
  const int grp = lane >> 2, tig = lane & 3;
  const int lr = lane & 7, lm = lane >> 3;
  const int qi0 = q0 + tsub * 16 + grp;  // chunk-local query tokens of rows grp, grp + 8
  const int64_t Tq = (int64_t)chunk_blocks * T;
  // Q fragments (A operand, rows = query tokens, k = head dim)
  uint32_t qa[KS][4];
  {
    const __nv_bfloat16* qb = q + ((b * Tq + qi0) * Hq + qh) * D;
    const int64_t rs8 = (int64_t)8 * Hq * D;  // 8 rows down
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int e = ks * 16 + 2 * tig;
      qa[ks][0] = *reinterpret_cast<const uint32_t*>(qb + e);
      qa[ks][1] = *reinterpret_cast<const uint32_t*>(qb + rs8 + e);
      qa[ks][2] = *reinterpret_cast<const uint32_t*>(qb + e + 8);
      qa[ks][3] = *reinterpret_cast<const uint32_t*>(qb + rs8 + e + 8);
    }
  }
  auto addr = [&](uint32_t base, int tok, int e) {
    const int hf = e >> 6, ch = (e & 63) >> 3;
    return base + (uint32_t)(hf * BOX + tok * 128 + ((ch ^ (tok & 7)) << 4));
  };
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};  // rows grp, grp + 8
  float o[NE][4];
#pragma unroll
  for (int et = 0; et < NE; ++et)
#pragma unroll
    for (int c = 0; c < 4; ++c) o[et][c] = 0.f;

  // units are consumed in groups of UG (UG * 16 keys per online-softmax step):
  // the QK products of the group are independent (ILP), the max / rescale once
  constexpr int UG = 4;
  for (int u0 = 0; u0 < nu; u0 += UG) {
    const int ng = min(UG, nu - u0);
    float sc[UG][2][4];
    uint32_t vmask = 0;  // bit (i * 8 + nn * 4 + c): logit visible (causal)
#pragma unroll
    for (int i = 0; i < UG; ++i) {
#pragma unroll
      for (int nn = 0; nn < 2; ++nn)
#pragma unroll
        for (int c = 0; c < 4; ++c) sc[i][nn][c] = 0.f;
      if (i < ng) {
        const int u = u0 + i;
        const int s = u % PF_STAGES;
        mbar_wait(&full[s], (u / PF_STAGES) & 1);
        const uint32_t kb = su32(dsm + (size_t)s * STAGE);
        // S = Q K^T: 16 query rows x 16 keys (2 n-tiles)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t r0, r1, r2, r3;
          ldsm_x4(addr(kb, (lm >> 1) * 8 + lr, ks * 16 + (lm & 1) * 8), r0, r1, r2, r3);
          mma16816_full(sc[i][0], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], r0, r1);
          mma16816_full(sc[i][1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], r2, r3);
        }
        const int kbase = u_kbase[u];
#pragma unroll
        for (int nn = 0; nn < 2; ++nn)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int key = kbase + nn * 8 + 2 * tig + (c & 1);
            const int qi = qi0 + ((c >> 1) ? 8 : 0);
            if (kbase < 0 || key <= qi) vmask |= 1u << (i * 8 + nn * 4 + c);
          }
      }
    }
    // online softmax over the group's slots (logits = k_scale[s] * S)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < UG; ++i) {
      if (i >= ng) break;
      const int sb = u_beg[u0 + i], se = u_beg[u0 + i + 1];
      for (int r = sb; r < se; ++r) {
        const float ksr = s_ks[r];
#pragma unroll
        for (int nn = 0; nn < 2; ++nn)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if ((vmask >> (i * 8 + nn * 4 + c)) & 1u) mx[c >> 1] = fmaxf(mx[c >> 1], sc[i][nn][c] * ksr);
      }
    }
    float alpha[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 1));
      mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 2));
      const float m_new = fmaxf(m_run[hr], mx[hr]);
      alpha[hr] = m_new == -INFINITY ? 1.f : __expf(m_run[hr] - m_new);
      m_run[hr] = m_new;
      l_run[hr] *= alpha[hr];
    }
    if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
      for (int et = 0; et < NE; ++et) {
        o[et][0] *= alpha[0];
        o[et][1] *= alpha[0];
        o[et][2] *= alpha[1];
        o[et][3] *= alpha[1];
      }
    }
#pragma unroll
    for (int i = 0; i < UG; ++i) {
      if (i >= ng) break;
      const int u = u0 + i;
      const int s = u % PF_STAGES;
      const uint32_t vb = su32(dsm + (size_t)s * STAGE) + TENS;
      float pe[2][4];
#pragma unroll
      for (int nn = 0; nn < 2; ++nn)
#pragma unroll
        for (int c = 0; c < 4; ++c) pe[nn][c] = 0.f;
      const int sb = u_beg[u], se = u_beg[u + 1];
      for (int r = sb; r < se; ++r) {
        const float ksr = s_ks[r], vsr = s_vs[r];
#pragma unroll
        for (int nn = 0; nn < 2; ++nn)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float m = m_run[c >> 1];
            const bool v = (vmask >> (i * 8 + nn * 4 + c)) & 1u;
            const float pr = (v && m != -INFINITY) ? __expf(sc[i][nn][c] * ksr - m) : 0.f;
            l_run[c >> 1] += pr;
            pe[nn][c] = fmaf(pr, vsr, pe[nn][c]);
          }
      }
      // O += P_eff V: A = P_eff (C layout of S maps to the A layout), B = V
      const uint32_t a0 = pack_bf16(pe[0][0], pe[0][1]);
      const uint32_t a1 = pack_bf16(pe[0][2], pe[0][3]);
      const uint32_t a2 = pack_bf16(pe[1][0], pe[1][1]);
      const uint32_t a3 = pack_bf16(pe[1][2], pe[1][3]);
#pragma unroll
      for (int et = 0; et < NE; et += 2) {
        uint32_t r0, r1, r2, r3;
        ldsm_x4_t(addr(vb, (lm & 1) * 8 + lr, et * 8 + (lm >> 1) * 8), r0, r1, r2, r3);
        mma16816_full(o[et], a0, a1, a2, a3, r0, r1);
        mma16816_full(o[et + 1], a0, a1, a2, a3, r2, r3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&empty[s]);
    }
  }
  // ---- normalise and store: out[b][token][qh][d] (fp32) ----
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    float l = l_run[hr];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int qi = qi0 + hr * 8;
    float* op = out + ((b * Tq + qi) * Hq + qh) * D;
#pragma unroll
    for (int et = 0; et < NE; ++et)
      *reinterpret_cast<float2*>(op + et * 8 + 2 * tig) =
          make_float2(o[et][2 * hr] * inv, o[et][2 * hr + 1] * inv);
  }
}

namespace {
template <int D>
cudaError_t chunk_prefill_t(const ChunkPrefillArgs& a, cudaStream_t s) {
  CUtensorMap km, vm;
  if (!make_map(&km, a.pool_k, a.g) || !make_map(&vm, a.pool_v, a.g)) return cudaErrorInvalidValue;
  constexpr int STAGE = 2 * (D / 64) * 16 * 128;
  const int smem = 1024 + PF_STAGES * STAGE + 2 * PF_STAGES * 8 + PF_MAXSLOTS * 4 * 6 + 16;
  auto kern = chunk_prefill_kernel<D, 16>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int G = a.Hq / a.g.h;
  const int rows = 16 * (PF_CONS / G);
  const int64_t Tq = (int64_t)a.chunk_blocks * a.g.t;
  dim3 grid((unsigned)(Tq / rows), (unsigned)a.g.h, (unsigned)a.B);
  kern<<<grid, PF_THREADS, smem, s>>>(km, vm, (const __nv_bfloat16*)a.q, a.g, a.layer, a.table,
                                      a.k_scale, a.v_scale, a.order, a.p_blocks, a.chunk_blocks,
                                      a.chunk, a.Hq, (float)a.sm_scale, a.dedup, a.out);
  return cudaGetLastError();
}
}  // namespace

bool chunk_prefill_supported(const ChunkPrefillArgs& a, const char** why) {
  const int G = a.g.h > 0 ? a.Hq / a.g.h : 0;
  if (a.g.head_mode) return *why = "folded tables only", false;
  if (a.g.t != 16) return *why = "16-token blocks only", false;
  if (a.g.d != 64 && a.g.d != 128) return *why = "head dim must be 64 or 128", false;
  if (G < 1 || a.Hq % a.g.h || PF_CONS % G) return *why = "GQA group must divide 8", false;
  if (a.p_blocks > PF_MAXSLOTS) return *why = "more than 2048 blocks per request", false;
  if (a.chunk < 0 || (int64_t)(a.chunk + 1) * a.chunk_blocks > a.p_blocks)
    return *why = "chunk outside the request", false;
  if (((int64_t)a.chunk_blocks * a.g.t) % (16 * (PF_CONS / G)))
    return *why = "chunk tokens must be a multiple of the query tile", false;
  return true;
}

cudaError_t launch_chunk_prefill(const ChunkPrefillArgs& a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  if (a.g.d == 128) return chunk_prefill_t<128>(a, s);
  return chunk_prefill_t<64>(a, s);
}

}  // namespace kvf
