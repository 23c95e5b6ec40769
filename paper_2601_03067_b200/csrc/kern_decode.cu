// K6: paged decode attention over the fused cache.
// Generalises the reference's exact single-query attention
// (attention.py:58-80 over refold, core.py:285-305) to a batch of requests,
// all query heads with GQA, and reads K/V straight from the fused pool:
//   K_slot = k_scale[slot] * pool_k[table[slot]]   (same for V)
// so shared physical blocks are never materialised per slot.
// Split-K (flash-decoding): CTA = (request, kv head, split of CB blocks),
// online softmax per query head of the GQA group, then a combine kernel.
#include "kernels.h"
#include <cstdlib>
#include <type_traits>
#include "vec_io.cuh"

namespace kvf {

namespace {
constexpr int CB = 16;       // blocks per split
constexpr int NTD = 128;     // threads per CTA
constexpr int MAXG = 8;      // max query heads per kv head
constexpr int MAXD = 128;    // max head dim
constexpr int MAXT = 32;     // max tokens per block

constexpr int CB_MIN = 4;    // smallest split of any path (workspace sizing)
int64_t nsplit_of(int64_t p_blocks, int cbs = CB) { return (p_blocks + cbs - 1) / cbs; }

template <typename A>
__device__ __forceinline__ A load_q(const void* q, int q_dtype, int64_t idx) {
  if (q_dtype == F64) return (A)((const double*)q)[idx];
  if (q_dtype == F32) return (A)((const float*)q)[idx];
  return (A)__bfloat162float(((const __nv_bfloat16*)q)[idx]);
}
}  // namespace

int64_t decode_workspace_size(int dtype, int64_t B, int Hq, int d, int64_t p_blocks, int t) {
  const int64_t acc = dtype == F64 ? 8 : 4;
  return B * Hq * nsplit_of(p_blocks, CB_MIN) * (int64_t)(d + 2) * acc;
}

template <typename T>
__global__ void __launch_bounds__(NTD)
decode_partial_kernel(const void* __restrict__ q, int q_dtype, const T* __restrict__ pool_k,
                      const T* __restrict__ pool_v, Geom g, int64_t layer,
                      const int32_t* __restrict__ table,
                      const typename AccOf<T>::type* __restrict__ k_scale,
                      const typename AccOf<T>::type* __restrict__ v_scale, int64_t p_blocks,
                      const int32_t* __restrict__ seq_blocks, int Hq,
                      typename AccOf<T>::type sm_scale, typename AccOf<T>::type* __restrict__ part,
                      typename AccOf<T>::type* __restrict__ probs) {
  using A = typename AccOf<T>::type;
  __shared__ A qs[MAXG][MAXD];
  __shared__ A ks[MAXT][MAXD + 1];
  __shared__ A logit[MAXG][MAXT];
  __shared__ A m_run[MAXG], l_run[MAXG], alpha[MAXG];

  const int d = g.d, t = g.t, h = g.h;
  const int G = Hq / h;
  const int64_t b = blockIdx.z;
  const int kvh = blockIdx.y;
  const int64_t split = blockIdx.x;
  const int64_t nsplit = gridDim.x;
  const int64_t unit = g.head_mode ? layer * h + kvh : layer;
  const int32_t* tab = table + unit * g.NB;
  const A* ksc = k_scale + unit * g.NB;
  const A* vsc = v_scale + unit * g.NB;
  const int64_t nblk = seq_blocks ? (int64_t)seq_blocks[b] : p_blocks;
  const int64_t j_begin = split * CB;
  const int64_t j_end = min((int64_t)(j_begin + CB), nblk);

  for (int x = threadIdx.x; x < G * d; x += NTD) {
    const int gg = x / d, e = x % d;
    qs[gg][e] = load_q<A>(q, q_dtype, (b * Hq + (int64_t)kvh * G + gg) * d + e);
  }
  if (threadIdx.x < MAXG) {
    m_run[threadIdx.x] = -INFINITY;
    l_run[threadIdx.x] = A(0);
  }
  // output accumulators: thread owns (gg, e) pairs x = threadIdx.x + k*NTD
  A o[(MAXG * MAXD) / NTD];
#pragma unroll
  for (int k = 0; k < (MAXG * MAXD) / NTD; ++k) o[k] = A(0);
  __syncthreads();

  const int64_t E = g.E();
  for (int64_t j = j_begin; j < j_end; ++j) {
    const int64_t slot = b * p_blocks + j;
    const int32_t phys = tab[slot];
    const A kscale = ksc[slot], vscale = vsc[slot];
    const T* kb = pool_k + (layer * g.NB + phys) * E + (int64_t)kvh * d;
    const T* vb = pool_v + (layer * g.NB + phys) * E + (int64_t)kvh * d;
    // K tile (t x d) -> smem
    for (int x = threadIdx.x; x < t * d; x += NTD) {
      const int tk = x / d, e = x % d;
      ks[tk][e] = to_acc(kb[(int64_t)tk * h * d + e]);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < G * t; x += NTD) {
      const int gg = x / t, tk = x % t;
      A acc = 0;
      for (int e = 0; e < d; ++e) acc += ks[tk][e] * qs[gg][e];
      logit[gg][tk] = acc * kscale * sm_scale;
    }
    __syncthreads();
    if (threadIdx.x < G) {
      const int gg = threadIdx.x;
      A mx = m_run[gg];
      for (int tk = 0; tk < t; ++tk) mx = max(mx, logit[gg][tk]);
      const A al = exp(m_run[gg] - mx);
      A l = l_run[gg] * al;
      for (int tk = 0; tk < t; ++tk) {
        if (probs) probs[((b * Hq + (int64_t)kvh * G + gg) * p_blocks + j) * t + tk] = logit[gg][tk];
        const A pv = exp(logit[gg][tk] - mx);
        logit[gg][tk] = pv;
        l += pv;
      }
      m_run[gg] = mx;
      l_run[gg] = l;
      alpha[gg] = al;
    }
    // V tile -> smem (reuse ks)
    for (int x = threadIdx.x; x < t * d; x += NTD) {
      const int tk = x / d, e = x % d;
      ks[tk][e] = to_acc(vb[(int64_t)tk * h * d + e]);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < (MAXG * MAXD) / NTD; ++k) {
      const int x = threadIdx.x + k * NTD;
      const int gg = x / d, e = x % d;
      if (gg < G) {
        A acc = 0;
        for (int tk = 0; tk < t; ++tk) acc += logit[gg][tk] * ks[tk][e];
        o[k] = o[k] * alpha[gg] + acc * vscale;
      }
    }
    __syncthreads();
  }
  // write partial: [b][qh][split][d + 2] = (o[0..d), m, l)
#pragma unroll
  for (int k = 0; k < (MAXG * MAXD) / NTD; ++k) {
    const int x = threadIdx.x + k * NTD;
    const int gg = x / d, e = x % d;
    if (gg < G) {
      A* pp = part + (((b * Hq + (int64_t)kvh * G + gg) * nsplit) + split) * (d + 2);
      pp[e] = o[k];
    }
  }
  if (threadIdx.x < G) {
    A* pp = part + (((b * Hq + (int64_t)kvh * G + threadIdx.x) * nsplit) + split) * (d + 2);
    pp[d] = m_run[threadIdx.x];
    pp[d + 1] = l_run[threadIdx.x];
  }
}

template <typename A>
__global__ void decode_combine_kernel(const A* __restrict__ part, int64_t nsplit, int d,
                                      int64_t p_blocks, int t, const int32_t* seq_blocks,
                                      int Hq, A* __restrict__ out, A* __restrict__ lse,
                                      A* __restrict__ probs, int cbs) {
  const int64_t bh = blockIdx.x;  // b * Hq + qh
  const A* pp = part + bh * nsplit * (d + 2);
  const int64_t b = bh / Hq;
  const int64_t nblk = seq_blocks ? (int64_t)seq_blocks[b] : p_blocks;
  const int64_t nused = (nblk + cbs - 1) / cbs;
  A M = -INFINITY;
  for (int64_t s = 0; s < nused; ++s) M = max(M, pp[s * (d + 2) + d]);
  A L = 0;
  for (int64_t s = 0; s < nused; ++s) L += pp[s * (d + 2) + d + 1] * exp(pp[s * (d + 2) + d] - M);
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    A acc = 0;
    for (int64_t s = 0; s < nused; ++s)
      acc += pp[s * (d + 2) + e] * exp(pp[s * (d + 2) + d] - M);
    out[bh * d + e] = acc / L;
  }
  if (threadIdx.x == 0) lse[bh] = M + log(L);
  if (probs) {
    const int64_t ntok = nblk * t;
    for (int64_t x = threadIdx.x; x < ntok; x += blockDim.x) {
      A* pr = probs + bh * p_blocks * t + x;
      *pr = exp(*pr - M) / L;
    }
  }
}

// ---------------------------------------------------------------------------
// Bandwidth path (bf16 / f32 pools, d in {64, 128}): CTA = (split of CB
// blocks, kv head, request) with one warp per query head of the GQA group.
// 32-token K/V tiles are gathered through the block table with cp.async
// (16-byte chunks, 3-stage ring, padded rows -> conflict-free smem), so every
// K/V byte is read from HBM once per (request, kv head) and shared by the
// group's warps. QK: lane = token, q broadcast from smem; PV: lane = 4 dims.
// ---------------------------------------------------------------------------
namespace {
constexpr int TOK = 32;
constexpr int STG = 3;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace

template <typename T, int D>
__global__ void __launch_bounds__(256)
decode_fast_kernel(const void* __restrict__ q, int q_dtype, const T* __restrict__ pool_k,
                   const T* __restrict__ pool_v, Geom g, int64_t layer,
                   const int32_t* __restrict__ table, const float* __restrict__ k_scale,
                   const float* __restrict__ v_scale, int64_t p_blocks,
                   const int32_t* __restrict__ seq_blocks, int Hq, float sm_scale,
                   float* __restrict__ part, float* __restrict__ probs) {
  constexpr int ROW = D * (int)sizeof(T) + 16;   // padded row bytes
  constexpr int CPR = D * (int)sizeof(T) / 16;   // 16-byte chunks per row
  constexpr int DPL = D / 32;                    // output dims per lane
  extern __shared__ __align__(16) uint8_t dsm[];
  uint8_t* kt = dsm;                              // [STG][TOK][ROW]
  uint8_t* vt = kt + STG * TOK * ROW;             // [STG][TOK][ROW]
  float* qs = reinterpret_cast<float*>(vt + STG * TOK * ROW);  // [G][D]
  float* sk = qs + 8 * D;                         // [STG][TOK]
  float* sv = sk + STG * TOK;                     // [STG][TOK]

  const int G = Hq / g.h;
  const int nthr = 32 * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.z;
  const int kvh = blockIdx.y;
  const int64_t split = blockIdx.x, nsplit = gridDim.x;
  const int64_t unit = g.head_mode ? layer * g.h + kvh : layer;
  const int32_t* tab = table + unit * g.NB;
  const float* ksc = k_scale + unit * g.NB;
  const float* vsc = v_scale + unit * g.NB;
  const int64_t nblk = seq_blocks ? (int64_t)seq_blocks[b] : p_blocks;
  const int64_t ntok = nblk * g.t;
  const int64_t T0 = split * (int64_t)CB * g.t;
  const int64_t T1 = min(T0 + (int64_t)CB * g.t, ntok);
  const int ntiles = T1 > T0 ? (int)((T1 - T0 + TOK - 1) / TOK) : 0;
  const int64_t E = g.E();
  const int64_t rstride = (int64_t)g.h * D;  // token stride inside a block

  for (int x = threadIdx.x; x < G * D; x += nthr) {
    const int gg = x / D, e = x % D;
    const int64_t qi = (b * Hq + (int64_t)kvh * G + gg) * D + e;
    qs[gg * D + e] = q_dtype == BF16 ? __bfloat162float(((const __nv_bfloat16*)q)[qi])
                                     : ((const float*)q)[qi];
  }

  auto issue = [&](int it) {
    const int st = it % STG;
    const int64_t tok0 = T0 + (int64_t)it * TOK;
    for (int c = threadIdx.x; c < TOK * CPR; c += nthr) {
      const int row = c / CPR, col = c % CPR;
      const int64_t tok = tok0 + row;
      const bool valid = tok < T1;
      const int64_t tk = valid ? tok : T0;
      const int64_t slot = b * p_blocks + tk / g.t;
      const int64_t off = (layer * g.NB + tab[slot]) * E + (tk % g.t) * rstride + (int64_t)kvh * D;
      cp_async16(kt + (st * TOK + row) * ROW + col * 16,
                 reinterpret_cast<const uint8_t*>(pool_k + off) + col * 16, valid);
      cp_async16(vt + (st * TOK + row) * ROW + col * 16,
                 reinterpret_cast<const uint8_t*>(pool_v + off) + col * 16, valid);
    }
    for (int row = threadIdx.x; row < TOK; row += nthr) {
      const int64_t tok = tok0 + row;
      const bool valid = tok < T1;
      const int64_t slot = b * p_blocks + (valid ? tok : T0) / g.t;
      sk[st * TOK + row] = valid ? ksc[slot] : 0.f;
      sv[st * TOK + row] = valid ? vsc[slot] : 0.f;
    }
    cp_commit();
  };

  float m_run = -INFINITY, l_run = 0.f;
  float o[DPL];
#pragma unroll
  for (int k = 0; k < DPL; ++k) o[k] = 0.f;
  const float* qg = qs + warp * D;

  for (int it = 0; it < STG - 1; ++it) {
    if (it < ntiles) issue(it);
    else cp_commit();
  }
  for (int it = 0; it < ntiles; ++it) {
    if (it + STG - 1 < ntiles) issue(it + STG - 1);
    else cp_commit();
    cp_wait<STG - 1>();
    __syncthreads();
    const int st = it % STG;
    const int64_t tok = T0 + (int64_t)it * TOK + lane;
    const bool valid = tok < T1;
    // ---- logits: lane = token ----
    const uint8_t* krow = kt + (st * TOK + lane) * ROW;
    float dot = 0.f;
#pragma unroll
    for (int c = 0; c < CPR; ++c) {
      constexpr int EPC = 16 / (int)sizeof(T);
      float kv[EPC];
      if constexpr (sizeof(T) == 2) {
        VecIO<__nv_bfloat16, 8>::unpack(*reinterpret_cast<const uint4*>(krow + c * 16), kv);
      } else {
        const float4 f = *reinterpret_cast<const float4*>(krow + c * 16);
        kv[0] = f.x; kv[1] = f.y; kv[2] = f.z; kv[3] = f.w;
      }
#pragma unroll
      for (int e = 0; e < EPC; ++e) dot = fmaf(kv[e], qg[c * EPC + e], dot);
    }
    const float logit = valid ? dot * sk[st * TOK + lane] * sm_scale : -INFINITY;
    if (probs && valid)
      probs[(b * Hq + (int64_t)kvh * G + warp) * p_blocks * g.t + tok] = logit;
    float mx = logit;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
    const float m_new = fmaxf(m_run, mx);
    const float alpha = m_new == -INFINITY ? 1.f : __expf(m_run - m_new);
    const float pr = valid ? __expf(logit - m_new) : 0.f;
    float ps = pr;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, s);
    l_run = l_run * alpha + ps;
    m_run = m_new;
    // ---- PV: lane = DPL output dims ----
    const float pv = pr * sv[st * TOK + lane];
#pragma unroll
    for (int k = 0; k < DPL; ++k) o[k] *= alpha;
#pragma unroll 8
    for (int tk = 0; tk < TOK; ++tk) {
      const float w = __shfl_sync(0xffffffffu, pv, tk);
      const uint8_t* vrow = vt + (st * TOK + tk) * ROW + lane * DPL * (int)sizeof(T);
      float vv[DPL];
      if constexpr (sizeof(T) == 2) {
        if constexpr (DPL == 4) {
          const uint2 u = *reinterpret_cast<const uint2*>(vrow);
          const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
          const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
          vv[0] = f0.x; vv[1] = f0.y; vv[2] = f1.x; vv[3] = f1.y;
        } else {
          const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vrow));
          vv[0] = f0.x; vv[1] = f0.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < DPL; ++k) vv[k] = reinterpret_cast<const float*>(vrow)[k];
      }
#pragma unroll
      for (int k = 0; k < DPL; ++k) o[k] = fmaf(w, vv[k], o[k]);
    }
    __syncthreads();
  }
  cp_wait<0>();
  float* pp = part + (((b * Hq + (int64_t)kvh * G + warp) * nsplit) + split) * (D + 2);
#pragma unroll
  for (int k = 0; k < DPL; ++k) pp[lane * DPL + k] = o[k];
  if (lane == 0) {
    pp[D] = m_run;
    pp[D + 1] = l_run;
  }
}

template <typename T, int D>
static cudaError_t decode_fast_t(const DecodeArgs& a, cudaStream_t s) {
  const int G = a.Hq / a.g.h;
  const int64_t nsplit = nsplit_of(a.p_blocks);
  const int smem = 2 * STG * TOK * (D * (int)sizeof(T) + 16) + 8 * D * 4 + 2 * STG * TOK * 4;
  static bool attr_set = false;  // one per <T, D> instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(decode_fast_kernel<T, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((unsigned)nsplit, a.g.h, (unsigned)a.B);
  decode_fast_kernel<T, D><<<grid, 32 * G, smem, s>>>(
      a.q, a.q_dtype, (const T*)a.pool_k, (const T*)a.pool_v, a.g, a.layer, a.table,
      (const float*)a.k_scale, (const float*)a.v_scale, a.p_blocks, a.seq_blocks, a.Hq,
      (float)a.sm_scale, (float*)a.ws, (float*)a.probs);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  decode_combine_kernel<float><<<(unsigned)(a.B * a.Hq), 128, 0, s>>>(
      (const float*)a.ws, nsplit, a.g.d, a.p_blocks, a.g.t, a.seq_blocks, a.Hq, (float*)a.out,
      (float*)a.lse, (float*)a.probs, CB);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Tensor-core path (bf16 pools, d in {64, 128}, G <= 8): flash-decoding with
// mma.sync m16n8k16 (bf16 in, fp32 accumulate). CTA = (split of CB blocks,
// kv head, request), 8 warps x one 32-token tile each. Per warp:
//   S^T = Q (G rows padded to 16) x K^T  -- K fragments via ldmatrix
//   online softmax per query head across the 4 lanes of a row group
//   O  += (P * v_scale) x V             -- P reused from the S accumulators,
//                                          V fragments via ldmatrix.trans
// Per-slot k_scale multiplies the logits, v_scale folds into P, so shared
// fused blocks are read as stored. The 8 warp partials are merged in smem
// into the same (o, m, l) split partial the combine kernel consumes.
// ---------------------------------------------------------------------------
namespace {
constexpr int MMA_WARPS = 4;  // 71 KB smem per CTA -> 3 CTAs / SM
constexpr int MMA_TT = 32;  // tokens per warp tile

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D = A(16x16, rows >= 8 zero) x B(16x8) + D ; a1 / a3 (rows 8..15) are zero
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
}  // namespace

template <int D, int TILES>
__global__ void __launch_bounds__(MMA_WARPS * 32)
decode_mma_kernel(const void* __restrict__ q, int q_dtype, const __nv_bfloat16* __restrict__ pool_k,
                  const __nv_bfloat16* __restrict__ pool_v, Geom g, int64_t layer,
                  const int32_t* __restrict__ table, const float* __restrict__ k_scale,
                  const float* __restrict__ v_scale, int64_t p_blocks,
                  const int32_t* __restrict__ seq_blocks, int Hq, float sm_scale,
                  float* __restrict__ part) {
  constexpr int ROWB = D * 2 + 16;  // padded row bytes (conflict-free ldmatrix)
  constexpr int CPR = D * 2 / 16;   // 16-byte chunks per row
  constexpr int KS = D / 16;        // k-steps over the head dim
  constexpr int NE = D / 8;         // n-tiles over the head dim (PV)
  constexpr int SBYTES = 2 * MMA_TT * ROWB + 2 * MMA_TT * 4;  // one stage
  extern __shared__ __align__(16) uint8_t dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, tig = lane & 3;
  uint8_t* wsm = dsm + warp * 2 * SBYTES;  // this warp's 2 stages

  const int G = Hq / g.h;
  const int64_t b = blockIdx.z;
  const int kvh = blockIdx.y;
  const int64_t split = blockIdx.x, nsplit = gridDim.x;
  const int64_t unit = g.head_mode ? layer * g.h + kvh : layer;
  const int32_t* tab = table + unit * g.NB;
  const float* ksc = k_scale + unit * g.NB;
  const float* vsc = v_scale + unit * g.NB;
  const int64_t nblk = seq_blocks ? (int64_t)seq_blocks[b] : p_blocks;
  const int64_t span = (int64_t)MMA_WARPS * MMA_TT * TILES;  // tokens per split
  const int64_t T1 = min((split + 1) * span, nblk * g.t);
  const int64_t E = g.E();
  const int64_t rstride = (int64_t)g.h * D;
  // warp w owns tiles w, w + MMA_WARPS, ... of the split
  auto tile_start = [&](int i) { return split * span + (int64_t)(i * MMA_WARPS + warp) * MMA_TT; };

  auto issue = [&](int i) {
    uint8_t* st = wsm + (i & 1) * SBYTES;
    uint8_t* ksm = st;
    uint8_t* vsm = st + MMA_TT * ROWB;
    float* sks = reinterpret_cast<float*>(st + 2 * MMA_TT * ROWB);
    float* svs = sks + MMA_TT;
    const int64_t t0 = tile_start(i);  // multiple of t: the tile spans MMA_TT / t whole blocks
    // one lane per block of the tile resolves table + scales (no dependent
    // global loads inside the copy loop)
    int64_t phys_l = 0;
    float ks_l = 0.f, vs_l = 0.f;
    const int nbt = MMA_TT / g.t;
    if (lane < nbt) {
      const int64_t blk = t0 / g.t + lane;
      if (blk * g.t < T1) {
        const int64_t slot = b * p_blocks + blk;
        phys_l = tab[slot];
        ks_l = ksc[slot] * sm_scale;
        vs_l = vsc[slot];
      }
    }
    for (int c = lane; c < MMA_TT * CPR; c += 32) {
      const int row = c / CPR, col = c % CPR;
      const int bl = row / g.t;
      const int64_t phys = __shfl_sync(0xffffffffu, phys_l, bl);
      const bool valid = t0 + row < T1;
      const int64_t off = (layer * g.NB + phys) * E + (row % g.t) * rstride + (int64_t)kvh * D;
      cp_async16(ksm + row * ROWB + col * 16,
                 reinterpret_cast<const uint8_t*>(pool_k + off) + col * 16, valid);
      cp_async16(vsm + row * ROWB + col * 16,
                 reinterpret_cast<const uint8_t*>(pool_v + off) + col * 16, valid);
    }
    {
      const bool valid = t0 + lane < T1;
      const float kk = __shfl_sync(0xffffffffu, ks_l, lane / g.t);
      const float vv = __shfl_sync(0xffffffffu, vs_l, lane / g.t);
      sks[lane] = valid ? kk : 0.f;
      svs[lane] = valid ? vv : 0.f;
    }
    cp_commit();
  };

  issue(0);
  // ---- Q fragments (rows = query heads of the group, zero beyond G) ----
  uint32_t qa[KS][2];
  {
    const bool real = grp < G;
    const int64_t qrow = (b * Hq + (int64_t)kvh * G + (real ? grp : 0)) * D;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int e0 = ks * 16 + 2 * tig;
      float x0 = 0.f, x1 = 0.f, x8 = 0.f, x9 = 0.f;
      if (real) {
        if (q_dtype == BF16) {
          const __nv_bfloat16* qp = (const __nv_bfloat16*)q + qrow;
          x0 = __bfloat162float(qp[e0]);
          x1 = __bfloat162float(qp[e0 + 1]);
          x8 = __bfloat162float(qp[e0 + 8]);
          x9 = __bfloat162float(qp[e0 + 9]);
        } else {
          const float* qp = (const float*)q + qrow;
          x0 = qp[e0];
          x1 = qp[e0 + 1];
          x8 = qp[e0 + 8];
          x9 = qp[e0 + 9];
        }
      }
      qa[ks][0] = pack_bf16(x0, x1);
      qa[ks][1] = pack_bf16(x8, x9);
    }
  }

  float m_run = -INFINITY, l_run = 0.f;
  float o[NE][4];
#pragma unroll
  for (int et = 0; et < NE; ++et)
#pragma unroll
    for (int k = 0; k < 4; ++k) o[et][k] = 0.f;
  const int lr = lane & 7, lm = lane >> 3;  // ldmatrix row / matrix index

  for (int i = 0; i < TILES; ++i) {
    if (i + 1 < TILES) {
      issue(i + 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncwarp();
    const uint8_t* st = wsm + (i & 1) * SBYTES;
    const uint32_t kbase = static_cast<uint32_t>(__cvta_generic_to_shared(st));
    const uint32_t vbase = kbase + MMA_TT * ROWB;
    const float* sks = reinterpret_cast<const float*>(st + 2 * MMA_TT * ROWB);
    const float* svs = sks + MMA_TT;
    const int64_t t0 = tile_start(i);
    // ---- S = Q K^T over 4 n-tiles of 8 tokens ----
    float s[4][4];
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int k = 0; k < 4; ++k) s[n][k] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
      for (int n = 0; n < 4; n += 2) {
        // matrices: (tok n*8, e), (tok n*8, e + 8), (tok n*8 + 8, e), (tok n*8 + 8, e + 8)
        const int tok = n * 8 + (lm >> 1) * 8 + lr;
        const int e = ks * 16 + (lm & 1) * 8;
        uint32_t r0, r1, r2, r3;
        ldsm_x4(kbase + tok * ROWB + e * 2, r0, r1, r2, r3);
        mma16816(s[n], qa[ks][0], qa[ks][1], r0, r1);
        mma16816(s[n + 1], qa[ks][0], qa[ks][1], r2, r3);
      }
    }
    // ---- online softmax (row = query head grp; 8 tokens per lane) ----
    float mx = -INFINITY;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int tl = n * 8 + 2 * tig + k;
        const float lg = (t0 + tl < T1) ? s[n][k] * sks[tl] : -INFINITY;
        s[n][k] = lg;
        mx = fmaxf(mx, lg);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    const float alpha = m_new == -INFINITY ? 1.f : __expf(m_run - m_new);
    float lsum = 0.f;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float p = m_new == -INFINITY ? 0.f : __expf(s[n][k] - m_new);
        s[n][k] = p;
        lsum += p;
      }
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    l_run = l_run * alpha + lsum;
    m_run = m_new;
#pragma unroll
    for (int et = 0; et < NE; ++et) {
      o[et][0] *= alpha;
      o[et][1] *= alpha;
    }
    // ---- O += (P * v_scale) V ----
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int tt = kk * 16 + 2 * tig;
      const uint32_t a0 = pack_bf16(s[2 * kk][0] * svs[tt], s[2 * kk][1] * svs[tt + 1]);
      const uint32_t a2 = pack_bf16(s[2 * kk + 1][0] * svs[tt + 8], s[2 * kk + 1][1] * svs[tt + 9]);
#pragma unroll
      for (int et = 0; et < NE; et += 2) {
        // matrices: (tok kk*16, e et*8), (tok + 8, e), (tok, e + 8), (tok + 8, e + 8)
        const int tok = kk * 16 + (lm & 1) * 8 + lr;
        const int e = et * 8 + (lm >> 1) * 8;
        uint32_t r0, r1, r2, r3;
        ldsm_x4_t(vbase + tok * ROWB + e * 2, r0, r1, r2, r3);
        mma16816(o[et], a0, a2, r0, r1);
        mma16816(o[et + 1], a0, a2, r2, r3);
      }
    }
    __syncwarp();  // stage (i & 1) is refilled by issue(i + 2)
  }
  // ---- merge the warp partials of this split ----
  __syncthreads();  // stage smem reused below
  float* wm = reinterpret_cast<float*>(dsm);  // [warps][8]
  float* wl = wm + MMA_WARPS * 8;              // [warps][8]
  float* wo = wl + MMA_WARPS * 8;              // [warps][8][D]
  if (grp < G) {
    if (tig == 0) {
      wm[warp * 8 + grp] = m_run;
      wl[warp * 8 + grp] = l_run;
    }
#pragma unroll
    for (int et = 0; et < NE; ++et) {
      wo[(warp * 8 + grp) * D + et * 8 + 2 * tig] = o[et][0];
      wo[(warp * 8 + grp) * D + et * 8 + 2 * tig + 1] = o[et][1];
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < G * D; x += MMA_WARPS * 32) {
    const int gg = x / D, e = x % D;
    float M = -INFINITY;
    for (int w = 0; w < MMA_WARPS; ++w) M = fmaxf(M, wm[w * 8 + gg]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < MMA_WARPS; ++w) {
      const float f = wm[w * 8 + gg] == -INFINITY ? 0.f : __expf(wm[w * 8 + gg] - M);
      L += wl[w * 8 + gg] * f;
      O += wo[(w * 8 + gg) * D + e] * f;
    }
    float* pp = part + (((b * Hq + (int64_t)kvh * G + gg) * nsplit) + split) * (D + 2);
    pp[e] = O;
    if (e == 0) {
      pp[D] = M;
      pp[D + 1] = L;
    }
  }
}

template <int D, int TILES>
static cudaError_t decode_mma_t(const DecodeArgs& a, cudaStream_t s) {
  constexpr int SBYTES = 2 * MMA_TT * (D * 2 + 16) + 2 * MMA_TT * 4;
  constexpr int SMEM = MMA_WARPS * 2 * SBYTES;
  static_assert(SMEM >= (2 * MMA_WARPS * 8 + MMA_WARPS * 8 * D) * 4, "combine area");
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(decode_mma_kernel<D, TILES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int cbs = MMA_WARPS * MMA_TT * TILES / a.g.t;  // blocks per split
  const int64_t nsplit = nsplit_of(a.p_blocks, cbs);
  dim3 grid((unsigned)nsplit, a.g.h, (unsigned)a.B);
  decode_mma_kernel<D, TILES><<<grid, MMA_WARPS * 32, SMEM, s>>>(
      a.q, a.q_dtype, (const __nv_bfloat16*)a.pool_k, (const __nv_bfloat16*)a.pool_v, a.g,
      a.layer, a.table, (const float*)a.k_scale, (const float*)a.v_scale, a.p_blocks,
      a.seq_blocks, a.Hq, (float)a.sm_scale, (float*)a.ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  decode_combine_kernel<float><<<(unsigned)(a.B * a.Hq), 128, 0, s>>>(
      (const float*)a.ws, nsplit, a.g.d, a.p_blocks, a.g.t, a.seq_blocks, a.Hq, (float*)a.out,
      (float*)a.lse, nullptr, cbs);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t decode_t(const DecodeArgs& a, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  // the warps' 32-token tiles must cover whole blocks of a split
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    const bool qok = a.q_dtype == BF16 || a.q_dtype == F32;
    // 32-token tiles per warp (double-buffered); KVF_DECODE_TILES overrides
    static const int tiles = [] {
      const char* e = getenv("KVF_DECODE_TILES");
      const int v = e ? atoi(e) : 2;
      return (v == 1 || v == 2 || v == 4) ? v : 2;
    }();
    const int span = MMA_WARPS * MMA_TT * tiles;
    if (qok && a.probs == nullptr && MMA_TT % a.g.t == 0 && span / a.g.t >= CB_MIN &&
        a.Hq / a.g.h <= 8) {
      if (a.g.d == 128) {
        if (tiles == 1) return decode_mma_t<128, 1>(a, s);
        if (tiles == 2) return decode_mma_t<128, 2>(a, s);
        return decode_mma_t<128, 4>(a, s);
      }
      if (a.g.d == 64) {
        if (tiles == 1) return decode_mma_t<64, 1>(a, s);
        if (tiles == 2) return decode_mma_t<64, 2>(a, s);
        return decode_mma_t<64, 4>(a, s);
      }
    }
  }
  if constexpr (!std::is_same<T, double>::value) {
    const bool qok = a.q_dtype == BF16 || a.q_dtype == F32;
    if (qok && (a.g.d == 128 || a.g.d == 64)) {
      if (a.g.d == 128) return decode_fast_t<T, 128>(a, s);
      return decode_fast_t<T, 64>(a, s);
    }
  }
  const int64_t nsplit = nsplit_of(a.p_blocks);
  dim3 grid((unsigned)nsplit, a.g.h, (unsigned)a.B);
  decode_partial_kernel<T><<<grid, NTD, 0, s>>>(
      a.q, a.q_dtype, (const T*)a.pool_k, (const T*)a.pool_v, a.g, a.layer, a.table,
      (const A*)a.k_scale, (const A*)a.v_scale, a.p_blocks, a.seq_blocks, a.Hq, (A)a.sm_scale,
      (A*)a.ws, (A*)a.probs);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  decode_combine_kernel<A><<<(unsigned)(a.B * a.Hq), 128, 0, s>>>(
      (const A*)a.ws, nsplit, a.g.d, a.p_blocks, a.g.t, a.seq_blocks, a.Hq, (A*)a.out,
      (A*)a.lse, (A*)a.probs, CB);
  return cudaGetLastError();
}

cudaError_t launch_paged_decode(const DecodeArgs& a, cudaStream_t s) {
  if (a.g.d > MAXD || a.g.t > MAXT || a.Hq % a.g.h != 0 || a.Hq / a.g.h > MAXG)
    return cudaErrorInvalidValue;
  if (a.ws_bytes < decode_workspace_size(a.dtype, a.B, a.Hq, a.g.d, a.p_blocks, a.g.t))
    return cudaErrorInvalidValue;
  if (a.B == 0) return cudaSuccess;
  switch (a.dtype) {
    case F64: return decode_t<double>(a, s);
    case F32: return decode_t<float>(a, s);
    default: return decode_t<__nv_bfloat16>(a, s);
  }
}

}  // namespace kvf
