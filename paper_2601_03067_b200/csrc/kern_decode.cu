// K6: paged decode attention over the fused cache.
// Generalises the reference's exact single-query attention
// (attention.py:58-80 over refold, core.py:285-305) to a batch of requests,
// all query heads with GQA, and reads K/V straight from the fused pool:
//   K_slot = k_scale[slot] * pool_k[table[slot]]   (same for V)
// so shared physical blocks are never materialised per slot.
// Split-K (flash-decoding): CTA = (request, kv head, split of CB blocks),
// online softmax per query head of the GQA group, then a combine kernel.
#include "kernels.h"
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

// Split combine without probabilities: one warp per (request, query head). Lane s
// holds split s's (m, l) (32 splits per pass), the split weights exp(m_s - M) are
// computed once and broadcast, and each lane accumulates 4 output elements from
// coalesced 128-B rows of the partials (the CTA-per-head kernel above re-reads
// every (m, l) in every thread and recomputes the weights per element).
template <int D>
__global__ void __launch_bounds__(256)
decode_combine_warp_kernel(const float* __restrict__ part, int64_t nsplit, int64_t p_blocks,
                           const int32_t* __restrict__ seq_blocks, int Hq, int64_t n_bh,
                           float* __restrict__ out, float* __restrict__ lse, int cbs) {
  constexpr int EPL = D / 32;  // output elements per lane
  const int lane = threadIdx.x & 31;
  const int64_t bh = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (bh >= n_bh) return;
  const float* pp = part + bh * nsplit * (D + 2);
  const int64_t b = bh / Hq;
  const int64_t nblk = seq_blocks ? (int64_t)seq_blocks[b] : p_blocks;
  const int64_t nused = (nblk + cbs - 1) / cbs;
  float M = -INFINITY;
  for (int64_t s0 = 0; s0 < nused; s0 += 32)
    if (s0 + lane < nused) M = fmaxf(M, pp[(s0 + lane) * (D + 2) + D]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float L = 0.f, acc[EPL];
#pragma unroll
  for (int k = 0; k < EPL; ++k) acc[k] = 0.f;
  for (int64_t s0 = 0; s0 < nused; s0 += 32) {
    float w = 0.f;
    if (s0 + lane < nused) {
      const float* ps = pp + (s0 + lane) * (D + 2);
      const float m = ps[D];
      w = m == -INFINITY ? 0.f : expf(m - M);
      L += ps[D + 1] * w;
    }
    const int ns = nused - s0 < 32 ? (int)(nused - s0) : 32;
#pragma unroll 4
    for (int j = 0; j < ns; ++j) {
      const float wj = __shfl_sync(0xffffffffu, w, j);
      const float* ps = pp + (s0 + j) * (D + 2);
#pragma unroll
      for (int k = 0; k < EPL; ++k) acc[k] = fmaf(ps[k * 32 + lane], wj, acc[k]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  const float inv = 1.f / L;
#pragma unroll
  for (int k = 0; k < EPL; ++k) out[bh * D + k * 32 + lane] = acc[k] * inv;
  if (lane == 0) lse[bh] = M + logf(L);
}

cudaError_t launch_decode_combine(const DecodeArgs& a, int64_t nsplit, int cbs, cudaStream_t s) {
  const int64_t n_bh = a.B * a.Hq;
  if (a.g.d == 128 || a.g.d == 64) {
    const unsigned grid = (unsigned)((n_bh * 32 + 255) / 256);
    if (a.g.d == 128)
      decode_combine_warp_kernel<128><<<grid, 256, 0, s>>>((const float*)a.ws, nsplit, a.p_blocks,
                                                           a.seq_blocks, a.Hq, n_bh, (float*)a.out,
                                                           (float*)a.lse, cbs);
    else
      decode_combine_warp_kernel<64><<<grid, 256, 0, s>>>((const float*)a.ws, nsplit, a.p_blocks,
                                                          a.seq_blocks, a.Hq, n_bh, (float*)a.out,
                                                          (float*)a.lse, cbs);
    return cudaGetLastError();
  }
  decode_combine_kernel<float><<<(unsigned)n_bh, 128, 0, s>>>(
      (const float*)a.ws, nsplit, a.g.d, a.p_blocks, a.g.t, a.seq_blocks, a.Hq, (float*)a.out,
      (float*)a.lse, nullptr, cbs);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t decode_t(const DecodeArgs& a, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  // bf16: TMA + mma.sync path; f32 (and bf16 shapes TMA cannot take): CUDA-core
  // cp.async path; f64 / probability output: the generic kernel
  if (decode_tma_supported(a)) return launch_decode_tma(a, s);
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
  if (a.sched != nullptr) return a.B == 0 ? cudaSuccess : launch_decode_sched(a, s);
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
