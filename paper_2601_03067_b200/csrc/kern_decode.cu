// K6: paged decode attention over the fused cache.
// Generalises the reference's exact single-query attention
// (attention.py:58-80 over refold, core.py:285-305) to a batch of requests,
// all query heads with GQA, and reads K/V straight from the fused pool:
//   K_slot = k_scale[slot] * pool_k[table[slot]]   (same for V)
// so shared physical blocks are never materialised per slot.
// Split-K (flash-decoding): CTA = (request, kv head, split of CB blocks),
// online softmax per query head of the GQA group, then a combine kernel.
#include "kernels.h"
#include "vec_io.cuh"

namespace kvf {

namespace {
constexpr int CB = 16;       // blocks per split
constexpr int NTD = 128;     // threads per CTA
constexpr int MAXG = 8;      // max query heads per kv head
constexpr int MAXD = 128;    // max head dim
constexpr int MAXT = 32;     // max tokens per block

int64_t nsplit_of(int64_t p_blocks) { return (p_blocks + CB - 1) / CB; }

template <typename A>
__device__ __forceinline__ A load_q(const void* q, int q_dtype, int64_t idx) {
  if (q_dtype == F64) return (A)((const double*)q)[idx];
  if (q_dtype == F32) return (A)((const float*)q)[idx];
  return (A)__bfloat162float(((const __nv_bfloat16*)q)[idx]);
}
}  // namespace

int64_t decode_workspace_size(int dtype, int64_t B, int Hq, int d, int64_t p_blocks, int t) {
  const int64_t acc = dtype == F64 ? 8 : 4;
  return B * Hq * nsplit_of(p_blocks) * (int64_t)(d + 2) * acc;
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
                                      A* __restrict__ probs) {
  const int64_t bh = blockIdx.x;  // b * Hq + qh
  const A* pp = part + bh * nsplit * (d + 2);
  const int64_t b = bh / Hq;
  const int64_t nblk = seq_blocks ? (int64_t)seq_blocks[b] : p_blocks;
  const int64_t nused = (nblk + CB - 1) / CB;
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

template <typename T>
static cudaError_t decode_t(const DecodeArgs& a, cudaStream_t s) {
  using A = typename AccOf<T>::type;
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
      (A*)a.lse, (A*)a.probs);
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
