// Exact-decision support for reduced-precision pools (SURVEY §8c parity).
//
// The reference keeps every fused key direction in float64
// (fusion.py:259-261, _unit 285-287) and decides `sim > thr` on those
// (fusion.py:246, 256). A bf16 pool stores a fused block rounded to bf16, so
// at tree levels >= 2 the stored direction is ~2^-9 away from the reference's
// and a pair near the threshold can be decided the other way, after which
// the trees diverge. Exact mode keeps, next to the paged pool:
//   shadow[slot][r]  fp32 unit direction of every key absorber (written by
//                    exact_merge_keys_kernel, summed in float64 from the
//                    members' float64 directions -- shadow rows for fused
//                    members, x / |x|_64 of the stored bf16 block otherwise),
//   sidx[u][NB]      absorber -> shadow slot (-1: never fused, the pool block
//                    is the original one and exact in float64 after widening).
// The pool still receives s_home * dir (bf16) and its stored norm, so the
// tensor-core similarity, decode and refold read the paged layout as before;
// only pairs within the re-score band are re-decided, from the shadow rows
// (kern_rescore.cu). Values follow the key decisions and are merged by the
// normal K4 kernel (kern_merge.cu, which = V only).
//
// convert_rows: the bf16 operand copy ("filter") that lets fp32 pools use the
// tcgen05 similarity: hi = bf16(x) and lo = bf16(x - hi) (rows [0, L*NB) and
// [L*NB, 2*L*NB)); the similarity kernel accumulates hi.hi + hi.lo + lo.hi over
// three K passes (~2^-16 relative per product, fp32-grade similarities) and
// pairs within the band are still re-decided from the fp32 pool in float64.
#include <algorithm>
#include "kernels.h"
#include "vec_io.cuh"

namespace kvf {

namespace {
__device__ __forceinline__ void load8_f32(const float* p, float* o) {
  VecIO<float, 4>::load(p, o);
  VecIO<float, 4>::load(p + 4, o + 4);
}
__device__ __forceinline__ void store8_f32(float* p, const float* v) {
  float rd[4];
  VecIO<float, 4>::store(p, v, rd);
  VecIO<float, 4>::store(p + 4, v + 4, rd);
}
}  // namespace

// CTA per key absorber of the level; thread owns chunks c = tid + q * blockDim
// (8 elements each) of the r-vector, float64 accumulators in registers.
template <int MAXQ>
__global__ void __launch_bounds__(512)
exact_merge_keys_kernel(__nv_bfloat16* __restrict__ pool, Geom g, float* __restrict__ knorm,
                        const float* __restrict__ oknorm, float* __restrict__ shadow, int64_t cap,
                        int32_t* __restrict__ sidx, int32_t* __restrict__ scount, int32_t* ws,
                        int64_t n_total) {
  __shared__ double red[32];
  __shared__ float redf[32];
  __shared__ int slot_sh;
  const LevelWs W(ws, n_total);
  const int tid = threadIdx.x, bd = blockDim.x;
  const int64_t r = g.r();
  const int64_t nch = r / 8;
  const int n_items = *W.count;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int64_t gid = W.list[it];
    const int64_t u = gid / g.NB, gb = u * g.NB;
    const int32_t l = (int32_t)(gid - gb);
    const int n = W.mcnt[gid], s0 = W.mstart[gid];
    double acc[MAXQ][8];
#pragma unroll
    for (int q = 0; q < MAXQ; ++q)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[q][e] = 0.0;
    // members in the reference's order: the absorber, then ascending right ids
    for (int v = 0; v <= n; ++v) {
      const int32_t id = v == 0 ? l : W.members[s0 + v - 1];
      const int32_t sv = sidx[gb + id];
      if (sv >= 0) {  // fused earlier: its float64-derived unit direction
        const float* row = shadow + (int64_t)sv * r;
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int64_t c = tid + (int64_t)q * bd;
          if (c < nch) {
            float x[8];
            load8_f32(row + c * 8, x);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[q][e] += (double)x[e];
          }
        }
      } else {  // original block: x / |x| in float64 (core.py:115-119); the second
                // pass re-reads the 32 KB vector from L1 instead of holding it
        const __nv_bfloat16* xb = pool + g.base(u, id);
        double ss = 0.0;
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int64_t c = tid + (int64_t)q * bd;
          if (c < nch) {
            float x[8];
            VecIO<__nv_bfloat16, 8>::load(xb + g.off(c * 8), x);
#pragma unroll
            for (int e = 0; e < 8; ++e) ss = fma((double)x[e], (double)x[e], ss);
          }
        }
        ss = block_sum(ss, red);
        const double nrm = sqrt(ss);
        const double inv = 1.0 / nrm;  // x * (1/|x|): within an ulp of the reference's x / |x|
        if (nrm > 0.0) {
#pragma unroll
          for (int q = 0; q < MAXQ; ++q) {
            const int64_t c = tid + (int64_t)q * bd;
            if (c < nch) {
              float x[8];
              VecIO<__nv_bfloat16, 8>::load(xb + g.off(c * 8), x);
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[q][e] = fma((double)x[e], inv, acc[q][e]);
            }
          }
        }
      }
    }
    double ss = 0.0;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q)
#pragma unroll
      for (int e = 0; e < 8; ++e) ss = fma(acc[q][e], acc[q][e], ss);
    const double nrm = sqrt(block_sum(ss, red));  // _unit: a zero sum stays zero
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    if (tid == 0) {
      int s = sidx[gid];
      if (s < 0) {
        s = atomicAdd(scount, 1);  // counts overflow attempts too (reported)
        if (s < cap) sidx[gid] = s; else s = -1;
      }
      slot_sh = s;
    }
    __syncthreads();
    const int slot = slot_sh;
    float* srow = slot >= 0 ? shadow + (int64_t)slot * r : nullptr;
    const float home = oknorm[gid];
    const double hs = home > 0.f ? (double)home : 1.0;
    __nv_bfloat16* xl = pool + g.base(u, l);
    float rs = 0.f;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int64_t c = tid + (int64_t)q * bd;
      if (c < nch) {
        float dir[8], y[8], rd[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double de = acc[q][e] * inv;
          dir[e] = (float)de;
          y[e] = (float)(de * hs);
        }
        if (srow) store8_f32(srow + c * 8, dir);
        VecIO<__nv_bfloat16, 8>::store(xl + g.off(c * 8), y, rd);
#pragma unroll
        for (int e = 0; e < 8; ++e) rs = fmaf(rd[e], rd[e], rs);
      }
    }
    const float nn = sqrtf(block_sum(rs, redf));
    if (tid == 0) knorm[gid] = nn;
    __syncthreads();
  }
}

cudaError_t launch_exact_merge_keys(void* pool_k, const Geom& g, float* knorm, const float* oknorm,
                                    float* shadow, int64_t cap, int32_t* sidx, int32_t* scount,
                                    int32_t* level_ws, cudaStream_t s) {
  const int64_t n_total = g.units() * g.NB;
  const int64_t nch = g.r() / 8;
  int bd = 512;
  while (bd > 64 && (int64_t)(bd / 2) * 4 >= nch) bd /= 2;
  const int grid = 148 * (bd >= 512 ? 2 : 4096 / bd);
  auto go = [&](auto kern) {
    kern<<<grid, bd, 0, s>>>((__nv_bfloat16*)pool_k, g, knorm, oknorm, shadow, cap, sidx, scount,
                             level_ws, n_total);
    return cudaGetLastError();
  };
  if (nch <= (int64_t)bd * 1) return go(exact_merge_keys_kernel<1>);
  if (nch <= (int64_t)bd * 2) return go(exact_merge_keys_kernel<2>);
  if (nch <= (int64_t)bd * 4) return go(exact_merge_keys_kernel<4>);
  return cudaErrorInvalidValue;  // r > 16384 (checked by the ABI)
}

// ---------------------------------------------------------------------------
// fp32 -> bf16 hi/lo operand copy: every vector (level_ws == null) or the key
// absorbers of the current level (after kvf_merge_groups rewrote them)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void split8(const float* src, __nv_bfloat16* hi, __nv_bfloat16* lo) {
  float x[8], rd[8], rest[8];
  load8_f32(src, x);
  VecIO<__nv_bfloat16, 8>::store(hi, x, rd);
#pragma unroll
  for (int e = 0; e < 8; ++e) rest[e] = x[e] - rd[e];  // exact in fp32
  VecIO<__nv_bfloat16, 8>::store(lo, rest, rd);
}

__global__ void convert_all_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                   int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x)
    split8(src + i * 8, dst + i * 8, dst + (n8 + i) * 8);
}

__global__ void convert_level_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                     Geom g, int32_t* ws, int64_t n_total) {
  const LevelWs W(ws, n_total);
  const int n_items = *W.count;
  const int64_t nch = g.r() / 8;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int64_t gid = W.list[it];
    const int64_t u = gid / g.NB;
    const int64_t base = g.base(u, gid - u * g.NB);
    const int64_t lo = g.L * g.NB * g.E();
    for (int64_t c = threadIdx.x; c < nch; c += blockDim.x) {
      const int64_t o = base + g.off(c * 8);
      split8(src + o, dst + o, dst + lo + o);
    }
  }
}

cudaError_t launch_convert_rows(const void* src, void* dst, const Geom& g, int32_t* level_ws,
                                cudaStream_t s) {
  if (!level_ws) {
    const int64_t n8 = g.L * g.NB * g.E() / 8;
    const int64_t blocks = (n8 + 255) / 256;
    convert_all_kernel<<<(int)std::min<int64_t>(blocks, 148 * 16), 256, 0, s>>>(
        (const float*)src, (__nv_bfloat16*)dst, n8);
  } else {
    convert_level_kernel<<<148 * 8, 256, 0, s>>>((const float*)src, (__nv_bfloat16*)dst, g,
                                                 level_ws, g.units() * g.NB);
  }
  return cudaGetLastError();
}

}  // namespace kvf
