// Exact re-score of near-threshold pairs deferred by the tcgen05 similarity
// epilogue. The tensor-core fp32 accumulator can be off by ~1e-4 relative after
// r/16 accumulation steps, which would flip strict '> thr' decisions
// (fusion.py:256) that the float64 reference takes the other way. Each queued
// pair (u, i, j) is recomputed here in float64 from the stored blocks --
// cos = <x_i, x_j> / sqrt(<x_i, x_i> <x_j, x_j>) -- and, if it exceeds thr,
// applied with the same order-independent atomicMin as the main epilogue.
// Exact mode (kern_exact.cu): a block with a shadow slot is read from its
// float64-derived fp32 unit direction instead of the rounded pool block.
#include "kernels.h"
#include "vec_io.cuh"

namespace kvf {

// One CTA per queued pair (the queue is short -- tens to hundreds of pairs per
// level -- so per-pair latency, not throughput, bounds the launch): 256
// threads split the r-element dot products, float64 accumulation (bf16 and
// fp32 products are exact in float64), fixed-order block reduction.
template <typename T, int VEC>
__global__ void __launch_bounds__(256)
rescore_kernel(const T* __restrict__ pool, Geom g, int64_t u0,
               const int4* __restrict__ list, const int32_t* __restrict__ count,
               int64_t cap, double thr, int32_t* absorber,
               const int32_t* __restrict__ merges, double* samples,
               const int64_t* __restrict__ sample_off, int64_t sample_stride,
               const float* __restrict__ shadow, const int32_t* __restrict__ sidx) {
  using A = typename AccOf<T>::type;
  __shared__ double red[3][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = min((int64_t)*count, cap);
  const int64_t nch = g.r() / VEC;
  for (int64_t w = blockIdx.x; w < n; w += gridDim.x) {
    const int4 e = list[w];
    const int64_t u = e.x;
    const T* x = pool + g.base(u, e.y);
    const T* y = pool + g.base(u, e.z);
    const int32_t sx = sidx ? sidx[u * g.NB + e.y] : -1;
    const int32_t sy = sidx ? sidx[u * g.NB + e.z] : -1;
    const float* xs = sx >= 0 ? shadow + (int64_t)sx * g.r() : nullptr;
    const float* ys = sy >= 0 ? shadow + (int64_t)sy * g.r() : nullptr;
    double dxy = 0.0, dxx = 0.0, dyy = 0.0;
    for (int64_t c = threadIdx.x; c < nch; c += blockDim.x) {
      A a[VEC], b[VEC];
      if (xs) {
#pragma unroll
        for (int q = 0; q < VEC; ++q) a[q] = (A)xs[c * VEC + q];
      } else {
        VecIO<T, VEC>::load_nc(x + g.off(c * VEC), a);
      }
      if (ys) {
#pragma unroll
        for (int q = 0; q < VEC; ++q) b[q] = (A)ys[c * VEC + q];
      } else {
        VecIO<T, VEC>::load_nc(y + g.off(c * VEC), b);
      }
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        const double da = (double)a[q], db = (double)b[q];
        dxy = fma(da, db, dxy);
        dxx = fma(da, da, dxx);
        dyy = fma(db, db, dyy);
      }
    }
    dxy = warp_sum(dxy);
    dxx = warp_sum(dxx);
    dyy = warp_sum(dyy);
    if (lane == 0) {
      red[0][warp] = dxy;
      red[1][warp] = dxx;
      red[2][warp] = dyy;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sxy = 0.0, sxx = 0.0, syy = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
        sxy += red[0][q];
        sxx += red[1][q];
        syy += red[2][q];
      }
      const double s = (sxx > 0.0 && syy > 0.0) ? sxy / sqrt(sxx * syy) : 0.0;
      if (s > thr) atomicMin(&absorber[u * g.NB + e.z], e.y);
      if (samples) {
        const int lb = merges[3 * e.w], mid = merges[3 * e.w + 1], re = merges[3 * e.w + 2];
        samples[(u - u0) * sample_stride + sample_off[e.w] + (int64_t)(e.y - lb) * (re - mid) +
                (e.z - mid)] = s;
      }
    }
    __syncthreads();
  }
}

template <typename T>
static cudaError_t rescore_t(const RescoreArgs& a, cudaStream_t s) {
  const int grid = 148 * 8;
  if (can_vectorize<T>(a.pool, a.g))
    rescore_kernel<T, Vec16<T>::N><<<grid, 256, 0, s>>>(
        (const T*)a.pool, a.g, a.u0, (const int4*)a.resc, a.resc_count, a.resc_cap, a.thr,
        a.absorber, a.merges, a.samples, a.sample_off, a.sample_stride, a.shadow, a.sidx);
  else
    rescore_kernel<T, 1><<<grid, 256, 0, s>>>(
        (const T*)a.pool, a.g, a.u0, (const int4*)a.resc, a.resc_count, a.resc_cap, a.thr,
        a.absorber, a.merges, a.samples, a.sample_off, a.sample_stride, a.shadow, a.sidx);
  return cudaGetLastError();
}

cudaError_t launch_rescore(const RescoreArgs& a, cudaStream_t s) {
  switch (a.dtype) {
    case F64: return rescore_t<double>(a, s);
    case F32: return rescore_t<float>(a, s);
    default: return rescore_t<__nv_bfloat16>(a, s);
  }
}

}  // namespace kvf
