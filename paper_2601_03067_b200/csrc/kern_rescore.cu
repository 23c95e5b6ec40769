// Exact re-score of near-threshold pairs deferred by the tcgen05 similarity
// epilogue. The tensor-core fp32 accumulator can be off by ~1e-4 relative after
// r/16 accumulation steps, which would flip strict '> thr' decisions
// (fusion.py:256) that the float64 reference takes the other way. Each queued
// pair (u, i, j) is recomputed here in float64 from the stored blocks --
// cos = <x_i, x_j> / sqrt(<x_i, x_i> <x_j, x_j>) -- and, if it exceeds thr,
// applied with the same order-independent atomicMin as the main epilogue.
#include "kernels.h"
#include "vec_io.cuh"

namespace kvf {

template <typename T, int VEC>
__global__ void rescore_kernel(const T* __restrict__ pool, Geom g, int64_t u0,
                               const int4* __restrict__ list, const int32_t* __restrict__ count,
                               int64_t cap, double thr, int32_t* absorber,
                               const int32_t* __restrict__ merges, double* samples,
                               const int64_t* __restrict__ sample_off, int64_t sample_stride) {
  using A = typename AccOf<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n = min((int64_t)*count, cap);
  const int64_t nch = g.r() / VEC;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < n; w += nw) {
    const int4 e = list[w];
    const int64_t u = e.x;
    const T* x = pool + g.base(u, e.y);
    const T* y = pool + g.base(u, e.z);
    double dxy = 0.0, dxx = 0.0, dyy = 0.0;
    for (int64_t c = lane; c < nch; c += 32) {
      A a[VEC], b[VEC];
      VecIO<T, VEC>::load_nc(x + g.off(c * VEC), a);
      VecIO<T, VEC>::load_nc(y + g.off(c * VEC), b);
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
      const double s = (dxx > 0.0 && dyy > 0.0) ? dxy / sqrt(dxx * dyy) : 0.0;
      if (s > thr) atomicMin(&absorber[u * g.NB + e.z], e.y);
      if (samples) {
        const int lb = merges[3 * e.w], mid = merges[3 * e.w + 1], re = merges[3 * e.w + 2];
        samples[(u - u0) * sample_stride + sample_off[e.w] + (int64_t)(e.y - lb) * (re - mid) +
                (e.z - mid)] = s;
      }
    }
  }
}

template <typename T>
static cudaError_t rescore_t(const RescoreArgs& a, cudaStream_t s) {
  const int grid = 148 * 4;
  if (can_vectorize<T>(a.pool, a.g))
    rescore_kernel<T, Vec16<T>::N><<<grid, 256, 0, s>>>(
        (const T*)a.pool, a.g, a.u0, (const int4*)a.resc, a.resc_count, a.resc_cap, a.thr,
        a.absorber, a.merges, a.samples, a.sample_off, a.sample_stride);
  else
    rescore_kernel<T, 1><<<grid, 256, 0, s>>>(
        (const T*)a.pool, a.g, a.u0, (const int4*)a.resc, a.resc_count, a.resc_cap, a.thr,
        a.absorber, a.merges, a.samples, a.sample_off, a.sample_stride);
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
