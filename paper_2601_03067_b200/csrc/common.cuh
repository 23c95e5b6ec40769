// Shared device helpers for the kvfuse B200 kernels (sm_100a).
//
// Data model:
//   pool  : (L, NB, t, h, d) contiguous, NB = B*p physical blocks per layer
//           (the reference's (L, B, p, t, h, d) cache, core.py:1-9).
//   unit  : one independent fusion problem -- a layer ("folded" mode, the
//           reference's semantics, block vector = all (t, h, d) entries in
//           C-order, core.py:128) or a (layer, kv-head) pair ("per_head").
//   vector: block i of unit u, r = t*h*d (folded) or t*d (per_head) entries,
//           stored as nseg segments of `seg` contiguous elements that are
//           `seg_stride` apart.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace kvf {

constexpr int32_t kNone = 0x7fffffff;  // "not absorbed" sentinel for absorber[]

enum DType : int { F64 = 0, F32 = 1, BF16 = 2 };

template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<double> { using type = double; };

__device__ __forceinline__ float to_acc(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_acc(float x) { return x; }
__device__ __forceinline__ double to_acc(double x) { return x; }

template <typename T, typename A> __device__ __forceinline__ T from_acc(A x);
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16, float>(float x) {
  return __float2bfloat16_rn(x);
}
template <> __device__ __forceinline__ float from_acc<float, float>(float x) { return x; }
template <> __device__ __forceinline__ double from_acc<double, double>(double x) { return x; }

// Geometry of the pool and of a fusion unit.
struct Geom {
  int64_t L, NB;      // layers, physical blocks per layer
  int32_t t, h, d;    // tokens per block, kv heads, head dim
  int32_t head_mode;  // 0 = folded (unit = layer), 1 = per_head (unit = layer*h + head)
  __host__ __device__ int64_t E() const { return (int64_t)t * h * d; }
  __host__ __device__ int64_t r() const { return head_mode ? (int64_t)t * d : E(); }
  __host__ __device__ int32_t seg() const { return head_mode ? d : (int32_t)E(); }
  __host__ __device__ int64_t seg_stride() const { return head_mode ? (int64_t)h * d : E(); }
  __host__ __device__ int64_t units() const { return head_mode ? L * h : L; }
  // element offset of vector (u, i), element 0
  __host__ __device__ int64_t base(int64_t u, int64_t i) const {
    int64_t layer = head_mode ? u / h : u;
    int64_t head = head_mode ? u % h : 0;
    return (layer * NB + i) * E() + head * d;
  }
  // offset of element k inside a vector
  __host__ __device__ int64_t off(int64_t k) const {
    if (!head_mode) return k;
    return (k / d) * ((int64_t)h * d) + (k % d);
  }
  // the same in 32-bit arithmetic (k < r <= INT32_MAX)
  __host__ __device__ int32_t off32(int32_t k) const {
    if (!head_mode) return k;
    return (k / d) * (h * d) + (k % d);
  }
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block-wide sum (fixed reduction tree). `red` needs 32 slots.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = 0;
  if (warp == 0) {
    r = lane < nw ? red[lane] : T(0);
    r = warp_sum(r);
    if (lane == 0) red[0] = r;
  }
  __syncthreads();
  r = red[0];
  __syncthreads();
  return r;
}

}  // namespace kvf
