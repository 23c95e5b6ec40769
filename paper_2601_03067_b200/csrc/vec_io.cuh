// 128-bit vectorised loads/stores of pool elements, widened to the
// accumulation type (fp32 for bf16/f32 pools, fp64 for f64 pools).
#pragma once
#include "common.cuh"

namespace kvf {

template <typename T> struct Vec16 { static constexpr int N = 16 / sizeof(T); };

template <typename T, int VEC> struct VecIO;

template <typename T> struct VecIO<T, 1> {
  using A = typename AccOf<T>::type;
  __device__ __forceinline__ static void load(const T* p, A* o) { o[0] = to_acc(p[0]); }
  __device__ __forceinline__ static void load_nc(const T* p, A* o) { o[0] = to_acc(__ldg(p)); }
  __device__ __forceinline__ static void store(T* p, const A* v, A* rounded) {
    T x = from_acc<T, A>(v[0]);
    p[0] = x;
    rounded[0] = to_acc(x);
  }
};

template <> struct VecIO<__nv_bfloat16, 8> {
  __device__ __forceinline__ static void unpack(uint4 u, float* o) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
  }
  __device__ __forceinline__ static void load(const __nv_bfloat16* p, float* o) {
    unpack(*reinterpret_cast<const uint4*>(p), o);
  }
  __device__ __forceinline__ static void load_nc(const __nv_bfloat16* p, float* o) {
    unpack(__ldg(reinterpret_cast<const uint4*>(p)), o);
  }
  __device__ __forceinline__ static void store(__nv_bfloat16* p, const float* v, float* rounded) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      float2 f = __bfloat1622float2(h[i]);
      rounded[2 * i] = f.x;
      rounded[2 * i + 1] = f.y;
    }
    *reinterpret_cast<uint4*>(p) = u;
  }
};

template <> struct VecIO<float, 4> {
  __device__ __forceinline__ static void load(const float* p, float* o) {
    float4 f = *reinterpret_cast<const float4*>(p);
    o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = f.w;
  }
  __device__ __forceinline__ static void load_nc(const float* p, float* o) {
    float4 f = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = f.w;
  }
  __device__ __forceinline__ static void store(float* p, const float* v, float* rounded) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
#pragma unroll
    for (int i = 0; i < 4; ++i) rounded[i] = v[i];
  }
};

template <> struct VecIO<double, 2> {
  __device__ __forceinline__ static void load(const double* p, double* o) {
    double2 f = *reinterpret_cast<const double2*>(p);
    o[0] = f.x; o[1] = f.y;
  }
  __device__ __forceinline__ static void load_nc(const double* p, double* o) {
    double2 f = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = f.x; o[1] = f.y;
  }
  __device__ __forceinline__ static void store(double* p, const double* v, double* rounded) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    rounded[0] = v[0];
    rounded[1] = v[1];
  }
};

// Vectorised access is legal when every VEC-chunk of a vector is contiguous
// and 16-byte aligned: d % VEC == 0 (then t*h*d and head offsets are too).
template <typename T>
inline bool can_vectorize(const void* pool, const Geom& g) {
  const int V = Vec16<T>::N;
  return (g.d % V == 0) && ((reinterpret_cast<uintptr_t>(pool) & 15) == 0);
}

}  // namespace kvf
