// Bandwidth-bound kernels of the fusion pipeline (sm_100a):
//   K1  block norms            (core.py:115-119)
//   --  state init             (fusion.py:208-228, core.py:191-201)
//   --  per-merge level stats  (fusion.py:249, 273-281)
//   K4  in-place block merge   (fusion.py:259-261, 285-287)
//   K5  table remap/refcounts  (core.py:217-227, fusion.py:262-264)
//   --  finalize: per-slot scales, live/free lists (fusion.py:316-324)
//   --  audit / redirect / gather / refold (core.py:232-241, 285-305)
#include <type_traits>
#include "kernels.h"
#include "vec_io.cuh"

namespace kvf {

// --------------------------------------------------------------------------
// NaN / Inf validation (PagedKvCache.__post_init__, core.py:73-74)
// --------------------------------------------------------------------------
__device__ __forceinline__ bool finite_of(double x) { return isfinite(x); }
__device__ __forceinline__ bool finite_of(float x) { return isfinite(x); }
__device__ __forceinline__ bool finite_of(__nv_bfloat16 x) { return isfinite(__bfloat162float(x)); }

template <typename T>
__global__ void count_nonfinite_kernel(const T* __restrict__ x, int64_t n,
                                       unsigned long long* count) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += finite_of(x[i]) ? 0ull : 1ull;
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

cudaError_t launch_count_nonfinite(const void* data, int dtype, int64_t n,
                                   unsigned long long* count, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
  switch (dtype) {
    case F64: count_nonfinite_kernel<<<grid, 256, 0, s>>>((const double*)data, n, count); break;
    case F32: count_nonfinite_kernel<<<grid, 256, 0, s>>>((const float*)data, n, count); break;
    default: count_nonfinite_kernel<<<grid, 256, 0, s>>>((const __nv_bfloat16*)data, n, count);
  }
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// K1: one warp per (unit, block) vector; deterministic lane order + xor tree.
// --------------------------------------------------------------------------
template <typename T, int VEC>
__global__ void block_norms_kernel(const T* __restrict__ pool, Geom g,
                                   typename AccOf<T>::type* __restrict__ norms) {
  using A = typename AccOf<T>::type;
  const int64_t nvec = g.units() * g.NB;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nvec) return;
  const int64_t u = w / g.NB, i = w % g.NB;
  const T* base = pool + g.base(u, i);
  const int64_t nch = g.r() / VEC;
  double acc = 0;  // float64 sums: stored norms within an ulp of the reference's (core.py:116)
  for (int64_t c = lane; c < nch; c += 32) {
    A v[VEC];
    VecIO<T, VEC>::load_nc(base + g.off(c * VEC), v);
#pragma unroll
    for (int q = 0; q < VEC; ++q) acc = fma((double)v[q], (double)v[q], acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) norms[w] = (A)sqrt(acc);
}

// Per-head units, bf16, d = 128, h = 8: one warp per physical block reads the block's
// contiguous 32 KB (a per-head warp would read 16 rows of 256 B at a 2 KB stride, and
// the eight heads' passes would reopen every DRAM page 8 times). A 512-B warp step
// covers two (token, head) rows: lanes 0-15 even heads, 16-31 odd heads, so step k of
// a lane adds to head 2 (k % 4) + lane / 16 -- four accumulators with static indices.
__global__ void block_norms_heads_kernel(const __nv_bfloat16* __restrict__ pool, Geom g,
                                         float* __restrict__ norms) {
  constexpr int D = 128, H = 8, T = 16;
  const int64_t nblk = g.L * g.NB;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nblk) return;
  const uint4* base = reinterpret_cast<const uint4*>(pool + w * (int64_t)(T * H * D));
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // float64 sums of exact 8-term fp32 partials
#pragma unroll 4
  for (int k = 0; k < T * H * D / 8 / 32; ++k) {  // 64 steps of 32 x 16 B
    const uint4 q = __ldg(base + k * 32 + lane);
    const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&q);
    float a = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(p2[e]);
      a = fmaf(f.x, f.x, a);
      a = fmaf(f.y, f.y, a);
    }
    acc[k & 3] += a;
  }
  const int64_t layer = w / g.NB, blk = w % g.NB;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double v = acc[j];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // within 16 lanes
    if ((lane & 15) == 0) {
      const int head = 2 * j + (lane >> 4);
      norms[(layer * H + head) * g.NB + blk] = (float)sqrt(v);
    }
  }
}

// Folded units, bf16: warp per block over its contiguous E elements, four independent
// 16-B loads in flight per lane (the generic loop above keeps one)
__global__ void block_norms_flat_kernel(const __nv_bfloat16* __restrict__ pool, int64_t nvec,
                                        int64_t E, float* __restrict__ norms) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nvec) return;
  const uint4* base = reinterpret_cast<const uint4*>(pool + w * E);
  const int64_t nch = E / 8;
  double acc = 0.0;  // float64 sums of 8-term fp32 partials (bf16 squares are exact in fp32)
#pragma unroll 4
  for (int64_t c = lane; c < nch; c += 32) {
    const uint4 q = __ldg(base + c);
    const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&q);
    float a = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(p2[e]);
      a = fmaf(f.x, f.x, a);
      a = fmaf(f.y, f.y, a);
    }
    acc += a;
  }
  acc = warp_sum(acc);
  if (lane == 0) norms[w] = (float)sqrt(acc);
}

// Folded units, float32: the same warp-per-block stream (four 16-B loads in flight)
__global__ void block_norms_flat_f32_kernel(const float* __restrict__ pool, int64_t nvec, int64_t E,
                                            float* __restrict__ norms) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nvec) return;
  const float4* base = reinterpret_cast<const float4*>(pool + w * E);
  const int64_t nch = E / 4;
  double acc = 0.0;
#pragma unroll 4
  for (int64_t c = lane; c < nch; c += 32) {
    const float4 q = __ldg(base + c);
    acc = fma((double)q.x, (double)q.x, acc);
    acc = fma((double)q.y, (double)q.y, acc);
    acc = fma((double)q.z, (double)q.z, acc);
    acc = fma((double)q.w, (double)q.w, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) norms[w] = (float)sqrt(acc);
}

template <typename T>
static cudaError_t norms_t(const void* pool, const Geom& g, void* norms, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  const int64_t nvec = g.units() * g.NB;
  const int64_t blocks = (nvec * 32 + 255) / 256;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (g.head_mode && g.d == 128 && g.h == 8 && g.t == 16 &&
        (reinterpret_cast<uintptr_t>(pool) & 15) == 0) {
      const int64_t nblk = g.L * g.NB;
      block_norms_heads_kernel<<<(unsigned)((nblk * 32 + 255) / 256), 256, 0, s>>>(
          (const __nv_bfloat16*)pool, g, (float*)norms);
      return cudaGetLastError();
    }
    if (!g.head_mode && g.E() % 8 == 0 && (reinterpret_cast<uintptr_t>(pool) & 15) == 0) {
      block_norms_flat_kernel<<<(unsigned)blocks, 256, 0, s>>>((const __nv_bfloat16*)pool, nvec, g.E(),
                                                               (float*)norms);
      return cudaGetLastError();
    }
  }
  if constexpr (std::is_same<T, float>::value) {
    if (!g.head_mode && g.E() % 4 == 0 && (reinterpret_cast<uintptr_t>(pool) & 15) == 0) {
      block_norms_flat_f32_kernel<<<(unsigned)blocks, 256, 0, s>>>((const float*)pool, nvec, g.E(),
                                                                   (float*)norms);
      return cudaGetLastError();
    }
  }
  if (can_vectorize<T>(pool, g))
    block_norms_kernel<T, Vec16<T>::N><<<(unsigned)blocks, 256, 0, s>>>((const T*)pool, g, (A*)norms);
  else
    block_norms_kernel<T, 1><<<(unsigned)blocks, 256, 0, s>>>((const T*)pool, g, (A*)norms);
  return cudaGetLastError();
}

cudaError_t launch_block_norms(const void* pool, int dtype, const Geom& g, void* norms,
                               cudaStream_t s) {
  switch (dtype) {
    case F64: return norms_t<double>(pool, g, norms, s);
    case F32: return norms_t<float>(pool, g, norms, s);
    default: return norms_t<__nv_bfloat16>(pool, g, norms, s);
  }
}

// --------------------------------------------------------------------------
// state init
// --------------------------------------------------------------------------
template <typename A>
__global__ void state_init_kernel(int64_t U, int64_t NB, const A* __restrict__ knorm,
                                  uint8_t* fusable, uint8_t* alive, int32_t* absorber,
                                  int32_t* table, int32_t* refcount) {
  const int64_t n = U * NB;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (knorm) fusable[x] = knorm[x] > A(0) ? 1 : 0;
    alive[x] = 1;
    absorber[x] = kNone;
    table[x] = (int32_t)(x % NB);
    refcount[x] = 1;
  }
}

cudaError_t launch_state_init(int dtype, int64_t U, int64_t NB, const void* knorm,
                              uint8_t* fusable, uint8_t* alive, int32_t* absorber,
                              int32_t* table, int32_t* refcount, cudaStream_t s) {
  const int64_t n = U * NB;
  const int grid = (int)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  if (n == 0) return cudaSuccess;
  if (dtype == F64)
    state_init_kernel<<<grid, 256, 0, s>>>(U, NB, (const double*)knorm, fusable, alive,
                                           absorber, table, refcount);
  else
    state_init_kernel<<<grid, 256, 0, s>>>(U, NB, (const float*)knorm, fusable, alive,
                                           absorber, table, refcount);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// K5: remap. Slot s follows its block if that block was absorbed this level;
// absorbed blocks hand their refcount to the absorber and die.
// --------------------------------------------------------------------------
__global__ void remap_kernel(int64_t u0, int64_t nU, int64_t NB, int64_t n_total,
                             const int32_t* __restrict__ absorber, int32_t* table,
                             int32_t* refcount, uint8_t* alive, int32_t* flag) {
  const int64_t n = nU * NB;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gb = (u0 + x / NB) * NB;
    const int64_t s = x % NB;
    const int32_t p = table[gb + s];
    const int32_t a = absorber[gb + p];
    if (a != kNone) table[gb + s] = a;
    const int32_t aj = absorber[gb + s];
    if (alive[gb + s] && aj != kNone) {
      atomicAdd(&refcount[gb + aj], refcount[gb + s]);
      refcount[gb + s] = 0;
      alive[gb + s] = 0;
    }
    flag[gb + s] = 0;  // member count (LevelWs::mcnt)
    flag[n_total + gb + s] = 0;  // member fill (LevelWs::mfill)
  }
}

cudaError_t launch_remap(int64_t u0, int64_t nU, int64_t NB, int64_t n_total,
                         const int32_t* absorber, int32_t* table, int32_t* refcount,
                         uint8_t* alive, int32_t* level_ws, cudaStream_t s) {
  const int64_t n = nU * NB;
  if (n == 0) return cudaSuccess;
  const int grid = (int)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  remap_kernel<<<grid, 256, 0, s>>>(u0, nU, NB, n_total, absorber, table, refcount, alive,
                                    level_ws);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// finalize
// --------------------------------------------------------------------------
template <typename A>
__global__ void scales_kernel(int64_t u0, int64_t nU, int64_t NB, const A* __restrict__ okn,
                              const A* __restrict__ ovn, const A* __restrict__ kn,
                              const A* __restrict__ vn, const int32_t* __restrict__ table,
                              A* ks, A* vs) {
  const int64_t n = nU * NB;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gb = (u0 + x / NB) * NB;
    const int64_t s = gb + x % NB;
    const int64_t p = gb + table[s];
    ks[s] = kn[p] > A(0) ? okn[s] / kn[p] : A(0);
    vs[s] = vn[p] > A(0) ? ovn[s] / vn[p] : A(0);
  }
}

// ordered stream compaction of alive / dead ids, one CTA per unit
__global__ void lists_kernel(int64_t u0, int64_t NB, const uint8_t* __restrict__ alive,
                             int32_t* live_ids, int32_t* live_count, int32_t* free_ids,
                             int32_t* free_count) {
  __shared__ int wl[32], wf[32];
  __shared__ int base_l, base_f;
  const int64_t u = u0 + blockIdx.x;
  const int64_t gb = u * NB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) base_l = base_f = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < NB; c0 += blockDim.x) {
    const int64_t i = c0 + threadIdx.x;
    const bool in = i < NB;
    const bool al = in && alive[gb + i];
    const unsigned bl = __ballot_sync(0xffffffffu, al);
    const unsigned bf = __ballot_sync(0xffffffffu, in && !al);
    if (lane == 0) {
      wl[warp] = __popc(bl);
      wf[warp] = __popc(bf);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int rl = base_l, rf = base_f;
      for (int w = 0; w < nw; ++w) {
        int a = wl[w], b = wf[w];
        wl[w] = rl;
        wf[w] = rf;
        rl += a;
        rf += b;
      }
      base_l = rl;
      base_f = rf;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    if (al) live_ids[gb + wl[warp] + __popc(bl & lt)] = (int32_t)i;
    else if (in) free_ids[gb + wf[warp] + __popc(bf & lt)] = (int32_t)i;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    live_count[u] = base_l;
    free_count[u] = base_f;
  }
}

cudaError_t launch_finalize(int dtype, int64_t u0, int64_t nU, int64_t NB, const void* okn,
                            const void* ovn, const void* kn, const void* vn,
                            const int32_t* table, const uint8_t* alive, void* ks, void* vs,
                            int32_t* live_ids, int32_t* live_count, int32_t* free_ids,
                            int32_t* free_count, cudaStream_t s) {
  const int64_t n = nU * NB;
  if (n == 0) return cudaSuccess;
  const int grid = (int)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  if (dtype == F64)
    scales_kernel<<<grid, 256, 0, s>>>(u0, nU, NB, (const double*)okn, (const double*)ovn,
                                       (const double*)kn, (const double*)vn, table,
                                       (double*)ks, (double*)vs);
  else
    scales_kernel<<<grid, 256, 0, s>>>(u0, nU, NB, (const float*)okn, (const float*)ovn,
                                       (const float*)kn, (const float*)vn, table, (float*)ks,
                                       (float*)vs);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (live_ids) {
    lists_kernel<<<(unsigned)nU, 1024, 0, s>>>(u0, NB, alive, live_ids, live_count, free_ids,
                                               free_count);
    e = cudaGetLastError();
  }
  return e;
}

// --------------------------------------------------------------------------
// audit / redirect
// --------------------------------------------------------------------------
__global__ void audit_hist_kernel(int64_t U, int64_t NB, const int32_t* __restrict__ table,
                                  const uint8_t* __restrict__ alive, int32_t* hist,
                                  int32_t* bad) {
  const int64_t n = U * NB;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gb = (x / NB) * NB;
    const int32_t p = table[x];
    if (p < 0 || p >= NB || !alive[gb + p]) {
      atomicOr(bad, 1);
    } else {
      atomicAdd(&hist[gb + p], 1);
    }
  }
}

__global__ void audit_cmp_kernel(int64_t n, const int32_t* __restrict__ hist,
                                 const int32_t* __restrict__ refcount,
                                 const uint8_t* __restrict__ alive, int32_t* bad) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const bool al = alive[x];
    if (hist[x] != refcount[x] || (al && refcount[x] <= 0) || (!al && refcount[x] != 0))
      atomicOr(bad, 2);
  }
}

cudaError_t launch_table_audit(int64_t U, int64_t NB, const int32_t* table,
                               const int32_t* refcount, const uint8_t* alive,
                               int32_t* scratch, int32_t* bad, cudaStream_t s) {
  const int64_t n = U * NB;
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int32_t), s);
  if (e != cudaSuccess || n == 0) return e;
  e = cudaMemsetAsync(scratch, 0, sizeof(int32_t) * n, s);
  if (e != cudaSuccess) return e;
  const int grid = (int)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  audit_hist_kernel<<<grid, 256, 0, s>>>(U, NB, table, alive, scratch, bad);
  audit_cmp_kernel<<<grid, 256, 0, s>>>(n, scratch, refcount, alive, bad);
  return cudaGetLastError();
}

__global__ void redirect_kernel(int64_t NB, int32_t* table, int32_t* refcount, uint8_t* alive,
                                int32_t from, int32_t to, int32_t* bad) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = from >= 0 && from < NB && to >= 0 && to < NB && alive[from] && alive[to] &&
         from != to;
    *bad = ok ? 0 : 1;
  }
  __syncthreads();
  if (!ok) return;
  for (int64_t s = threadIdx.x; s < NB; s += blockDim.x)
    if (table[s] == from) table[s] = to;
  __syncthreads();
  if (threadIdx.x == 0) {
    refcount[to] += refcount[from];
    refcount[from] = 0;
    alive[from] = 0;
  }
}

cudaError_t launch_table_redirect(int64_t NB, int32_t* table, int32_t* refcount,
                                  uint8_t* alive, int32_t from, int32_t to, int32_t* bad,
                                  cudaStream_t s) {
  redirect_kernel<<<1, 1024, 0, s>>>(NB, table, refcount, alive, from, to, bad);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// gather / refold
// --------------------------------------------------------------------------
template <typename T>
__global__ void gather_kernel(const T* __restrict__ pool, Geom g, int64_t u,
                              const int32_t* __restrict__ ids,
                              const typename AccOf<T>::type* __restrict__ norms,
                              const typename AccOf<T>::type* __restrict__ scales,
                              typename AccOf<T>::type* __restrict__ out) {
  using A = typename AccOf<T>::type;
  const int64_t k = blockIdx.x;
  const int32_t id = ids[k];
  A sc = A(1);
  if (norms) {
    const A nv = norms[u * g.NB + id];
    sc = nv > A(0) ? A(1) / nv : A(0);
  }
  if (scales) sc *= scales[k];
  const T* x = pool + g.base(u, id);
  const int64_t r = g.r();
  for (int64_t e = threadIdx.x; e < r; e += blockDim.x) out[k * r + e] = to_acc(x[g.off(e)]) * sc;
}

cudaError_t launch_gather_vectors(const void* pool, int dtype, const Geom& g, int64_t u,
                                  const int32_t* ids, int64_t n, const void* norms,
                                  const void* scales, void* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  switch (dtype) {
    case F64:
      gather_kernel<<<(unsigned)n, 256, 0, s>>>((const double*)pool, g, u, ids,
                                                (const double*)norms, (const double*)scales, (double*)out);
      break;
    case F32:
      gather_kernel<<<(unsigned)n, 256, 0, s>>>((const float*)pool, g, u, ids,
                                                (const float*)norms, (const float*)scales, (float*)out);
      break;
    default:
      gather_kernel<<<(unsigned)n, 256, 0, s>>>((const __nv_bfloat16*)pool, g, u, ids,
                                                (const float*)norms, (const float*)scales, (float*)out);
  }
  return cudaGetLastError();
}

template <typename T>
__global__ void refold_kernel(const T* __restrict__ pool, Geom g, int64_t layer,
                              const int32_t* __restrict__ table,
                              const typename AccOf<T>::type* __restrict__ scale,
                              typename AccOf<T>::type* __restrict__ out) {
  const int64_t s = blockIdx.x;
  const int64_t E = g.E();
  for (int64_t q = threadIdx.x; q < E; q += blockDim.x) {
    const int hh = (int)((q / g.d) % g.h);
    const int64_t u = g.head_mode ? layer * g.h + hh : layer;
    const int64_t slot = u * g.NB + s;
    const int32_t p = table[slot];
    out[s * E + q] = scale[slot] * to_acc(pool[(layer * g.NB + p) * E + q]);
  }
}

cudaError_t launch_refold(const void* pool, int dtype, const Geom& g, int64_t layer,
                          const int32_t* table, const void* scale, void* out,
                          cudaStream_t s) {
  if (g.NB == 0) return cudaSuccess;
  switch (dtype) {
    case F64:
      refold_kernel<<<(unsigned)g.NB, 256, 0, s>>>((const double*)pool, g, layer, table,
                                                   (const double*)scale, (double*)out);
      break;
    case F32:
      refold_kernel<<<(unsigned)g.NB, 256, 0, s>>>((const float*)pool, g, layer, table,
                                                   (const float*)scale, (float*)out);
      break;
    default:
      refold_kernel<<<(unsigned)g.NB, 256, 0, s>>>((const __nv_bfloat16*)pool, g, layer, table,
                                                   (const float*)scale, (float*)out);
  }
  return cudaGetLastError();
}

}  // namespace kvf

namespace kvf {

// --------------------------------------------------------------------------
// compaction helpers for the top tree levels: ascending alive list + rank,
// and a staged copy of the alive K rows (contiguous per unit) for TMA
// --------------------------------------------------------------------------
__global__ void alive_rank_kernel(int64_t u0, int64_t NB, const uint8_t* __restrict__ alive,
                                  int32_t* live, int32_t* rank, int32_t* count) {
  __shared__ int wl[32];
  __shared__ int base;
  const int64_t u = u0 + blockIdx.x;
  const int64_t gb = u * NB;
  int32_t* rk = rank + u * (NB + 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < NB; c0 += blockDim.x) {
    const int64_t i = c0 + threadIdx.x;
    const bool al = i < NB && alive[gb + i];
    const unsigned bl = __ballot_sync(0xffffffffu, al);
    if (lane == 0) wl[warp] = __popc(bl);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = base;
      for (int w = 0; w < nw; ++w) {
        const int a = wl[w];
        wl[w] = run;
        run += a;
      }
      base = run;
    }
    __syncthreads();
    const int pos = wl[warp] + __popc(bl & ((1u << lane) - 1u));
    if (i < NB) rk[i] = pos;
    if (al) live[gb + pos] = (int32_t)i;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    rk[NB] = base;
    count[u] = base;
  }
}

cudaError_t launch_alive_rank(int64_t u0, int64_t nU, int64_t NB, const uint8_t* alive,
                              int32_t* live, int32_t* rank, int32_t* count, cudaStream_t s) {
  if (nU == 0) return cudaSuccess;
  alive_rank_kernel<<<(unsigned)nU, 1024, 0, s>>>(u0, NB, alive, live, rank, count);
  return cudaGetLastError();
}

// one warp per staged row; 16-byte vectors (bf16 x 8)
__global__ void stage_rows_kernel(const __nv_bfloat16* __restrict__ pool, Geom g, int64_t u0,
                                  const int32_t* __restrict__ live,
                                  const int32_t* __restrict__ count, __nv_bfloat16* staged) {
  const int64_t ul = blockIdx.y, u = u0 + ul;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (k >= count[u]) return;
  const int32_t id = live[u * g.NB + k];
  const __nv_bfloat16* src = pool + g.base(u, id);
  __nv_bfloat16* dst = staged + (ul * g.NB + k) * g.r();
  const int64_t nch = g.r() / 8;
#pragma unroll 4
  for (int64_t c = lane; c < nch; c += 32)
    *reinterpret_cast<uint4*>(dst + c * 8) =
        __ldg(reinterpret_cast<const uint4*>(src + g.off(c * 8)));
}

cudaError_t launch_stage_rows(const void* pool, int dtype, const Geom& g, int64_t u0, int64_t nU,
                              const int32_t* live, const int32_t* count, void* staged,
                              cudaStream_t s) {
  if (dtype != BF16 || g.d % 8 != 0) return cudaErrorInvalidValue;
  if (nU == 0) return cudaSuccess;
  dim3 grid((unsigned)((g.NB + 7) / 8), (unsigned)nU);
  stage_rows_kernel<<<grid, 256, 0, s>>>((const __nv_bfloat16*)pool, g, u0, live, count,
                                         (__nv_bfloat16*)staged);
  return cudaGetLastError();
}

}  // namespace kvf
