// Bandwidth-bound kernels of the fusion pipeline (sm_100a):
//   K1  block norms            (core.py:115-119)
//   --  state init             (fusion.py:208-228, core.py:191-201)
//   --  per-merge level stats  (fusion.py:249, 273-281)
//   K4  in-place block merge   (fusion.py:259-261, 285-287)
//   K5  table remap/refcounts  (core.py:217-227, fusion.py:262-264)
//   --  finalize: per-slot scales, live/free lists (fusion.py:316-324)
//   --  audit / redirect / gather / refold (core.py:232-241, 285-305)
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
  A acc = 0;
  for (int64_t c = lane; c < nch; c += 32) {
    A v[VEC];
    VecIO<T, VEC>::load_nc(base + g.off(c * VEC), v);
#pragma unroll
    for (int q = 0; q < VEC; ++q) acc += v[q] * v[q];
  }
  acc = warp_sum(acc);
  if (lane == 0) norms[w] = sqrt(acc);
}

template <typename T>
static cudaError_t norms_t(const void* pool, const Geom& g, void* norms, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  const int64_t nvec = g.units() * g.NB;
  const int64_t blocks = (nvec * 32 + 255) / 256;
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
    fusable[x] = knorm[x] > A(0) ? 1 : 0;
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
// Level statistics + absorber marking: one CTA per (merge, unit).
// --------------------------------------------------------------------------
__global__ void level_stats_kernel(int64_t u0, int64_t NB, const uint8_t* __restrict__ fusable,
                                   const uint8_t* __restrict__ alive,
                                   const int32_t* __restrict__ absorber,
                                   const int32_t* __restrict__ merges, int nm,
                                   const int32_t* __restrict__ tile_off, int nt,
                                   const double* __restrict__ partials, double* stats,
                                   int32_t* flag, int32_t* list, int32_t* count) {
  __shared__ double red[32];
  const int m = blockIdx.x;
  const int64_t ul = blockIdx.y, u = u0 + ul;
  const int64_t gb = u * NB;
  const int lb = merges[3 * m], mid = merges[3 * m + 1], re = merges[3 * m + 2];
  double nl = 0, nr = 0, nf = 0;
  for (int i = lb + threadIdx.x; i < mid; i += blockDim.x)
    nl += (alive[gb + i] && fusable[gb + i]) ? 1.0 : 0.0;
  for (int j = mid + threadIdx.x; j < re; j += blockDim.x) {
    const bool al = alive[gb + j];
    nr += (al && fusable[gb + j]) ? 1.0 : 0.0;
    const int32_t a = absorber[gb + j];
    if (al && a != kNone) {
      nf += 1.0;
      if (atomicAdd(&flag[gb + a], 1) == 0) {  // flag = member count of absorber a
        const int pos = atomicAdd(count, 1);
        list[pos] = (int32_t)(gb + a);
      }
    }
  }
  // similarity partials of this merge's tiles (fixed order => deterministic)
  double c = 0, s1 = 0, s2 = 0, mn = INFINITY, mx = -INFINITY;
  const double* pb = partials + ul * (int64_t)nt * 5;
  for (int tt = tile_off[m] + threadIdx.x; tt < tile_off[m + 1]; tt += blockDim.x) {
    const double* q = pb + (int64_t)tt * 5;
    c += q[0];
    s1 += q[1];
    s2 += q[2];
    mn = fmin(mn, q[3]);
    mx = fmax(mx, q[4]);
  }
  nl = block_sum(nl, red);
  nr = block_sum(nr, red);
  nf = block_sum(nf, red);
  c = block_sum(c, red);
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  // min / max are order independent
  __shared__ double smn[32], smx[32];
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    double* o = stats + (ul * nm + m) * 8;
    o[0] = nl; o[1] = nr; o[2] = nf; o[3] = c; o[4] = s1; o[5] = s2;
    o[6] = c > 0 ? mn : 0.0;
    o[7] = c > 0 ? mx : 0.0;
  }
}

cudaError_t launch_level_stats(int64_t u0, int64_t nU, int64_t NB, const uint8_t* fusable,
                               const uint8_t* alive, const int32_t* absorber,
                               const int32_t* merges, int nm, const int32_t* tile_off,
                               int nt, const double* partials, double* stats,
                               int32_t* flag, int32_t* list, int32_t* count, cudaStream_t s) {
  if (nm == 0 || nU == 0) return cudaSuccess;
  dim3 grid(nm, (unsigned)nU);
  level_stats_kernel<<<grid, 256, 0, s>>>(u0, NB, fusable, alive, absorber, merges, nm,
                                          tile_off, nt, partials, stats, flag, list, count);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// K4: merge. Persistent grid (x = absorber list stride, y = 0:K / 1:V).
// Member lists are bucketed per absorber (count -> segment -> scatter); each
// CTA sorts its absorber's members ascending (rank sort in smem) so the fp
// summation order is fixed and the result is bitwise deterministic. Groups
// larger than the smem list fall back to an ordered scan of the right range.
// --------------------------------------------------------------------------
constexpr int kMaxSorted = 512;

__global__ void member_seg_kernel(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                                  const int32_t* __restrict__ mcnt, int32_t* mstart,
                                  int32_t* cursor) {
  const int n = *count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t a = list[i];
    mstart[a] = atomicAdd(cursor, mcnt[a]);
  }
}

__global__ void member_scatter_kernel(int64_t n, int64_t NB, const uint8_t* __restrict__ alive,
                                      const int32_t* __restrict__ absorber,
                                      const int32_t* __restrict__ mstart, int32_t* mfill,
                                      int32_t* members) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int32_t aj = absorber[x];
    if (aj != kNone && alive[x]) {
      const int64_t a = (x / NB) * NB + aj;
      const int slot = atomicAdd(&mfill[a], 1);
      members[mstart[a] + slot] = (int32_t)(x % NB);
    }
  }
}

template <typename T, int VEC>
__global__ void __launch_bounds__(512, 1)
merge_kernel(T* __restrict__ pool_k, T* __restrict__ pool_v, Geom g,
             typename AccOf<T>::type* __restrict__ knorm,
             typename AccOf<T>::type* __restrict__ vnorm,
             const typename AccOf<T>::type* __restrict__ oknorm,
             const typename AccOf<T>::type* __restrict__ ovnorm,
             const int32_t* __restrict__ absorber, const int32_t* __restrict__ merges,
             const int32_t* __restrict__ row_merge, int bpr,
             const int32_t* __restrict__ list, const int32_t* __restrict__ count,
             const int32_t* __restrict__ mcnt, const int32_t* __restrict__ mstart,
             const int32_t* __restrict__ members_g) {
  using A = typename AccOf<T>::type;
  constexpr int MAXQ = 32 / VEC;
  __shared__ A red[32];
  __shared__ int32_t raw[kMaxSorted];
  __shared__ int32_t members[kMaxSorted];
  __shared__ int warp_cnt[16];
  __shared__ int nmem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bd = blockDim.x;
  const bool is_v = blockIdx.y == 1;
  T* pool = is_v ? pool_v : pool_k;
  A* norm = is_v ? vnorm : knorm;
  const A* onorm = is_v ? ovnorm : oknorm;
  const int64_t nch = g.r() / VEC;
  const int n_items = *count;

  auto accumulate = [&](A (&acc)[MAXQ][VEC], int64_t u, int n) {
    const int64_t gb = u * g.NB;
    for (int k = 0; k < n; ++k) {
      const int32_t jm = members[k];
      const A nj = norm[gb + jm];
      const A inv = nj > A(0) ? A(1) / nj : A(0);
      const T* xj = pool + g.base(u, jm);
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int64_t c = tid + (int64_t)q * bd;
        if (c < nch) {
          A v[VEC];
          VecIO<T, VEC>::load(xj + g.off(c * VEC), v);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[q][e] += v[e] * inv;
        }
      }
    }
  };

  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int64_t gid = list[it];
    const int64_t u = gid / g.NB;
    const int32_t l = (int32_t)(gid % g.NB);
    const int64_t gb = u * g.NB;
    const int nmemb = mcnt[gid];
    A acc[MAXQ][VEC];
    {
      const A nl = norm[gid];
      const A inv = nl > A(0) ? A(1) / nl : A(0);
      const T* xl = pool + g.base(u, l);
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int64_t c = tid + (int64_t)q * bd;
        if (c < nch) {
          VecIO<T, VEC>::load(xl + g.off(c * VEC), acc[q]);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[q][e] *= inv;
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[q][e] = A(0);
        }
      }
    }
    if (nmemb <= kMaxSorted) {
      const int s0 = mstart[gid];
      for (int k = tid; k < nmemb; k += bd) raw[k] = members_g[s0 + k];
      __syncthreads();
      for (int k = tid; k < nmemb; k += bd) {  // rank sort (ids are distinct)
        const int32_t v = raw[k];
        int rank = 0;
        for (int q = 0; q < nmemb; ++q) rank += raw[q] < v;
        members[rank] = v;
      }
      __syncthreads();
      accumulate(acc, u, nmemb);
      __syncthreads();
    } else {
      const int m = row_merge[l / bpr];
      const int mid = merges[3 * m + 1], re = merges[3 * m + 2];
      for (int j0 = mid; j0 < re; j0 += bd) {
        const int j = j0 + tid;
        const bool match = j < re && absorber[gb + j] == l;
        const unsigned bal = __ballot_sync(0xffffffffu, match);
        if (lane == 0) warp_cnt[warp] = __popc(bal);
        __syncthreads();
        if (tid == 0) {
          int run = 0;
          for (int w = 0; w < (bd >> 5); ++w) {
            const int cnum = warp_cnt[w];
            warp_cnt[w] = run;
            run += cnum;
          }
          nmem = run;
        }
        __syncthreads();
        if (match) members[warp_cnt[warp] + __popc(bal & ((1u << lane) - 1u))] = j;
        __syncthreads();
        accumulate(acc, u, nmem);
        __syncthreads();
      }
    }
    A ss = 0;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) ss += acc[q][e] * acc[q][e];
    const A nrm = sqrt(block_sum(ss, red));
    const A home = onorm[gid];
    const A sc = nrm > A(0) ? (home > A(0) ? home : A(1)) / nrm : A(0);
    T* xl = pool + g.base(u, l);
    A rs = 0;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int64_t c = tid + (int64_t)q * bd;
      if (c < nch) {
        A v[VEC], rd[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[e] = acc[q][e] * sc;
        VecIO<T, VEC>::store(xl + g.off(c * VEC), v, rd);
#pragma unroll
        for (int e = 0; e < VEC; ++e) rs += rd[e] * rd[e];
      }
    }
    const A nn = sqrt(block_sum(rs, red));
    if (tid == 0) norm[gid] = nn;
    __syncthreads();
  }
}

struct MergeWs {  // int32 workspace: [mfill | cursor | pad | mstart | members]
  int32_t *mfill, *cursor, *mstart, *members;
  MergeWs(int32_t* ws, int64_t n) : mfill(ws), cursor(ws + n), mstart(ws + n + 32), members(ws + 2 * n + 32) {}
};

template <typename T, int VEC>
static cudaError_t merge_t(void* pk, void* pv, const Geom& g, void* kn, void* vn,
                           const void* okn, const void* ovn, const int32_t* absorber,
                           const uint8_t* alive, const int32_t* merges, const int32_t* row_merge,
                           int bpr, const int32_t* list, const int32_t* count, const int32_t* mcnt,
                           int32_t* ws, int64_t cap, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  const int64_t nch = g.r() / VEC;
  int bd = 512;
  while (bd > 64 && (int64_t)(bd / 2) * (32 / VEC) >= nch) bd /= 2;  // small vectors: small CTAs
  if (nch > (int64_t)bd * (32 / VEC)) return cudaErrorInvalidValue;
  const int64_t n = g.units() * g.NB;
  MergeWs w(ws, n);
  cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(int32_t) * (n + 1), s);
  if (e != cudaSuccess) return e;
  const int sgrid = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  member_seg_kernel<<<sgrid, 256, 0, s>>>(list, count, mcnt, w.mstart, w.cursor);
  member_scatter_kernel<<<sgrid, 256, 0, s>>>(n, g.NB, alive, absorber, w.mstart, w.mfill,
                                              w.members);
  int64_t gx = cap < 148 * 4 ? cap : 148 * 4;
  if (gx < 1) gx = 1;
  dim3 grid((unsigned)gx, 2);
  merge_kernel<T, VEC><<<grid, bd, 0, s>>>((T*)pk, (T*)pv, g, (A*)kn, (A*)vn, (const A*)okn,
                                           (const A*)ovn, absorber, merges, row_merge, bpr,
                                           list, count, mcnt, w.mstart, w.members);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t merge_dispatch(void* pk, void* pv, const Geom& g, void* kn, void* vn,
                                  const void* okn, const void* ovn, const int32_t* absorber,
                                  const uint8_t* alive, const int32_t* merges,
                                  const int32_t* row_merge, int bpr, const int32_t* list,
                                  const int32_t* count, const int32_t* mcnt, int32_t* ws,
                                  int64_t cap, cudaStream_t s) {
  if (can_vectorize<T>(pk, g) && can_vectorize<T>(pv, g))
    return merge_t<T, Vec16<T>::N>(pk, pv, g, kn, vn, okn, ovn, absorber, alive, merges,
                                   row_merge, bpr, list, count, mcnt, ws, cap, s);
  return merge_t<T, 1>(pk, pv, g, kn, vn, okn, ovn, absorber, alive, merges, row_merge, bpr,
                       list, count, mcnt, ws, cap, s);
}

int64_t merge_workspace_ints(int64_t n_total) { return 3 * n_total + 64; }

cudaError_t launch_merge_groups(void* pool_k, void* pool_v, int dtype, const Geom& g,
                                void* knorm, void* vnorm, const void* oknorm,
                                const void* ovnorm, const int32_t* absorber,
                                const uint8_t* alive, const int32_t* merges,
                                const int32_t* row_merge, int bpr, const int32_t* list,
                                const int32_t* count, const int32_t* mcnt, int32_t* ws,
                                int64_t cap, cudaStream_t s) {
  switch (dtype) {
    case F64:
      return merge_dispatch<double>(pool_k, pool_v, g, knorm, vnorm, oknorm, ovnorm, absorber,
                                    alive, merges, row_merge, bpr, list, count, mcnt, ws, cap, s);
    case F32:
      return merge_dispatch<float>(pool_k, pool_v, g, knorm, vnorm, oknorm, ovnorm, absorber,
                                   alive, merges, row_merge, bpr, list, count, mcnt, ws, cap, s);
    default:
      return merge_dispatch<__nv_bfloat16>(pool_k, pool_v, g, knorm, vnorm, oknorm, ovnorm,
                                           absorber, alive, merges, row_merge, bpr, list, count,
                                           mcnt, ws, cap, s);
  }
}

// --------------------------------------------------------------------------
// K5: remap. Slot s follows its block if that block was absorbed this level;
// absorbed blocks hand their refcount to the absorber and die.
// --------------------------------------------------------------------------
__global__ void remap_kernel(int64_t u0, int64_t nU, int64_t NB,
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
    flag[gb + s] = 0;
  }
}

cudaError_t launch_remap(int64_t u0, int64_t nU, int64_t NB, const int32_t* absorber,
                         int32_t* table, int32_t* refcount, uint8_t* alive, int32_t* flag,
                         cudaStream_t s) {
  const int64_t n = nU * NB;
  if (n == 0) return cudaSuccess;
  const int grid = (int)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  remap_kernel<<<grid, 256, 0, s>>>(u0, nU, NB, absorber, table, refcount, alive, flag);
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
