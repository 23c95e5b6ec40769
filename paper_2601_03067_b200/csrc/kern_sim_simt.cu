// K2 + K3 on CUDA cores: similarity tile + first-match selection epilogue.
// Used for float64 / float32 pools (parity and the CPU-runnable config) and
// as the cross-check of the tcgen05 path for bf16. Replaces fusion.py:244-265:
//   sim = kdir[left] @ kdir[right].T ; absorber(j) = first left row with
//   sim > thr among alive, fusable blocks (strict '>', fusion.py:256).
// One CTA computes a 64 x 64 tile of one merge of one unit.
#include "kernels.h"

namespace kvf {

namespace {
constexpr int TM = kSimtTile, TN = kSimtTile, KC = 32, NT = 256;

template <typename T>
__device__ __forceinline__ void load_chunk(typename AccOf<T>::type (*S)[TM + 1],
                                           const T* __restrict__ pool, const Geom& g,
                                           int64_t u, int start, int nvalid, int64_t k0,
                                           int64_t r) {
  using A = typename AccOf<T>::type;
  // KC consecutive elements per row -> consecutive threads (coalesced)
#pragma unroll
  for (int e = 0; e < (TM * KC) / NT; ++e) {
    const int idx = threadIdx.x + e * NT;
    const int row = idx / KC, kk = idx % KC;
    const int64_t k = k0 + kk;
    A v = A(0);
    if (row < nvalid && k < r) v = to_acc(pool[g.base(u, start + row) + g.off(k)]);
    S[kk][row] = v;
  }
}
}  // namespace

template <typename T>
__global__ void __launch_bounds__(NT)
sim_simt_kernel(const T* __restrict__ pool, Geom g, int64_t u0,
                const typename AccOf<T>::type* __restrict__ knorm,
                const uint8_t* __restrict__ fusable, const uint8_t* __restrict__ alive,
                int32_t* __restrict__ absorber, const int32_t* __restrict__ merges,
                const int32_t* __restrict__ tiles, int nt, typename AccOf<T>::type thr,
                double* __restrict__ partials, double* __restrict__ samples,
                const int64_t* __restrict__ sample_off, int64_t sample_stride) {
  using A = typename AccOf<T>::type;
  __shared__ A As[KC][TM + 1];
  __shared__ A Bs[KC][TN + 1];
  __shared__ A inv_i[TM], inv_j[TN];
  __shared__ uint8_t ok_i[TM], ok_j[TN];
  __shared__ int32_t colmin[TN];
  __shared__ double red[32];

  const int tile = blockIdx.x;
  const int64_t ul = blockIdx.y, u = u0 + ul;
  const int64_t gb = u * g.NB;
  const int m = tiles[3 * tile], i0 = tiles[3 * tile + 1], j0 = tiles[3 * tile + 2];
  const int lb = merges[3 * m], mid = merges[3 * m + 1], re = merges[3 * m + 2];
  const int left_n = mid - lb, right_n = re - mid;
  const int ni = min(TM, left_n - i0), nj = min(TN, right_n - j0);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;

  if (threadIdx.x < TM) {
    const int r_ = threadIdx.x;
    const int64_t bi = gb + lb + i0 + r_;
    bool ok = r_ < ni && alive[bi] && fusable[bi];
    A nv = ok ? knorm[bi] : A(0);
    ok_i[r_] = ok;
    inv_i[r_] = nv > A(0) ? A(1) / nv : A(0);
  } else if (threadIdx.x < TM + TN) {
    const int c_ = threadIdx.x - TM;
    const int64_t bj = gb + mid + j0 + c_;
    bool ok = c_ < nj && alive[bj] && fusable[bj];
    A nv = ok ? knorm[bj] : A(0);
    ok_j[c_] = ok;
    inv_j[c_] = nv > A(0) ? A(1) / nv : A(0);
    colmin[c_] = kNone;
  }

  // two-level accumulation: KC-long partial dot products in A, summed in
  // double across chunks (a long sequential fp32 sum over r = 16K terms would
  // cost ~1e-5 of similarity accuracy)
  double accd[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) accd[a][b] = 0.0;

  const int64_t r = g.r();
  for (int64_t k0 = 0; k0 < r; k0 += KC) {
    __syncthreads();
    load_chunk<T>(As, pool, g, u, lb + i0, ni, k0, r);
    load_chunk<T>(Bs, pool, g, u, mid + j0, nj, k0, r);
    __syncthreads();
    A acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = A(0);
#pragma unroll 8
    for (int kk = 0; kk < KC; ++kk) {
      A av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += av[a] * bv[b];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) accd[a][b] += (double)acc[a][b];
  }
  __syncthreads();
  A acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = (A)accd[a][b];

  // epilogue: scale, mask, stats, per-column first match
  double cnt = 0, s1 = 0, s2 = 0, mn = INFINITY, mx = -INFINITY;
  double* samp = nullptr;
  if (samples) samp = samples + ul * sample_stride + sample_off[m];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int c_ = tx + 16 * b;
    int32_t best = kNone;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r_ = ty + 16 * a;
      const bool ok = ok_i[r_] && ok_j[c_];
      const A s = acc[a][b] * inv_i[r_] * inv_j[c_];
      if (ok) {
        const double sd = (double)s;
        cnt += 1.0;
        s1 += sd;
        s2 += sd * sd;
        mn = fmin(mn, sd);
        mx = fmax(mx, sd);
        if (s > thr) best = min(best, (int32_t)(lb + i0 + r_));
      }
      if (samp && r_ < ni && c_ < nj)
        samp[(int64_t)(i0 + r_) * right_n + (j0 + c_)] = ok ? (double)s : (double)NAN;
    }
    if (best != kNone) atomicMin(&colmin[c_], best);
  }
  cnt = block_sum(cnt, red);
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double smn[NT / 32], smx[NT / 32];
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x < TN) {
    const int32_t cm = colmin[threadIdx.x];
    if (cm != kNone) atomicMin(&absorber[gb + mid + j0 + threadIdx.x], cm);
  }
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    double* o = partials + (ul * nt + tile) * 5;
    o[0] = cnt;
    o[1] = s1;
    o[2] = s2;
    o[3] = mn;
    o[4] = mx;
  }
}

template <typename T>
static cudaError_t sim_simt_t(const SimArgs& a, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  A thr;
  if (sizeof(A) == 8) {
    thr = (A)a.thr;
  } else {
    // largest float <= thr: (float)sim > thr_f  <=>  (double)sim > thr
    float f = (float)a.thr;
    if ((double)f > a.thr) f = nextafterf(f, -INFINITY);
    thr = (A)f;
  }
  dim3 grid(a.nt, (unsigned)a.nU);
  sim_simt_kernel<T><<<grid, NT, 0, s>>>((const T*)a.pool, a.g, a.u0, (const A*)a.knorm,
                                         a.fusable, a.alive, a.absorber, a.merges, a.tiles,
                                         a.nt, thr, a.partials, a.samples, a.sample_off,
                                         a.sample_stride);
  return cudaGetLastError();
}

cudaError_t launch_sim_simt(const SimArgs& a, cudaStream_t s) {
  if (a.nt == 0 || a.nU == 0) return cudaSuccess;
  switch (a.dtype) {
    case F64: return sim_simt_t<double>(a, s);
    case F32: return sim_simt_t<float>(a, s);
    default: return sim_simt_t<__nv_bfloat16>(a, s);
  }
}

}  // namespace kvf
