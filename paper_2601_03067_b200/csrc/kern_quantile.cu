// Exact quantile of the similarity samples on the device (SURVEY §8f rank 3:
// percentile mode of the threshold controller, fusion.py:418-437, without
// copying the samples to the host).
//
// np.quantile(samples, q) with numpy's default 'linear' method: h = (n-1) q,
// k0 = floor(h), k1 = min(k0 + 1, n - 1), t = h - k0, result = lerp(x_k0,
// x_k1, t) with numpy's two-sided lerp (b - (b-a)(1-t) when t >= 0.5). The
// samples are any number of float64 device segments (per-level sample rows of
// a fusion run); NaN entries (masked pairs) are skipped. Order statistics come
// from an 8-pass radix select over order-preserving 64-bit keys, both ranks in
// the same passes (per-block shared-memory histograms, then global adds).
#include "kernels.h"

namespace kvf {

namespace {
struct QSeg {
  const double* ptr;
  int64_t len;
};
constexpr int QMAXSEG = 128;  // segments per launch (passed by value, 2 KB of parameters)
struct QSegs {
  QSeg s[QMAXSEG];
  int n;
};
struct QState {
  unsigned long long n;       // valid (non-NaN) samples
  unsigned long long rank[2]; // remaining rank inside the current prefix
  unsigned long long prefix[2];
  double t;                   // interpolation weight
  int empty;
};
constexpr int QB = 256;  // threads per block

__device__ __forceinline__ unsigned long long okey(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unkey(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void q_count_kernel(const __grid_constant__ QSegs segs, QState* st) {
  unsigned long long c = 0;
  for (int s = 0; s < segs.n; ++s) {
    const double* p = segs.s[s].ptr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < segs.s[s].len;
         i += (int64_t)gridDim.x * blockDim.x)
      c += isnan(p[i]) ? 0ull : 1ull;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&st->n, c);
}

__global__ void q_init_kernel(QState* st, double q) {
  const unsigned long long n = st->n;
  st->empty = n == 0;
  if (n == 0) return;
  const double h = (double)(n - 1) * q;
  double k0 = floor(h);
  if (k0 < 0) k0 = 0;
  if (k0 > (double)(n - 1)) k0 = (double)(n - 1);
  const unsigned long long i0 = (unsigned long long)k0;
  const unsigned long long i1 = i0 + 1 < n ? i0 + 1 : n - 1;
  st->t = h - k0;
  st->rank[0] = i0;
  st->rank[1] = i1;
  st->prefix[0] = st->prefix[1] = 0;
}

// histogram of digit `shift` of the keys that share both targets' prefixes above it
__global__ void q_hist_kernel(const __grid_constant__ QSegs segs, const QState* st, int shift,
                              unsigned long long* hist /* [2][256] */) {
  __shared__ unsigned int h[2][256];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const unsigned long long hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
  const unsigned long long p0 = st->prefix[0] & hi_mask, p1 = st->prefix[1] & hi_mask;
  for (int s = 0; s < segs.n; ++s) {
    const double* p = segs.s[s].ptr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < segs.s[s].len;
         i += (int64_t)gridDim.x * blockDim.x) {
      const double x = p[i];
      if (isnan(x)) continue;
      const unsigned long long k = okey(x);
      const unsigned d = (unsigned)((k >> shift) & 255u);
      if ((k & hi_mask) == p0) atomicAdd(&h[0][d], 1u);
      if ((k & hi_mask) == p1) atomicAdd(&h[1][d], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    const unsigned v = (&h[0][0])[i];
    if (v) atomicAdd(&hist[i], (unsigned long long)v);
  }
}

__global__ void q_pick_kernel(QState* st, int shift, unsigned long long* hist) {
  if (threadIdx.x < 2 && !st->empty) {
    const int r = threadIdx.x;
    unsigned long long rem = st->rank[r], run = 0;
    unsigned d = 0;
    for (; d < 255; ++d) {
      const unsigned long long c = hist[r * 256 + d];
      if (run + c > rem) break;
      run += c;
    }
    st->rank[r] = rem - run;
    st->prefix[r] |= (unsigned long long)d << shift;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) hist[i] = 0;  // ready for the next pass
}

__global__ void q_final_kernel(const QState* st, double* out) {
  if (st->empty) {
    *out = __longlong_as_double(0x7ff8000000000000ll);  // NaN: no samples
    return;
  }
  const double a = unkey(st->prefix[0]), b = unkey(st->prefix[1]);
  const double t = st->t;
  const double diff = b - a;
  *out = t >= 0.5 ? b - diff * (1.0 - t) : a + diff * t;  // numpy _lerp
}
}  // namespace

int64_t quantile_ws_bytes() { return 512 * 8 + 128; }

cudaError_t launch_quantile(const void* const* parts, const int64_t* lens, int nseg, double q,
                            double* out, void* ws, cudaStream_t s) {
  auto* hist = reinterpret_cast<unsigned long long*>(ws);
  auto* st = reinterpret_cast<QState*>(reinterpret_cast<uint8_t*>(ws) + 512 * 8);
  cudaError_t e = cudaMemsetAsync(ws, 0, quantile_ws_bytes(), s);
  if (e != cudaSuccess) return e;
  const int grid = 148 * 4;
  // segments travel as kernel parameters, QMAXSEG per launch (no host sync)
  auto for_chunks = [&](auto&& launch) {
    for (int c0 = 0; c0 < nseg || (c0 == 0 && nseg == 0); c0 += QMAXSEG) {
      QSegs sg;
      sg.n = nseg - c0 < QMAXSEG ? nseg - c0 : QMAXSEG;
      for (int i = 0; i < sg.n; ++i)
        sg.s[i] = QSeg{reinterpret_cast<const double*>(parts[c0 + i]), lens[c0 + i]};
      launch(sg);
      if (nseg == 0) break;
    }
  };
  for_chunks([&](const QSegs& sg) { q_count_kernel<<<grid, QB, 0, s>>>(sg, st); });
  q_init_kernel<<<1, 1, 0, s>>>(st, q);
  for (int shift = 56; shift >= 0; shift -= 8) {
    for_chunks([&](const QSegs& sg) { q_hist_kernel<<<grid, QB, 0, s>>>(sg, st, shift, hist); });
    q_pick_kernel<<<1, 256, 0, s>>>(st, shift, hist);
  }
  q_final_kernel<<<1, 1, 0, s>>>(st, out);
  return cudaGetLastError();
}

}  // namespace kvf
