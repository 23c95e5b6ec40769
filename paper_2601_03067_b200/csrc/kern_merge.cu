// Per-level bookkeeping and K4 (merge) of the fusion tree.
//
// level_stats (CTA per (merge, unit)):
//   * MergeRecord counters (fusion.py:273-281): alive fusable left / right
//     blocks, fused count, similarity moments reduced in fixed order from the
//     similarity kernel's per-tile partials;
//   * member lists: per absorber l of this merge, the ascending list of right
//     blocks j with absorber[j] == l (the `rids` of fusion.py:256-259) built
//     with an ordered, warp-sequential scatter, so every merge sums its members
//     in ascending order -> bitwise deterministic results without sorting.
// merge (K4, fusion.py:259-261, _unit 285-287): for each (absorber, K|V)
//   dir = unit(dir_l + sum_j dir_j) rewritten in place as s_home * dir.
//   Main path: persistent CTAs, one producer warp streaming every needed block
//   vector into a shared-memory ring with cp.async.bulk (mbarrier complete_tx),
//   eight consumer warps accumulating in registers (fp32) -> HBM-bound.
//   Fallback (fp64 pools, unaligned pools): register-only CTA per item.
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include "kernels.h"
#include "vec_io.cuh"

namespace kvf {

// ---------------------------------------------------------------------------
// level statistics + ordered member segments
// ---------------------------------------------------------------------------
namespace {
constexpr int LS_THREADS = 512;
constexpr int LS_WARPS = LS_THREADS / 32;

// deterministic block-exclusive scan of one int per thread; returns the
// exclusive prefix, writes the block total to *total
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int w = 0; w < LS_WARPS; ++w) {
      const int t = wsum[w];
      wsum[w] = run;
      run += t;
    }
    *total = run;
  }
  __syncthreads();
  const int r = wsum[warp] + x - v;
  __syncthreads();
  return r;
}
}  // namespace

__global__ void __launch_bounds__(LS_THREADS)
level_stats_kernel(int64_t u0, int64_t NB, int64_t n_total, const uint8_t* __restrict__ fusable,
                   const uint8_t* __restrict__ alive, const int32_t* __restrict__ absorber,
                   const int32_t* __restrict__ merges, int nm,
                   const int32_t* __restrict__ tile_off, int nt,
                   const double* __restrict__ partials, double* stats, int32_t* ws) {
  __shared__ double red[32];
  __shared__ int wsum[LS_WARPS];
  __shared__ int tot_c, tot_f, run_c, lbase, seg_base;
  LevelWs W(ws, n_total);
  const int m = blockIdx.x;
  const int64_t ul = blockIdx.y, u = u0 + ul;
  const int64_t gb = u * NB;
  const int lb = merges[3 * m], mid = merges[3 * m + 1], re = merges[3 * m + 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  // pass A: counters + member counts per absorber
  double nl = 0, nr = 0, nf = 0;
  for (int i = lb + threadIdx.x; i < mid; i += blockDim.x)
    nl += (alive[gb + i] && fusable[gb + i]) ? 1.0 : 0.0;
  for (int j = mid + threadIdx.x; j < re; j += blockDim.x) {
    const bool al = alive[gb + j];
    nr += (al && fusable[gb + j]) ? 1.0 : 0.0;
    const int32_t a = absorber[gb + j];
    if (al && a != kNone) {
      nf += 1.0;
      atomicAdd(&W.mcnt[gb + a], 1);
    }
  }
  nl = block_sum(nl, red);
  nr = block_sum(nr, red);
  nf = block_sum(nf, red);
  if (threadIdx.x == 0) {
    seg_base = nf > 0 ? atomicAdd(W.cursor, (int)nf) : 0;
    run_c = 0;
  }
  __syncthreads();

  // pass B: member segments + absorber list, ascending over the left range
  if (nf > 0) {
    for (int c0 = lb; c0 < mid; c0 += blockDim.x) {
      const int i = c0 + threadIdx.x;
      const int c = i < mid ? W.mcnt[gb + i] : 0;
      const int oc = block_excl_scan(c, wsum, &tot_c);
      const int of = block_excl_scan(c > 0 ? 1 : 0, wsum, &tot_f);
      if (threadIdx.x == 0) lbase = tot_f > 0 ? atomicAdd(W.count, tot_f) : 0;
      __syncthreads();
      if (c > 0) {
        W.mstart[gb + i] = seg_base + run_c + oc;
        W.list[lbase + of] = (int32_t)(gb + i);
      }
      __syncthreads();
      if (threadIdx.x == 0) run_c += tot_c;
      __syncthreads();
    }
    // pass C: ordered scatter of members (warps take turns -> ascending j)
    for (int c0 = mid; c0 < re; c0 += blockDim.x) {
      const int j = c0 + threadIdx.x;
      int key = -1 - lane;
      if (j < re) {
        const int32_t a = absorber[gb + j];
        if (a != kNone && alive[gb + j]) key = a;
      }
      if (!__syncthreads_or(key >= 0)) continue;
      for (int w = 0; w < LS_WARPS; ++w) {
        if (warp == w) {
          const unsigned grp = __match_any_sync(0xffffffffu, key);
          if (key >= 0) {
            const int leader = __ffs(grp) - 1;
            int b = 0;
            if (lane == leader) {
              b = W.mfill[gb + key];
              W.mfill[gb + key] = b + __popc(grp);
            }
            b = __shfl_sync(grp, b, leader);
            W.members[W.mstart[gb + key] + b + __popc(grp & ((1u << lane) - 1u))] = j;
          }
        }
        __syncthreads();
      }
    }
  }

  // similarity moments of this merge's tiles (fixed order => deterministic)
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
  c = block_sum(c, red);
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  __shared__ double smn[LS_WARPS], smx[LS_WARPS];
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    smn[warp] = mn;
    smx[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < LS_WARPS; ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    double* o = stats + (ul * nm + m) * 8;
    o[0] = nl; o[1] = nr; o[2] = nf; o[3] = c; o[4] = s1; o[5] = s2;
    o[6] = c > 0 ? mn : 0.0;
    o[7] = c > 0 ? mx : 0.0;
  }
}

// ---------------------------------------------------------------------------
// level statistics for few, large merges (the top levels: one CTA per merge
// walked 262,144 blocks serially at cfg5, 10 ms for the top level). C CTAs per
// (merge, unit) stride over the merge's range; the same outputs in five launches:
//   ls_count    counters (integer-valued doubles, exact in any order) + member counts
//   ls_segments absorber list and member segment bases (ascending inside a CTA step)
//   ls_scatter  members appended with an atomic fill; moments of the CTA's share of
//               the merge's tile partials, written over the share's first slot
//   ls_sort     each absorber's member segment sorted ascending (the deterministic
//               summation order of the one-CTA path)
//   ls_moments  the C shares reduced in order
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ void merge_range(const int32_t* merges, int m, int& lb, int& mid, int& re) {
  lb = merges[3 * m];
  mid = merges[3 * m + 1];
  re = merges[3 * m + 2];
}
// [a, b) = share c of C of the merge's partial slots [t0, t1)
__device__ __forceinline__ void slot_share(int t0, int t1, int c, int C, int& a, int& b) {
  const int64_t n = t1 - t0;
  a = t0 + (int)(n * c / C);
  b = t0 + (int)(n * (c + 1) / C);
}
}  // namespace

__global__ void __launch_bounds__(LS_THREADS)
ls_count_kernel(int64_t u0, int64_t NB, const uint8_t* __restrict__ fusable,
                const uint8_t* __restrict__ alive, const int32_t* __restrict__ absorber,
                const int32_t* __restrict__ merges, int nm, double* stats, int32_t* ws,
                int64_t n_total) {
  __shared__ double red[32];
  LevelWs W(ws, n_total);
  const int C = gridDim.x, c = blockIdx.x, m = blockIdx.y;
  const int64_t ul = blockIdx.z, gb = (u0 + ul) * NB;
  int lb, mid, re;
  merge_range(merges, m, lb, mid, re);
  double nl = 0, nr = 0, nf = 0;
  for (int i = lb + c * LS_THREADS + threadIdx.x; i < re; i += C * LS_THREADS) {
    const bool al = alive[gb + i], fu = fusable[gb + i];
    if (i < mid) {
      nl += (al && fu) ? 1.0 : 0.0;
    } else {
      nr += (al && fu) ? 1.0 : 0.0;
      const int32_t a = absorber[gb + i];
      if (al && a != kNone) {
        nf += 1.0;
        atomicAdd(&W.mcnt[gb + a], 1);
      }
    }
  }
  nl = block_sum(nl, red);
  nr = block_sum(nr, red);
  nf = block_sum(nf, red);
  if (threadIdx.x == 0) {
    double* o = stats + (ul * nm + m) * 8;
    atomicAdd(o + 0, nl);
    atomicAdd(o + 1, nr);
    atomicAdd(o + 2, nf);
  }
}

__global__ void __launch_bounds__(LS_THREADS)
ls_segments_kernel(int64_t u0, int64_t NB, const int32_t* __restrict__ merges, int32_t* ws,
                   int64_t n_total) {
  __shared__ int wsum[LS_WARPS];
  __shared__ int tot_c, tot_f, cbase, lbase;
  LevelWs W(ws, n_total);
  const int C = gridDim.x, c = blockIdx.x, m = blockIdx.y;
  const int64_t gb = (u0 + blockIdx.z) * NB;
  int lb, mid, re;
  merge_range(merges, m, lb, mid, re);
  for (int c0 = lb + c * LS_THREADS; c0 < mid; c0 += C * LS_THREADS) {
    const int i = c0 + threadIdx.x;
    const int n = i < mid ? W.mcnt[gb + i] : 0;
    const int oc = block_excl_scan(n, wsum, &tot_c);
    const int of = block_excl_scan(n > 0 ? 1 : 0, wsum, &tot_f);
    if (tot_f == 0) continue;  // block-uniform
    if (threadIdx.x == 0) {
      cbase = atomicAdd(W.cursor, tot_c);
      lbase = atomicAdd(W.count, tot_f);
    }
    __syncthreads();
    if (n > 0) {
      W.mstart[gb + i] = cbase + oc;
      W.list[lbase + of] = (int32_t)(gb + i);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(LS_THREADS)
ls_scatter_kernel(int64_t u0, int64_t NB, const uint8_t* __restrict__ alive,
                  const int32_t* __restrict__ absorber, const int32_t* __restrict__ merges,
                  const int32_t* __restrict__ tile_off, int nt, double* partials, int32_t* ws,
                  int64_t n_total) {
  __shared__ double red[32];
  __shared__ double smn[LS_WARPS], smx[LS_WARPS];
  LevelWs W(ws, n_total);
  const int C = gridDim.x, c = blockIdx.x, m = blockIdx.y;
  const int64_t ul = blockIdx.z, gb = (u0 + ul) * NB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int lb, mid, re;
  merge_range(merges, m, lb, mid, re);
  for (int j = mid + c * LS_THREADS + threadIdx.x; j < re; j += C * LS_THREADS) {
    const int32_t a = absorber[gb + j];
    if (a != kNone && alive[gb + j]) {
      const int pos = atomicAdd(&W.mfill[gb + a], 1);
      W.members[W.mstart[gb + a] + pos] = j;
    }
  }
  // this CTA's share of the merge's tile partials (fixed range, fixed order)
  int a0, a1;
  slot_share(tile_off[m], tile_off[m + 1], c, C, a0, a1);
  double* pb = partials + ul * (int64_t)nt * 5;
  double cn = 0, s1 = 0, s2 = 0, mn = INFINITY, mx = -INFINITY;
  for (int tt = a0 + threadIdx.x; tt < a1; tt += blockDim.x) {
    const double* q = pb + (int64_t)tt * 5;
    cn += q[0];
    s1 += q[1];
    s2 += q[2];
    mn = fmin(mn, q[3]);
    mx = fmax(mx, q[4]);
  }
  cn = block_sum(cn, red);
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    smn[warp] = mn;
    smx[warp] = mx;
  }
  __syncthreads();  // every thread has read its share before the first slot is overwritten
  if (threadIdx.x == 0 && a1 > a0) {
    for (int w = 1; w < LS_WARPS; ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    double* o = pb + (int64_t)a0 * 5;
    o[0] = cn; o[1] = s1; o[2] = s2; o[3] = mn; o[4] = mx;
  }
}

__global__ void ls_sort_kernel(int32_t* ws, int64_t n_total) {
  LevelWs W(ws, n_total);
  const int n_items = *W.count;
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n_items; it += gridDim.x * blockDim.x) {
    const int64_t gid = W.list[it];
    int32_t* seg = W.members + W.mstart[gid];
    const int n = W.mcnt[gid];
    for (int x = 1; x < n; ++x) {  // insertion sort: segments hold a few members
      const int32_t v = seg[x];
      int y = x - 1;
      while (y >= 0 && seg[y] > v) {
        seg[y + 1] = seg[y];
        --y;
      }
      seg[y + 1] = v;
    }
  }
}

__global__ void ls_moments_kernel(const int32_t* __restrict__ tile_off, int nt, int nm, int C,
                                  const double* __restrict__ partials, double* stats) {
  const int m = blockIdx.x;
  const int64_t ul = blockIdx.y;
  if (threadIdx.x != 0) return;
  const double* pb = partials + ul * (int64_t)nt * 5;
  double cn = 0, s1 = 0, s2 = 0, mn = INFINITY, mx = -INFINITY;
  for (int c = 0; c < C; ++c) {
    int a0, a1;
    slot_share(tile_off[m], tile_off[m + 1], c, C, a0, a1);
    if (a1 <= a0) continue;
    const double* q = pb + (int64_t)a0 * 5;
    cn += q[0];
    s1 += q[1];
    s2 += q[2];
    mn = fmin(mn, q[3]);
    mx = fmax(mx, q[4]);
  }
  double* o = stats + (ul * nm + m) * 8;
  o[3] = cn; o[4] = s1; o[5] = s2;
  o[6] = cn > 0 ? mn : 0.0;
  o[7] = cn > 0 ? mx : 0.0;
}

cudaError_t launch_level_stats(int64_t u0, int64_t nU, int64_t NB, int64_t n_total,
                               const uint8_t* fusable, const uint8_t* alive,
                               const int32_t* absorber, const int32_t* merges, int nm,
                               const int32_t* tile_off, int nt, const double* partials,
                               double* stats, int32_t* level_ws, cudaStream_t s) {
  LevelWs W(level_ws, n_total);
  // count, cursor, merge item fetch counter
  cudaError_t e = cudaMemsetAsync(W.count, 0, 3 * sizeof(int32_t), s);
  if (e != cudaSuccess || nm == 0 || nU == 0) return e;
  // few, large merges (fewer CTAs than two waves, >= 8192 blocks per merge on average):
  // C CTAs per merge (KVF_LS_CHUNKED=0/1 forces the one-CTA / chunked path)
  const char* force = getenv("KVF_LS_CHUNKED");
  const int64_t per_merge = NB / nm;
  bool chunked = nm * nU < 2 * 148 && per_merge >= 8192;
  if (force) chunked = force[0] == '1';
  if (chunked) {
    int C = (int)std::max<int64_t>(1, std::min<int64_t>((2 * 148 + nm * nU - 1) / (nm * nU),
                                                         std::max<int64_t>(1, per_merge / 2048)));
    dim3 g3(C, nm, (unsigned)nU);
    e = cudaMemsetAsync(stats, 0, sizeof(double) * 8 * nm * nU, s);
    if (e != cudaSuccess) return e;
    double* part = const_cast<double*>(partials);
    ls_count_kernel<<<g3, LS_THREADS, 0, s>>>(u0, NB, fusable, alive, absorber, merges, nm, stats,
                                              level_ws, n_total);
    ls_segments_kernel<<<g3, LS_THREADS, 0, s>>>(u0, NB, merges, level_ws, n_total);
    ls_scatter_kernel<<<g3, LS_THREADS, 0, s>>>(u0, NB, alive, absorber, merges, tile_off, nt, part,
                                                level_ws, n_total);
    ls_sort_kernel<<<148, 256, 0, s>>>(level_ws, n_total);
    ls_moments_kernel<<<dim3(nm, (unsigned)nU), 32, 0, s>>>(tile_off, nt, nm, C, part, stats);
    return cudaGetLastError();
  }
  dim3 grid(nm, (unsigned)nU);
  level_stats_kernel<<<grid, LS_THREADS, 0, s>>>(u0, NB, n_total, fusable, alive, absorber,
                                                 merges, nm, tile_off, nt, partials, stats,
                                                 level_ws);
  return cudaGetLastError();
}

// Item selection of the merge kernels: which = 3 merges K and V (items 2a, 2a+1
// = K, V of absorber a), 1 = K only, 2 = V only (the exact-decision mode merges
// the keys separately, kern_exact.cu)
struct ItemSel {
  int which;
  __device__ __forceinline__ int64_t n(int64_t count) const { return which == 3 ? 2 * count : count; }
  __device__ __forceinline__ bool is_v(int64_t it) const { return which == 3 ? (it & 1) : which == 2; }
  __device__ __forceinline__ int64_t idx(int64_t it) const { return which == 3 ? (it >> 1) : it; }
};

// ---------------------------------------------------------------------------
// K4 main path: bulk-copy ring + register accumulation
// ---------------------------------------------------------------------------
namespace {
constexpr int MG_CONSUMERS = 256;
constexpr int MG_THREADS = MG_CONSUMERS + 32;
constexpr int MG_MAX_BUF = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ float consumer_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, cw = (threadIdx.x >> 5) - 1;
  v = warp_sum(v);
  if (lane == 0) red[cw] = v;
  asm volatile("bar.sync 1, %0;" ::"n"(MG_CONSUMERS) : "memory");
  float t = 0.f;
#pragma unroll
  for (int w = 0; w < MG_CONSUMERS / 32; ++w) t += red[w];
  asm volatile("bar.sync 1, %0;" ::"n"(MG_CONSUMERS) : "memory");
  return t;
}
}  // namespace

// Per-slot metadata handed from the producer to the consumers with the data
struct SlotMeta {
  float inv;   // 1 / stored norm of the vector in the slot (0 for zero vectors)
  float home;  // item: original norm of the absorber's home slot
  int32_t gid; // item: global absorber id u * NB + l
  int32_t flags;  // bit0: last slot of the item, bit1: V tensor, bit2: end of the work
  int32_t sh;  // exact mode, keys: shadow row of this vector or -1
  int32_t ash; // exact mode, keys: the absorber's shadow row (-1: none yet)
  int32_t half;  // 0: the slot holds a pool vector; 1 / 2: first / second half of the
                 // fp32 shadow row sh (ring-fed shadow rows); -1: consumers read row sh
};

// Exact-decision mode (kern_exact.cu): fused key directions live as fp32 shadow
// rows; members with a row are read from it (unit vectors, inv = 1) and every key
// absorber's new unit direction is written to its row (allocated on first fusion)
struct ExactArgs {
  float* shadow;     // [cap][r] or null (mode off)
  int64_t cap;
  int32_t* sidx;     // [U][NB]
  int32_t* scount;   // rows taken (can exceed cap: overflow is reported)
  int write_rows = 1;  // 0 at the tree's last level: rows are read, never written again
};

template <typename T, int EPT>
__global__ void __launch_bounds__(MG_THREADS, 2)
merge_tma_kernel(T* __restrict__ pool_k, T* __restrict__ pool_v, Geom g, float* __restrict__ knorm,
                 float* __restrict__ vnorm, const float* __restrict__ oknorm,
                 const float* __restrict__ ovnorm, int32_t* ws, int64_t n_total, int nbuf,
                 int slot_bytes, ItemSel sel, ExactArgs ex, int ring_shadow) {
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int CPT = EPT / VEC;  // 16-byte chunks per consumer thread
  extern __shared__ __align__(128) uint8_t msm[];
  uint8_t* ring = msm;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)nbuf * slot_bytes);
  uint64_t* empty = full + MG_MAX_BUF;
  SlotMeta* meta = reinterpret_cast<SlotMeta*>(empty + MG_MAX_BUF);
  // per-item reductions, double-buffered by item parity so each needs one barrier:
  // red[2][8] norm of the member sum, red2[2][8] stored norm (written by consumer 0 of
  // the next item, after that item's barrier), slot_bc[2] the absorber's shadow row
  float* red = reinterpret_cast<float*>(meta + MG_MAX_BUF);
  float* red2 = red + 16;
  int* slot_bc = reinterpret_cast<int*>(red2 + 16);
  const LevelWs W(ws, n_total);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = g.r();
  const uint32_t vbytes = (uint32_t)(r * (int64_t)sizeof(T));
  const int n_items = (int)sel.n(*W.count);

  if (threadIdx.x == 0) {
    for (int s = 0; s < nbuf; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MG_CONSUMERS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // producer warp: item headers, member ids and their norms are loaded by the
    // whole warp one item ahead, so the copy issue never waits on them
    struct Item {
      int32_t gid, n, id;  // id / inv / sh: lane k holds vector k of the item (k <= 31)
      float inv, home;
      int32_t sh;
      bool valid;
    };
    auto load_item = [&](int it) {
      Item x;
      x.valid = it < n_items;
      x.gid = 0;
      x.n = 0;
      x.id = 0;
      x.inv = 0.f;
      x.home = 0.f;
      x.sh = -1;
      if (!x.valid) return x;
      const bool is_v = sel.is_v(it);
      const float* norm = is_v ? vnorm : knorm;
      x.gid = W.list[sel.idx(it)];
      x.n = W.mcnt[x.gid];
      const int64_t gb = (x.gid / g.NB) * g.NB;
      const int s0 = W.mstart[x.gid];
      x.home = (is_v ? ovnorm : oknorm)[x.gid];
      if (lane <= x.n) {
        x.id = lane == 0 ? (int32_t)(x.gid - gb) : W.members[s0 + lane - 1];
        const float nv = norm[gb + x.id];
        x.inv = nv > 0.f ? 1.f / nv : 0.f;
        if (ex.shadow && !is_v) {
          x.sh = ex.sidx[gb + x.id];
          if (x.sh >= 0) x.inv = 1.f;  // shadow rows are unit directions
        }
      }
      return x;
    };
    // items are fetched dynamically (item sizes vary with the member count); every
    // producer's last fetch is the one past the end, and the numerically last of
    // those resets the counter for the next launch
    auto fetch = [&]() {
      int v = 0;
      if (lane == 0) {
        v = atomicAdd(W.fetch, 1);
        if (v == n_items + (int)gridDim.x - 1) atomicExch(W.fetch, 0);
      }
      return __shfl_sync(0xffffffffu, v, 0);
    };
    // one slot: wait for it, publish the metadata, start its copy (or just arrive)
    auto put = [&](uint32_t qq, const SlotMeta& mt, const void* src, uint32_t bytes, bool rows) {
      const int s = qq % nbuf;
      mbar_wait(&empty[s], ((qq / nbuf) & 1) ^ 1);
      meta[s] = mt;
      if (src == nullptr) {
        mbar_arrive(&full[s]);
        return;
      }
      mbar_expect_tx(&full[s], bytes);  // release: meta visible after the wait
      uint8_t* dst = ring + (size_t)s * slot_bytes;
      if (!rows) {
        bulk_g2s(dst, src, bytes, &full[s]);
      } else {  // per-head pool vector: one bulk copy per token row
        const uint32_t segb = (uint32_t)(g.d * sizeof(T));
        for (int tk = 0; tk < g.t; ++tk)
          bulk_g2s(dst + tk * segb, reinterpret_cast<const T*>(src) + (int64_t)tk * g.h * g.d, segb,
                   &full[s]);
      }
    };
    uint32_t q = 0;
    int it = fetch();
    Item cur = load_item(it);
    while (cur.valid) {
      const int it_next = fetch();
      const Item nxt = load_item(it_next);
      const bool is_v = sel.is_v(it);
      const T* pool = is_v ? pool_v : pool_k;
      const int64_t u = cur.gid / g.NB;
      const int64_t gb = u * g.NB;
      const int s0 = W.mstart[cur.gid];
      const int32_t ash = __shfl_sync(0xffffffffu, cur.sh, 0);
      for (int v = 0; v <= cur.n; ++v) {
        int32_t id, sh;
        float inv;
        if (v < 32) {
          id = __shfl_sync(0xffffffffu, cur.id, v);
          inv = __shfl_sync(0xffffffffu, cur.inv, v);
          sh = __shfl_sync(0xffffffffu, cur.sh, v);
        } else {  // large groups: beyond the warp-wide prefetch
          id = W.members[s0 + v - 1];
          const float nv = (is_v ? vnorm : knorm)[gb + id];
          inv = nv > 0.f ? 1.f / nv : 0.f;
          sh = (ex.shadow && !is_v) ? ex.sidx[gb + id] : -1;
          if (sh >= 0) inv = 1.f;
        }
        SlotMeta mt;
        mt.inv = inv;
        mt.home = cur.home;
        mt.gid = cur.gid;
        mt.flags = (v == cur.n ? 1 : 0) | (is_v ? 2 : 0);
        mt.sh = sh;
        mt.ash = ash;
        if (sh >= 0 && ring_shadow) {  // fp32 shadow row: two slots of r / 2 floats
          const float* row = ex.shadow + (int64_t)sh * r;
          const uint32_t hb = (uint32_t)(r / 2 * sizeof(float));
          if (lane == 0) {
            SlotMeta m1 = mt;
            m1.flags &= ~1;
            m1.half = 1;
            put(q, m1, row, hb, false);
            mt.half = 2;
            put(q + 1, mt, row + r / 2, hb, false);
          }
          q += 2;
        } else {
          mt.half = sh >= 0 ? -1 : 0;
          if (lane == 0)
            put(q, mt, sh >= 0 ? nullptr : (const void*)(pool + g.base(u, id)), vbytes, g.head_mode != 0);
          q += 1;
        }
      }
      cur = nxt;
      it = it_next;
    }
    if (lane == 0) {  // end of the work for this CTA's consumers
      SlotMeta mt;
      mt.flags = 4;
      mt.half = 0;
      mt.sh = -1;
      put(q, mt, nullptr, 0, false);
    }
    return;
  }
  // consumers: everything per vector comes from the slot (data + meta)
  const int ct = threadIdx.x - 32;
  const int nch = (int)(r / VEC);
  const int nch_h = nch / 2;  // 16-byte chunks of T in the first half of a vector
  uint32_t q = 0;
  float acc[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) acc[e] = 0.f;
  const int cw = ct >> 5;
  int par = 0;
  float* prev_norm = nullptr;  // consumer 0: where the previous item's stored norm goes
  auto finish_prev = [&](int pp) {  // after a barrier: every warp's partial is in red2[pp]
    if (ct == 0 && prev_norm) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < MG_CONSUMERS / 32; ++w) t += red2[pp * 8 + w];
      *prev_norm = sqrtf(t);
    }
  };
  for (;;) {
    SlotMeta mt;
    bool done = false;
    for (;;) {
      const int s = q % nbuf;
      mbar_wait(&full[s], (q / nbuf) & 1);
      mt = meta[s];
      if (mt.flags & 4) {
        done = true;
        break;
      }
      const T* sp = reinterpret_cast<const T*>(ring + (size_t)s * slot_bytes);
      if (mt.half > 0) {  // exact mode: half of a fused member's fp32 unit direction
        const float* hs = reinterpret_cast<const float*>(ring + (size_t)s * slot_bytes);
        const int c_lo = mt.half == 1 ? 0 : nch_h, c_hi = mt.half == 1 ? nch_h : nch;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          const int c = ct + k * MG_CONSUMERS;
          if (c >= c_lo && c < c_hi) {
#pragma unroll
            for (int e4 = 0; e4 < VEC; e4 += 4) {
              const float4 f = *reinterpret_cast<const float4*>(hs + (c - c_lo) * VEC + e4);
              acc[k * VEC + e4 + 0] += f.x;
              acc[k * VEC + e4 + 1] += f.y;
              acc[k * VEC + e4 + 2] += f.z;
              acc[k * VEC + e4 + 3] += f.w;
            }
          }
        }
      } else if (mt.sh >= 0) {  // exact mode: fused member, its fp32 unit direction
        const float* row = ex.shadow + (int64_t)mt.sh * r;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          const int c = ct + k * MG_CONSUMERS;
          if (c < nch) {
#pragma unroll
            for (int e4 = 0; e4 < VEC; e4 += 4) {
              const float4 f = __ldg(reinterpret_cast<const float4*>(row + c * VEC + e4));
              acc[k * VEC + e4 + 0] += f.x;
              acc[k * VEC + e4 + 1] += f.y;
              acc[k * VEC + e4 + 2] += f.z;
              acc[k * VEC + e4 + 3] += f.w;
            }
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          const int c = ct + k * MG_CONSUMERS;
          if (c < nch) {
            float x[VEC];
            VecIO<T, VEC>::load(sp + c * VEC, x);
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[k * VEC + e] = fmaf(x[e], mt.inv, acc[k * VEC + e]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      ++q;
      if (mt.flags & 1) break;
    }
    if (done) {
      asm volatile("bar.sync 1, %0;" ::"n"(MG_CONSUMERS) : "memory");
      finish_prev(par ^ 1);
      break;
    }
    const bool is_v = mt.flags & 2;
    T* pool = is_v ? pool_v : pool_k;
    float* norm = is_v ? vnorm : knorm;
    const int64_t u = mt.gid / g.NB;
    const int32_t l = (int32_t)(mt.gid % g.NB);
    // exact mode, keys: the absorber's shadow row (taken on its first fusion); published
    // through the norm reduction's barriers (every consumer reads it before the next
    // item's reduction, the only place it is written again)
    const bool want_row = ex.shadow && !is_v && ex.write_rows;
    if (want_row && ct == 0) {
      int sl = mt.ash;
      if (sl < 0) {
        sl = atomicAdd(ex.scount, 1);
        if (sl < ex.cap) ex.sidx[mt.gid] = sl; else sl = -1;
      }
      slot_bc[par] = sl;
    }
    float ss = 0.f;
#pragma unroll
    for (int e = 0; e < EPT; ++e) ss = fmaf(acc[e], acc[e], ss);
    ss = warp_sum(ss);
    if (lane == 0) red[par * 8 + cw] = ss;
    asm volatile("bar.sync 1, %0;" ::"n"(MG_CONSUMERS) : "memory");
    finish_prev(par ^ 1);
    float nsum = 0.f;
#pragma unroll
    for (int w = 0; w < MG_CONSUMERS / 32; ++w) nsum += red[par * 8 + w];
    const float nrm = sqrtf(nsum);
    const float sc = nrm > 0.f ? (mt.home > 0.f ? mt.home : 1.f) / nrm : 0.f;
    T* xl = pool + g.base(u, l);
    float* srow = nullptr;
    const float inv_n = nrm > 0.f ? 1.f / nrm : 0.f;
    if (want_row) {
      const int sl = slot_bc[par];
      if (sl >= 0) srow = ex.shadow + (int64_t)sl * r;
    }
    float rs = 0.f;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int c = ct + k * MG_CONSUMERS;
      if (c < nch) {
        float y[VEC], rd[VEC];
        if (srow) {
#pragma unroll
          for (int e4 = 0; e4 < VEC; e4 += 4)
            *reinterpret_cast<float4*>(srow + c * VEC + e4) =
                make_float4(acc[k * VEC + e4] * inv_n, acc[k * VEC + e4 + 1] * inv_n,
                            acc[k * VEC + e4 + 2] * inv_n, acc[k * VEC + e4 + 3] * inv_n);
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = acc[k * VEC + e] * sc;
        VecIO<T, VEC>::store(xl + g.off32(c * VEC), y, rd);
#pragma unroll
        for (int e = 0; e < VEC; ++e) rs = fmaf(rd[e], rd[e], rs);
      }
    }
#pragma unroll
    for (int e = 0; e < EPT; ++e) acc[e] = 0.f;
    rs = warp_sum(rs);
    if (lane == 0) red2[par * 8 + cw] = rs;
    prev_norm = norm + mt.gid;
    par ^= 1;
  }
}

// ---------------------------------------------------------------------------
// K4 fallback: one CTA per (absorber, K|V), register accumulation, members
// read from the ordered segments (fp64 pools, unaligned pools, large r)
// ---------------------------------------------------------------------------
template <typename T, int VEC>
__global__ void __launch_bounds__(512)
merge_reg_kernel(T* __restrict__ pool_k, T* __restrict__ pool_v, Geom g,
                 typename AccOf<T>::type* __restrict__ knorm,
                 typename AccOf<T>::type* __restrict__ vnorm,
                 const typename AccOf<T>::type* __restrict__ oknorm,
                 const typename AccOf<T>::type* __restrict__ ovnorm, int32_t* ws,
                 int64_t n_total, ItemSel sel) {
  using A = typename AccOf<T>::type;
  constexpr int MAXQ = 32 / VEC;
  __shared__ A red[32];
  const LevelWs W(ws, n_total);
  const int tid = threadIdx.x, bd = blockDim.x;
  const bool is_v = sel.which == 3 ? blockIdx.y == 1 : sel.which == 2;
  T* pool = is_v ? pool_v : pool_k;
  A* norm = is_v ? vnorm : knorm;
  const A* onorm = is_v ? ovnorm : oknorm;
  const int64_t nch = g.r() / VEC;
  const int n_items = *W.count;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int64_t gid = W.list[it];
    const int64_t u = gid / g.NB;
    const int64_t gb = u * g.NB;
    const int32_t l = (int32_t)(gid % g.NB);
    const int n = W.mcnt[gid], s0 = W.mstart[gid];
    A acc[MAXQ][VEC];
#pragma unroll
    for (int q = 0; q < MAXQ; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[q][e] = A(0);
    for (int v = 0; v <= n; ++v) {
      const int32_t id = v == 0 ? l : W.members[s0 + v - 1];
      const A nv = norm[gb + id];
      const A inv = nv > A(0) ? A(1) / nv : A(0);
      const T* x = pool + g.base(u, id);
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int64_t c = tid + (int64_t)q * bd;
        if (c < nch) {
          A y[VEC];
          VecIO<T, VEC>::load(x + g.off(c * VEC), y);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[q][e] += y[e] * inv;
        }
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
        A y[VEC], rd[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = acc[q][e] * sc;
        VecIO<T, VEC>::store(xl + g.off(c * VEC), y, rd);
#pragma unroll
        for (int e = 0; e < VEC; ++e) rs += rd[e] * rd[e];
      }
    }
    const A nn = sqrt(block_sum(rs, red));
    if (tid == 0) norm[gid] = nn;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K4 for short vectors (per-head units, r * sizeof(T) <= 4 KB): one warp per
// (absorber, K|V) item, CPL 16-byte chunks per lane in registers, warp-tree
// norms. Many items in flight per SM instead of one block-wide reduction per
// 4 KB vector.
// ---------------------------------------------------------------------------
template <typename T, int VEC, int CPL>
__global__ void __launch_bounds__(256, 2)
merge_warp_kernel(T* __restrict__ pool_k, T* __restrict__ pool_v, Geom g,
                  float* __restrict__ knorm, float* __restrict__ vnorm,
                  const float* __restrict__ oknorm, const float* __restrict__ ovnorm,
                  int32_t* ws, int64_t n_total, ItemSel sel) {
  const LevelWs W(ws, n_total);
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_items = sel.n(*W.count);
  for (int64_t it = warp; it < n_items; it += nwarps) {
    const bool is_v = sel.is_v(it);
    T* pool = is_v ? pool_v : pool_k;
    float* norm = is_v ? vnorm : knorm;
    const int64_t gid = W.list[sel.idx(it)];
    const int64_t u = gid / g.NB;
    const int64_t gb = u * g.NB;
    const int32_t l = (int32_t)(gid % g.NB);
    const int n = W.mcnt[gid], s0 = W.mstart[gid];
    // lane k holds vector k's id and 1/norm (k = 0: the absorber itself)
    int32_t id_l = l;
    float inv_l = 0.f;
    if (lane <= n) {
      if (lane > 0) id_l = W.members[s0 + lane - 1];
      const float nv = norm[gb + id_l];
      inv_l = nv > 0.f ? 1.f / nv : 0.f;
    }
    float acc[CPL][VEC];
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[q][e] = 0.f;
    for (int v = 0; v <= n; ++v) {
      int32_t id;
      float inv;
      if (v < 32) {
        id = __shfl_sync(0xffffffffu, id_l, v);
        inv = __shfl_sync(0xffffffffu, inv_l, v);
      } else {  // groups beyond one warp of members
        id = W.members[s0 + v - 1];
        const float nv = norm[gb + id];
        inv = nv > 0.f ? 1.f / nv : 0.f;
      }
      const T* x = pool + g.base(u, id);
      uint4 raw[CPL];  // 16-byte chunks kept packed until use (register budget)
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        raw[q] = __ldg(reinterpret_cast<const uint4*>(x + g.off((int64_t)(q * 32 + lane) * VEC)));
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        float y[VEC];
        VecIO<T, VEC>::load(reinterpret_cast<const T*>(&raw[q]), y);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[q][e] = fmaf(y[e], inv, acc[q][e]);
      }
    }
    float ss = 0.f;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) ss = fmaf(acc[q][e], acc[q][e], ss);
    const float nrm = sqrtf(warp_sum(ss));
    const float home = (is_v ? ovnorm : oknorm)[gid];
    const float sc = nrm > 0.f ? (home > 0.f ? home : 1.f) / nrm : 0.f;
    T* xl = pool + g.base(u, l);
    float rs = 0.f;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      float yv[VEC], rd[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) yv[e] = acc[q][e] * sc;
      VecIO<T, VEC>::store(xl + g.off((int64_t)(q * 32 + lane) * VEC), yv, rd);
#pragma unroll
      for (int e = 0; e < VEC; ++e) rs = fmaf(rd[e], rd[e], rs);
    }
    rs = warp_sum(rs);
    if (lane == 0) norm[gid] = sqrtf(rs);
  }
}


// ---------------------------------------------------------------------------
// K4 for short vectors (per-head units, bf16): warp per item with a per-warp
// shared-memory ring. The item loop of merge_warp_kernel keeps one vector in
// flight per warp (its registers hold the accumulators); here NS - 1 member
// vectors stream into the ring by bulk copies (one per token row, issued by t
// lanes in parallel) while the warp accumulates the current one, running
// across item boundaries. Slot metadata (1/norm, item id, last flag) travels
// with the slot, so the consuming side never looks an item up.
// ---------------------------------------------------------------------------
struct RingSlotMeta {
  float inv, home;
  int32_t gid, flags;  // flags: bit0 last slot of the item, bit1 V tensor
  int32_t sh, ash;     // exact mode, keys: the vector's / the absorber's shadow row (-1: none)
  int32_t half;        // exact mode: 1 / 2 = first / second half of the fp32 shadow row sh
                       // in the slot (ring-fed), -1 = read row sh from global, 0 = pool vector
};
template <int CPL, int NS>
__global__ void __launch_bounds__(256, 2)
merge_ring_kernel(__nv_bfloat16* __restrict__ pool_k, __nv_bfloat16* __restrict__ pool_v, Geom g,
                  float* __restrict__ knorm, float* __restrict__ vnorm,
                  const float* __restrict__ oknorm, const float* __restrict__ ovnorm,
                  int32_t* ws, int64_t n_total, ItemSel sel, ExactArgs ex, int ring_shadow) {
  constexpr int VB = CPL * 512;  // vector bytes (32 lanes x CPL x 16 B)
  extern __shared__ __align__(128) uint8_t rsm[];
  const LevelWs W(ws, n_total);
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = rsm + (size_t)wl * NS * VB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rsm + (size_t)(blockDim.x >> 5) * NS * VB) + wl * NS;
  RingSlotMeta* smeta = reinterpret_cast<RingSlotMeta*>(
                            reinterpret_cast<uint64_t*>(rsm + (size_t)(blockDim.x >> 5) * NS * VB) +
                            (blockDim.x >> 5) * NS) + wl * NS;
  if (lane == 0)
    for (int q = 0; q < NS; ++q) mbar_init(&bars[q], 1);
  __syncwarp();
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_items = sel.n(*W.count);
  const uint32_t segb = (uint32_t)(g.d * 2);
  const int64_t rstride = (int64_t)g.h * g.d;  // elements between token rows

  // ---- issue side: item it_i, vector v_i; lane k holds vector k's id and 1/norm ----
  int64_t it_i = gw;
  int v_i = 0, n_i = 0, s0_i = 0;
  int64_t gid_i = 0;
  int32_t id_l = 0, sh_l = -1, ash_i = -1;
  float inv_l = 0.f, home_i = 0.f;
  auto load_item = [&]() {  // all lanes
    if (it_i >= n_items) return;
    const bool is_v = sel.is_v(it_i);
    const float* norm = is_v ? vnorm : knorm;
    gid_i = W.list[sel.idx(it_i)];
    n_i = W.mcnt[gid_i];
    s0_i = W.mstart[gid_i];
    home_i = (is_v ? ovnorm : oknorm)[gid_i];
    const int64_t gb = (gid_i / g.NB) * g.NB;
    id_l = (int32_t)(gid_i - gb);
    inv_l = 0.f;
    sh_l = -1;
    if (lane <= n_i) {
      if (lane > 0) id_l = W.members[s0_i + lane - 1];
      const float nv = norm[gb + id_l];
      inv_l = nv > 0.f ? 1.f / nv : 0.f;
      if (ex.shadow && !is_v) {
        sh_l = ex.sidx[gb + id_l];
        if (sh_l >= 0) inv_l = 1.f;  // shadow rows are unit directions
      }
    }
    ash_i = __shfl_sync(0xffffffffu, sh_l, 0);
  };
  uint32_t q_i = 0, q_c = 0;
  auto issue = [&]() {  // all lanes
    if (it_i >= n_items) return;
    const bool is_v = sel.is_v(it_i);
    int32_t id, sh;
    float inv;
    if (v_i < 32) {
      id = __shfl_sync(0xffffffffu, id_l, v_i);
      inv = __shfl_sync(0xffffffffu, inv_l, v_i);
      sh = __shfl_sync(0xffffffffu, sh_l, v_i);
    } else {  // groups beyond one warp of members
      const int64_t gb = (gid_i / g.NB) * g.NB;
      id = W.members[s0_i + v_i - 1];
      const float nv = (is_v ? vnorm : knorm)[gb + id];
      inv = nv > 0.f ? 1.f / nv : 0.f;
      sh = (ex.shadow && !is_v) ? ex.sidx[gb + id] : -1;
      if (sh >= 0) inv = 1.f;
    }
    // the warp consumes slot q_c while issuing: a vector may only take slots the consumer
    // has released (q_i + need - q_c <= NS); a shadow row needing two waits a round
    if (q_i + ((sh >= 0 && ring_shadow) ? 2u : 1u) - q_c > (uint32_t)NS) return;
    const int s = q_i % NS;
    const int64_t u = gid_i / g.NB;
    if (sh >= 0 && ring_shadow) {
      // fp32 shadow row (2 * VB bytes): two slots of VB bytes, one bulk copy each
      if (lane == 0) {
        const char* row = reinterpret_cast<const char*>(ex.shadow + (int64_t)sh * g.r());
        for (int hf = 0; hf < 2; ++hf) {
          const int sl = (q_i + hf) % NS;
          RingSlotMeta m;
          m.inv = inv;
          m.home = home_i;
          m.gid = (int32_t)gid_i;
          m.flags = (hf == 1 && v_i == n_i ? 1 : 0) | (is_v ? 2 : 0);
          m.sh = sh;
          m.ash = ash_i;
          m.half = 1 + hf;
          smeta[sl] = m;
          mbar_expect_tx(&bars[sl], (uint32_t)VB);
          bulk_g2s(ring + (size_t)sl * VB, row + (size_t)hf * VB, (uint32_t)VB, &bars[sl]);
        }
      }
      __syncwarp();
      q_i += 2;
    } else {
      if (lane == 0) {
        RingSlotMeta m;
        m.inv = inv;
        m.home = home_i;
        m.gid = (int32_t)gid_i;
        m.flags = (v_i == n_i ? 1 : 0) | (is_v ? 2 : 0);
        m.sh = sh;
        m.ash = ash_i;
        m.half = sh >= 0 ? -1 : 0;
        smeta[s] = m;
        if (sh >= 0)
          mbar_arrive(&bars[s]);  // shadow row: the consumer reads it from global memory
        else
          mbar_expect_tx(&bars[s], (uint32_t)VB);  // release: slot meta visible after the wait
      }
      __syncwarp();
      if (sh < 0 && lane < g.t) {
        const __nv_bfloat16* src = (is_v ? pool_v : pool_k) + g.base(u, id) + lane * rstride;
        bulk_g2s(ring + (size_t)s * VB + lane * segb, src, segb, &bars[s]);
      }
      ++q_i;
    }
    if (++v_i > n_i) {
      v_i = 0;
      it_i += nw;
      load_item();
    }
  };

  load_item();
  for (int k = 0; k < NS - 1; ++k) issue();
  float acc[CPL][8];
#pragma unroll
  for (int q = 0; q < CPL; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[q][e] = 0.f;
  for (int64_t it = gw; it < n_items;) {
    issue();
    const int s = q_c % NS;
    mbar_wait(&bars[s], (q_c / NS) & 1);
    const RingSlotMeta m = smeta[s];
    const uint4* sp = reinterpret_cast<const uint4*>(ring + (size_t)s * VB);
    if (m.half > 0) {  // exact mode: half of a fused key member's fp32 unit direction
      const float* hs = reinterpret_cast<const float*>(ring + (size_t)s * VB);
      const int q0 = m.half == 1 ? 0 : CPL / 2;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        if (q < q0 || q >= q0 + CPL / 2) continue;  // static per unrolled q
        const float4 a = *reinterpret_cast<const float4*>(hs + ((q - q0) * 32 + lane) * 8);
        const float4 b = *reinterpret_cast<const float4*>(hs + ((q - q0) * 32 + lane) * 8 + 4);
        acc[q][0] += a.x; acc[q][1] += a.y; acc[q][2] += a.z; acc[q][3] += a.w;
        acc[q][4] += b.x; acc[q][5] += b.y; acc[q][6] += b.z; acc[q][7] += b.w;
      }
    } else if (m.sh >= 0) {  // exact mode: fused key member, its fp32 unit direction
      const float* row = ex.shadow + (int64_t)m.sh * g.r();
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(row + (q * 32 + lane) * 8));
        const float4 b = __ldg(reinterpret_cast<const float4*>(row + (q * 32 + lane) * 8 + 4));
        acc[q][0] += a.x; acc[q][1] += a.y; acc[q][2] += a.z; acc[q][3] += a.w;
        acc[q][4] += b.x; acc[q][5] += b.y; acc[q][6] += b.z; acc[q][7] += b.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const uint4 raw = sp[q * 32 + lane];
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(p2[e]);
          acc[q][2 * e] = fmaf(f.x, m.inv, acc[q][2 * e]);
          acc[q][2 * e + 1] = fmaf(f.y, m.inv, acc[q][2 * e + 1]);
        }
      }
    }
    __syncwarp();  // the slot may be refilled by the next issue
    ++q_c;
    if (!(m.flags & 1)) continue;
    // item complete: x_l <- home * unit(sum), stored norm of the written bf16 vector
    const bool is_v = m.flags & 2;
    __nv_bfloat16* pool = is_v ? pool_v : pool_k;
    float* norm = is_v ? vnorm : knorm;
    float ss = 0.f;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < 8; ++e) ss = fmaf(acc[q][e], acc[q][e], ss);
    const float nrm = sqrtf(warp_sum(ss));
    const float sc = nrm > 0.f ? (m.home > 0.f ? m.home : 1.f) / nrm : 0.f;
    const int64_t u = m.gid / g.NB;
    const int32_t l = (int32_t)(m.gid % g.NB);
    __nv_bfloat16* xl = pool + g.base(u, l);
    // exact mode, keys: the absorber's shadow row (taken on its first fusion)
    float* srow = nullptr;
    const float inv_n = nrm > 0.f ? 1.f / nrm : 0.f;
    if (ex.shadow && !is_v && ex.write_rows) {
      int sl = m.ash;
      if (sl < 0) {
        if (lane == 0) {
          sl = atomicAdd(ex.scount, 1);
          if (sl < ex.cap) ex.sidx[m.gid] = sl;
        }
        sl = __shfl_sync(0xffffffffu, sl, 0);
        if (sl >= ex.cap) sl = -1;
      }
      if (sl >= 0) srow = ex.shadow + (int64_t)sl * g.r();
    }
    float rs = 0.f;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      float yv[8], rd[8];
      if (srow) {
        float* d8 = srow + (q * 32 + lane) * 8;
        *reinterpret_cast<float4*>(d8) = make_float4(acc[q][0] * inv_n, acc[q][1] * inv_n,
                                                     acc[q][2] * inv_n, acc[q][3] * inv_n);
        *reinterpret_cast<float4*>(d8 + 4) = make_float4(acc[q][4] * inv_n, acc[q][5] * inv_n,
                                                         acc[q][6] * inv_n, acc[q][7] * inv_n);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) yv[e] = acc[q][e] * sc;
      VecIO<__nv_bfloat16, 8>::store(xl + g.off((int64_t)(q * 32 + lane) * 8), yv, rd);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        rs = fmaf(rd[e], rd[e], rs);
        acc[q][e] = 0.f;
      }
    }
    rs = warp_sum(rs);
    if (lane == 0) norm[m.gid] = sqrtf(rs);
    it += nw;
  }
}

namespace {
// Long vectors (r > 16384: folded units of 32-token blocks, MHA-sized heads): CTA per
// (absorber, K|V) in two passes over column chunks -- pass 1 the norm of the member
// sum, pass 2 the sum again, scaled and written -- so registers stay bounded for any r.
template <typename T, int VEC>
__global__ void __launch_bounds__(256)
merge_long_kernel(T* __restrict__ pool_k, T* __restrict__ pool_v, Geom g,
                  typename AccOf<T>::type* __restrict__ knorm,
                  typename AccOf<T>::type* __restrict__ vnorm,
                  const typename AccOf<T>::type* __restrict__ oknorm,
                  const typename AccOf<T>::type* __restrict__ ovnorm, int32_t* ws,
                  int64_t n_total, ItemSel sel) {
  using A = typename AccOf<T>::type;
  __shared__ A red[32];
  const LevelWs W(ws, n_total);
  const int tid = threadIdx.x, bd = blockDim.x;
  const int64_t nch = g.r() / VEC;
  const int64_t n_items = sel.n(*W.count);
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const bool is_v = sel.is_v(it);
    T* pool = is_v ? pool_v : pool_k;
    A* norm = is_v ? vnorm : knorm;
    const int64_t gid = W.list[sel.idx(it)];
    const int64_t u = gid / g.NB, gb = u * g.NB;
    const int32_t l = (int32_t)(gid % g.NB);
    const int n = W.mcnt[gid], s0 = W.mstart[gid];
    // every thread walks the same member order, so both passes sum identically
    auto member_sum = [&](int64_t c, A (&y)[VEC]) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) y[e] = A(0);
      for (int v = 0; v <= n; ++v) {
        const int32_t id = v == 0 ? l : W.members[s0 + v - 1];
        const A nv = norm[gb + id];
        const A inv = nv > A(0) ? A(1) / nv : A(0);
        A x[VEC];
        VecIO<T, VEC>::load(pool + g.base(u, id) + g.off(c * VEC), x);
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] += x[e] * inv;
      }
    };
    A ss = 0;
    for (int64_t c = tid; c < nch; c += bd) {
      A y[VEC];
      member_sum(c, y);
#pragma unroll
      for (int e = 0; e < VEC; ++e) ss += y[e] * y[e];
    }
    const A nrm = sqrt(block_sum(ss, red));
    const A home = (is_v ? ovnorm : oknorm)[gid];
    const A sc = nrm > A(0) ? (home > A(0) ? home : A(1)) / nrm : A(0);
    // pass 2 reads the absorber's own chunk before overwriting it (same thread, same c)
    A rs = 0;
    for (int64_t c = tid; c < nch; c += bd) {
      A y[VEC], rd[VEC];
      member_sum(c, y);
#pragma unroll
      for (int e = 0; e < VEC; ++e) y[e] *= sc;
      VecIO<T, VEC>::store(pool + g.base(u, l) + g.off(c * VEC), y, rd);
#pragma unroll
      for (int e = 0; e < VEC; ++e) rs += rd[e] * rd[e];
    }
    const A nn = sqrt(block_sum(rs, red));
    if (tid == 0) norm[gid] = nn;
    __syncthreads();
  }
}

template <typename T, int VEC>
cudaError_t merge_reg(void* pk, void* pv, const Geom& g, void* kn, void* vn, const void* okn,
                      const void* ovn, int32_t* ws, int64_t n_total, ItemSel sel, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  const int64_t nch = g.r() / VEC;
  int bd = 512;
  while (bd > 64 && (int64_t)(bd / 2) * (32 / VEC) >= nch) bd /= 2;
  if (nch > (int64_t)bd * (32 / VEC)) {  // beyond the register-resident path
    merge_long_kernel<T, VEC><<<dim3(148 * 4), 256, 0, s>>>((T*)pk, (T*)pv, g, (A*)kn, (A*)vn,
                                                           (const A*)okn, (const A*)ovn, ws, n_total,
                                                           sel);
    return cudaGetLastError();
  }
  dim3 grid(148 * 4, sel.which == 3 ? 2 : 1);
  merge_reg_kernel<T, VEC><<<grid, bd, 0, s>>>((T*)pk, (T*)pv, g, (A*)kn, (A*)vn, (const A*)okn,
                                               (const A*)ovn, ws, n_total, sel);
  return cudaGetLastError();
}

template <typename T, int EPT>
cudaError_t merge_tma(void* pk, void* pv, const Geom& g, void* kn, void* vn, const void* okn,
                      const void* ovn, int32_t* ws, int64_t n_total, int nbuf, int slot_bytes, ItemSel sel,
                      ExactArgs ex, cudaStream_t s) {
  const int smem = nbuf * slot_bytes + 2 * MG_MAX_BUF * 8 + MG_MAX_BUF * (int)sizeof(SlotMeta) + 256;
  static int attr = 0;  // per instantiation
  if (attr < smem) {
    cudaError_t e = cudaFuncSetAttribute(merge_tma_kernel<T, EPT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  // two CTAs per SM: one CTA's per-item tail (norm reduction, write-back,
  // stored-norm reduction) overlaps the other's streaming. Measured on 4 cfg2
  // layers (6 levels): 1 CTA x 6 slots 4.98 ms, 2 x 3 slots 3.47 ms, 3 x 2 4.33 ms.
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  static const int per_sm = [] {  // tuning knob for A/B measurements
    const char* e = getenv("KVF_MERGE_CTAS_PER_SM");
    return e ? std::max(1, atoi(e)) : 2;
  }();
  // exact mode: fp32 shadow rows stream through the ring as two half-row slots (a bf16
  // slot holds r / 2 floats) instead of plain loads by the consumers; KVF_MERGE_SHADOW_DIRECT
  // restores the plain loads (A/B)
  static const bool direct = getenv("KVF_MERGE_SHADOW_DIRECT") != nullptr;
  const int ring_shadow = ex.shadow && sizeof(T) == 2 && g.r() % 16 == 0 && !direct ? 1 : 0;
  merge_tma_kernel<T, EPT><<<per_sm * n_sm, MG_THREADS, smem, s>>>((T*)pk, (T*)pv, g, (float*)kn, (float*)vn,
                                                         (const float*)okn, (const float*)ovn, ws,
                                                         n_total, nbuf, slot_bytes, sel, ex, ring_shadow);
  return cudaGetLastError();
}

template <typename T>
cudaError_t merge_dispatch(void* pk, void* pv, const Geom& g, void* kn, void* vn, const void* okn,
                           const void* ovn, int32_t* ws, int64_t n_total, ItemSel sel,
                           ExactArgs ex, cudaStream_t s) {
  constexpr int VEC = Vec16<T>::N;
  const int64_t r = g.r();
  const int64_t vbytes = r * (int64_t)sizeof(T);
  const int slot_bytes = (int)((vbytes + 127) / 128 * 128);
  const char* ev = getenv("KVF_MERGE_CTAS_PER_SM");
  const int per_sm = ev ? std::max(1, atoi(ev)) : 2;
  // ring slots per CTA: ~128 KB of copies in flight per SM (more outstanding TMA bytes
  // per SM lower the delivered rate; cfg2 merges: 3 x 32 KB slots x 2 CTAs 18.1 ms,
  // 2 x 32 KB x 2 CTAs 17.5 ms per 2 steps); KVF_MERGE_NBUF overrides (measurements)
  const char* eb = getenv("KVF_MERGE_NBUF");
  const int64_t fit = std::min<int64_t>(MG_MAX_BUF, (200 * 1024 / per_sm) / slot_bytes);  // smem
  // exact mode streams fp32 shadow rows as two slots each: one slot deeper (cfg2, 32 layers:
  // merges 14.3 ms with 2 slots, 13.8 ms with 3)
  const int64_t want = (128 * 1024 / per_sm) / slot_bytes + (ex.shadow && !g.head_mode ? 1 : 0);
  const int nbuf = (int)std::min<int64_t>(fit, eb ? std::max(2, atoi(eb)) : std::max<int64_t>(2, want));
  const bool tma_ok = !std::is_same<T, double>::value && can_vectorize<T>(pk, g) &&
                      can_vectorize<T>(pv, g) && nbuf >= 2 && r <= 64 * MG_CONSUMERS &&
                      (g.d * (int64_t)sizeof(T)) % 16 == 0;
  const bool ring_ok = std::is_same<T, __nv_bfloat16>::value && g.head_mode &&
                       (vbytes == 4096 || vbytes == 2048) && g.t <= 32 && (g.d * 2) % 16 == 0 &&
                       can_vectorize<T>(pk, g) && can_vectorize<T>(pv, g) && !getenv("KVF_MERGE_NO_RING");
  if (ex.shadow) {  // exact mode (bf16 pools, keys)
    if (!std::is_same<T, __nv_bfloat16>::value) return cudaErrorInvalidValue;
    if (!(((tma_ok && !g.head_mode) || ring_ok) && (sel.which & 1))) {
      // keys on the float64 CTA-per-absorber kernel, values below on the usual path
      if (sel.which & 1) {
        cudaError_t e = launch_exact_merge_keys(pk, g, (float*)kn, (const float*)okn, ex.shadow, ex.cap,
                                                ex.sidx, ex.scount, ws, s);
        if (e != cudaSuccess || sel.which == 1) return e;
      }
      sel = ItemSel{2};
      ex = ExactArgs{nullptr, 0, nullptr, nullptr, 0};
    }
  }
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (ex.shadow && !g.head_mode) {  // folded exact mode: keys and values in one ring pass
      const int64_t ept = (r + MG_CONSUMERS - 1) / MG_CONSUMERS;
      if (ept <= 8)
        return merge_tma<T, 8>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, nbuf, slot_bytes, sel, ex, s);
      if (ept <= 16)
        return merge_tma<T, 16>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, nbuf, slot_bytes, sel, ex, s);
      if (ept <= 32)
        return merge_tma<T, 32>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, nbuf, slot_bytes, sel, ex, s);
      return merge_tma<T, 64>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, nbuf, slot_bytes, sel, ex, s);
    }
    // per-head units of 2 or 4 KB: warp per item, per-warp smem ring (3 slots)
    if (ring_ok) {
      auto go = [&](auto kern, int ns, int wpb, int per_sm) {
        const int smem = wpb * ns * (int)vbytes + wpb * ns * (8 + (int)sizeof(RingSlotMeta));
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        // exact mode: fp32 shadow rows through the ring as two half-row slots
        // (KVF_MERGE_SHADOW_DIRECT: plain loads by the consuming warp, A/B)
        static const bool direct = getenv("KVF_MERGE_SHADOW_DIRECT") != nullptr;
        const int ring_shadow = ex.shadow && !direct ? 1 : 0;  // CPL = 4 or 8: even halves
        kern<<<148 * per_sm, wpb * 32, smem, s>>>((__nv_bfloat16*)pk, (__nv_bfloat16*)pv, g, (float*)kn,
                                                  (float*)vn, (const float*)okn, (const float*)ovn, ws,
                                                  n_total, sel, ex, ring_shadow);
        return cudaGetLastError();
      };
      // measured (cfg2 per-head, 2 steps): 8 warps x 3 slots x 2 CTAs/SM 23.6 ms; 6 x 4 x 2 28.6;
      // 4 x 5 x 3 51.2; 8 x 3 x 1 41.1 (merge_warp_kernel: 28.2)
      return vbytes == 4096 ? go(merge_ring_kernel<8, 3>, 3, 8, 2) : go(merge_ring_kernel<4, 3>, 3, 8, 2);
    }
  }
  if constexpr (!std::is_same<T, double>::value) {
    // short vectors (per-head units): warp per item
    const bool vec_ok = can_vectorize<T>(pk, g) && can_vectorize<T>(pv, g);
    if (vec_ok && vbytes <= 4096 && r % (32 * VEC) == 0) {
      const int cpl = (int)(r / (32 * VEC));
      auto launch = [&](auto kern) {
        kern<<<148 * 8, 256, 0, s>>>((T*)pk, (T*)pv, g, (float*)kn, (float*)vn, (const float*)okn,
                                     (const float*)ovn, ws, n_total, sel);
        return cudaGetLastError();
      };
      if (cpl == 1) return launch(merge_warp_kernel<T, VEC, 1>);
      if (cpl == 2) return launch(merge_warp_kernel<T, VEC, 2>);
      if (cpl == 4) return launch(merge_warp_kernel<T, VEC, 4>);
      if (cpl == 8) return launch(merge_warp_kernel<T, VEC, 8>);
    }
    if (tma_ok) {
      const int64_t ept = (r + MG_CONSUMERS - 1) / MG_CONSUMERS;
      if (ept <= 8)
        return merge_tma<T, 8>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, nbuf, slot_bytes, sel, ex, s);
      if (ept <= 16)
        return merge_tma<T, 16>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, nbuf, slot_bytes, sel, ex, s);
      if (ept <= 32)
        return merge_tma<T, 32>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, nbuf, slot_bytes, sel, ex, s);
      return merge_tma<T, 64>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, nbuf, slot_bytes, sel, ex, s);
    }
  }
  if (can_vectorize<T>(pk, g) && can_vectorize<T>(pv, g))
    return merge_reg<T, VEC>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, sel, s);
  return merge_reg<T, 1>(pk, pv, g, kn, vn, okn, ovn, ws, n_total, sel, s);
}
}  // namespace

cudaError_t launch_merge_groups(void* pool_k, void* pool_v, int dtype, const Geom& g,
                                void* knorm, void* vnorm, const void* oknorm,
                                const void* ovnorm, int32_t* level_ws, int which, float* shadow,
                                int64_t shadow_cap, int32_t* sidx, int32_t* scount, cudaStream_t s) {
  const int write_rows = (which & kMergeLastLevel) ? 0 : 1;
  which &= ~kMergeLastLevel;
  if (which < 1 || which > 3) return cudaErrorInvalidValue;
  const ItemSel sel{which};
  const ExactArgs ex{shadow, shadow_cap, sidx, scount, write_rows};
  if (shadow && dtype != BF16) return cudaErrorInvalidValue;
  const int64_t n_total = g.units() * g.NB;
  switch (dtype) {
    case F64:
      return merge_dispatch<double>(pool_k, pool_v, g, knorm, vnorm, oknorm, ovnorm, level_ws,
                                    n_total, sel, ex, s);
    case F32:
      return merge_dispatch<float>(pool_k, pool_v, g, knorm, vnorm, oknorm, ovnorm, level_ws,
                                   n_total, sel, ex, s);
    default:
      return merge_dispatch<__nv_bfloat16>(pool_k, pool_v, g, knorm, vnorm, oknorm, ovnorm,
                                           level_ws, n_total, sel, ex, s);
  }
}

}  // namespace kvf
