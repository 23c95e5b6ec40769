// Sharing-aware paged decode over a fused cache (
// fused blocks shared by several requests should be
// fetched once, not once per request).
//
// After BFF a physical block is referenced by slots of several requests, at
// unrelated positions. Softmax is permutation invariant, so:
//   * each request's slots are visited in ascending physical-block order and
//     cut into items of IB slots (one (o, m, l) partial per item and query
//     head, merged by decode_combine_kernel exactly like flash-decoding
//     splits);
//   * all items of a KV head are swept in ascending order of their middle
//     slot's physical block, heads one after another, by persistent warps.
// Requests that share a block then fetch it within a short window: the first
// read comes from HBM, the others from L2, so DRAM traffic falls from the
// logical bytes towards the unique (fused) bytes.
//
// The schedule is built once per table (kvf_decode_schedule): a per-request
// bitonic sort in shared memory, then a counting sort of the items by first
// physical block (histogram, scan, scatter). The scatter also gathers each
// item's physical ids and K/V scales into contiguous arrays, so the decode
// warps load their slot metadata with one independent load per lane.
//
// Decode warp loop: one block (its head slice, K and V) per warp tile, 2-stage
// TMA ring per warp running across item boundaries, 12 warps per SM for
// 16-token blocks (the loop is issue-latency bound: more warps beat deeper rings).
// S^T = K Q^T puts the block's tokens on the mma M dimension and the GQA group
// on N (half the mma.sync of a query-rows-on-M layout at G = 4); P^T is moved
// to the B-operand layout with movmatrix and O^T = V^T P^T accumulates with the
// head dimension on M (bf16 in, fp32 accumulate, swizzle-aware ldmatrix).
// Slot metadata and query fragments of item n+1 are fetched while item n
// computes.
#include <algorithm>
#include <cstdlib>
#include "kernels.h"
#include "tma_util.cuh"

namespace kvf {

using namespace tma;
namespace {
// query fragments of (b, kvh): rows = query heads of the GQA group (zero past G)
template <int D>
__device__ __forceinline__ void load_q_frags(uint32_t (&qa)[D / 16][2], const void* q, int q_dtype,
                                             int64_t b, int kvh, int G, int Hq, int grp, int tig) {
  const bool real = grp < G;
  const int64_t qrow = (b * Hq + (int64_t)kvh * G + (real ? grp : 0)) * D;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    const int e0 = ks * 16 + 2 * tig;
    if (!real) {
      qa[ks][0] = qa[ks][1] = 0u;
    } else if (q_dtype == BF16) {
      const uint32_t* qp = reinterpret_cast<const uint32_t*>((const __nv_bfloat16*)q + qrow);
      qa[ks][0] = __ldg(qp + e0 / 2);
      qa[ks][1] = __ldg(qp + (e0 + 8) / 2);
    } else {
      const float2* qp = reinterpret_cast<const float2*>((const float*)q + qrow);
      const float2 a = __ldg(qp + e0 / 2), c = __ldg(qp + (e0 + 8) / 2);
      qa[ks][0] = pack_bf16(a.x, a.y);
      qa[ks][1] = pack_bf16(c.x, c.y);
    }
  }
}
}  // namespace

template <int D, int T, int DW, int DNS, int IB, bool DEDUP>
__global__ void __launch_bounds__(DW * 32)
decode_sched_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                    const void* __restrict__ q, int q_dtype, Geom g, int64_t layer, int64_t B,
                    int64_t p_blocks, int Hq, float sm_scale, const int32_t* __restrict__ meta,
                    const int32_t* __restrict__ sphys, const float* __restrict__ sks,
                    const float* __restrict__ svs, const int32_t* __restrict__ n_items_p,
                    int64_t cap, float* __restrict__ part, int head_minor, int l2_mode) {
  static_assert(2 * IB <= 32, "slot metadata of two items must fit in one warp");
  static_assert(T == 16 || T == 32, "blocks of 16 or 32 tokens");
  static_assert(IB >= DNS - 1, "the copy lookahead may not pass the next item");
  constexpr int HALVES = D / 64;
  constexpr int KS = D / 16;   // k-steps of S^T = K Q^T (head dim)
  constexpr int MT = T / 16;   // token m-tiles of S^T = k-steps of O^T = V^T P^T
  constexpr int DT = D / 16;   // head-dim m-tiles of O^T
  constexpr int BOX = T * 128;                 // one (block, d half) box
  constexpr int TENS = HALVES * BOX;           // one block's K (or V) head slice
  constexpr int STAGE = 2 * TENS;
  constexpr uint32_t IBMASK = IB == 32 ? 0xffffffffu : ((1u << IB) - 1u);
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* dsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, tig = lane & 3;
  uint8_t* wst = dsm + (size_t)warp * DNS * STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + (size_t)DW * DNS * STAGE) + warp * DNS;

  const int G = Hq / g.h;
  const int64_t nit = (p_blocks + IB - 1) / IB;
  const int64_t n_items = *n_items_p;
  const int64_t total = n_items * g.h;
  const int64_t NW = (int64_t)gridDim.x * DW;
  const int64_t gidx0 = (int64_t)blockIdx.x * DW + warp;
  if (gidx0 >= total) return;  // warp-uniform; no CTA-wide barrier below
  const int64_t my_items = (total - gidx0 + NW - 1) / NW;
  const int rowbase = (int)(layer * g.NB);

  // schedule row of work index gi: head-major sweep, or (folded schedules) head-minor --
  // the KV heads of one item run on adjacent warps, so a block's head slices are read
  // together instead of in h separate sweeps
  auto row_of = [&](int64_t gi, int& kvh) {
    if (head_minor) {
      kvh = (int)(gi % g.h);
      return gi / g.h;
    }
    kvh = (int)(gi / n_items);
    return (g.head_mode ? (int64_t)kvh * cap : 0) + gi % n_items;
  };
  // slot metadata of work index gi into lanes [par*IB, par*IB + IB)
  int32_t phys_l = 0;
  float ks_l = 0.f, vs_l = 0.f;
  bool once_l = false;  // the slot's block is referenced by no other slot of this unit
  auto load_info = [&](int par, int64_t gi) {
    if (gi >= total || lane < par * IB || lane >= par * IB + IB) return;
    int kvh;
    const int64_t e = row_of(gi, kvh) * IB + (lane - par * IB);
    phys_l = __ldg(sphys + e);
    const float kraw = __ldg(sks + e);  // sign bit: single-reference block (schedule build)
    once_l = signbit(kraw);
    ks_l = fabsf(kraw) * sm_scale;
    vs_l = __ldg(svs + e);
  };
  // repeats inside an item: bit j set when slot j maps to the same physical
  // block as slot j - 1 (a request's slots are sorted by physical block, so a
  // block the request references several times forms one run). A run is
  // loaded once, its S = K q^T computed once and reused with each slot's
  // scale, and its P V done once on the scale-weighted sum of the slots' P
  // (computation reuse of shared blocks).
  auto dup_mask = [&](int par) -> uint32_t {
    if constexpr (!DEDUP) return 0u;
    const int32_t prev = __shfl_up_sync(0xffffffffu, phys_l, 1);
    const bool d = lane > par * IB && lane < par * IB + IB && phys_l >= 0 && prev == phys_l;
    return (__ballot_sync(0xffffffffu, d) >> (par * IB)) & IBMASK;
  };

  if (lane == 0) {
    for (int s = 0; s < DNS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  load_info(0, gidx0);
  load_info(1, gidx0 + NW);
  int kvh_cur, kvh_nxt = 0;
  int32_t meta_cur = __ldg(meta + row_of(gidx0, kvh_cur));
  int32_t meta_nxt = 0;
  if (my_items > 1) meta_nxt = __ldg(meta + row_of(gidx0 + NW, kvh_nxt));
  uint32_t qa[KS][2];
  load_q_frags<D>(qa, q, q_dtype, meta_cur / nit, kvh_cur, G, Hq, grp, tig);
  __syncwarp();

  // copy issue: the next run head (item is_n, slot is_j) into stage is_stage
  int is_stage = 0, is_j = 0, is_par = 0;
  int64_t is_n = 0, cur_n = 0;
  uint32_t is_dmask = dup_mask(0);
  // L2 policy of the block copies (l2_mode 1: blocks read by one slot only are evict-first,
  // so the L2 keeps the shared blocks until their other readers arrive; 2: shared blocks
  // additionally evict-last; 0: no hint)
  const uint64_t pol_once = l2_policy_evict_first();
  const uint64_t pol_shared = l2_mode == 2 ? l2_policy_evict_last() : l2_policy_evict_normal();
  auto issue_next = [&]() {  // all lanes (shuffles, ballots); lane 0 issues the copies
    while (DEDUP && is_n < my_items && ((is_dmask >> is_j) & 1u)) {  // repeats load nothing
      if (++is_j == IB) {
        is_j = 0;
        is_par ^= 1;
        ++is_n;
        is_dmask = dup_mask(is_par);
      }
    }
    if (is_n >= my_items) return;
    const int32_t ph = __shfl_sync(0xffffffffu, phys_l, is_par * IB + is_j);
    const bool once = __shfl_sync(0xffffffffu, once_l ? 1 : 0, is_par * IB + is_j) != 0;
    if (lane == 0) {
      const int kvh = is_n == cur_n ? kvh_cur : kvh_nxt;  // issue runs at most one item ahead
      uint8_t* st = wst + (size_t)is_stage * STAGE;
      const int row = rowbase + (ph < 0 ? 0 : ph);  // padding loads block 0 (p = 0)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[is_stage], (uint32_t)STAGE);
      if (l2_mode) {
        const uint64_t pol = once ? pol_once : pol_shared;
#pragma unroll
        for (int hf = 0; hf < HALVES; ++hf) {
          tma4_hint(st + hf * BOX, &kmap, &bars[is_stage], hf * 64, kvh, 0, row, pol);
          tma4_hint(st + TENS + hf * BOX, &vmap, &bars[is_stage], hf * 64, kvh, 0, row, pol);
        }
      } else {
#pragma unroll
        for (int hf = 0; hf < HALVES; ++hf) {
          tma4(st + hf * BOX, &kmap, &bars[is_stage], hf * 64, kvh, 0, row);
          tma4(st + TENS + hf * BOX, &vmap, &bars[is_stage], hf * 64, kvh, 0, row);
        }
      }
    }
    if (++is_stage == DNS) is_stage = 0;
    if (++is_j == IB) {
      is_j = 0;
      is_par ^= 1;
      ++is_n;
      if (is_n < my_items) is_dmask = dup_mask(is_par);
    }
  };
  for (int i = 0; i < DNS - 1; ++i) issue_next();
  const int lr = lane & 7, lm = lane >> 3;
  // swizzled smem address of (token, element) inside a block's head slice
  auto addr = [&](uint32_t base, int tok, int e) {
    const int hf = e >> 6, ch = (e & 63) >> 3;
    return base + (uint32_t)(hf * BOX + tok * 128 + ((ch ^ (tok & 7)) << 4));
  };
  int cs_stage = 0;
  uint32_t cs_phase = 0;

  for (int64_t n = 0; n < my_items; ++n) {
    const int64_t gi = gidx0 + n * NW;
    const int par = (int)(n & 1);
    const bool has_next = n + 1 < my_items;
    const int64_t b = meta_cur / nit, k = meta_cur % nit;
    const int kvh = kvh_cur;
    cur_n = n;
    const uint32_t dmask = dup_mask(par);
    if (n > 0) load_info(par ^ 1, gi + NW);  // item n+1 replaces item n-1 (consumed)
    int32_t meta_nn = 0;
    int kvh_nn = 0;
    if (n + 2 < my_items) meta_nn = __ldg(meta + row_of(gi + 2 * NW, kvh_nn));
    uint32_t qn[KS][2];
    // per-thread state for heads 2*tig, 2*tig+1: running max (warp-uniform per
    // head), partial denominator over this thread's tokens, O^T fragments
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float o[DT][4];
#pragma unroll
    for (int mt = 0; mt < DT; ++mt)
#pragma unroll
      for (int c = 0; c < 4; ++c) o[mt][c] = 0.f;

    bool q_next_loaded = false;
#pragma unroll 1
    for (int j = 0; j < IB;) {
      int len = 1;  // run of slots on the same physical block
      if constexpr (DEDUP)
        while (j + len < IB && ((dmask >> (j + len)) & 1u)) ++len;
      issue_next();
      if (!q_next_loaded && has_next) {  // next item's query rows, consumed after this item
        load_q_frags<D>(qn, q, q_dtype, meta_nxt / nit, kvh_nxt, G, Hq, grp, tig);
        q_next_loaded = true;
      }
      const bool valid = __shfl_sync(0xffffffffu, phys_l, par * IB + j) >= 0;
      mbar_wait(&bars[cs_stage], cs_phase);
      const uint32_t kb = su32(wst + (size_t)cs_stage * STAGE);
      const uint32_t vb = kb + TENS;
      if (++cs_stage == DNS) {
        cs_stage = 0;
        cs_phase ^= 1u;
      }
      // ---- S^T[token][head] = K Q^T once per run: tokens on M, query heads on N ----
      float sa[MT][4], sb[MT][4];  // even / odd k-steps (shorter mma chains)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int c = 0; c < 4; ++c) sa[mt][c] = sb[mt][c] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4(addr(kb, mt * 16 + (lm & 1) * 8 + lr, ks * 16 + (lm >> 1) * 8), a0, a1, a2, a3);
          if (ks & 1)
            mma16816_full(sb[mt], a0, a1, a2, a3, qa[ks][0], qa[ks][1]);
          else
            mma16816_full(sa[mt], a0, a1, a2, a3, qa[ks][0], qa[ks][1]);
        }
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int c = 0; c < 4; ++c) sa[mt][c] += sb[mt][c];
      // ---- online softmax over the run's slots (logits = slot scale x S) ----
      float mx[2] = {-INFINITY, -INFINITY};
      for (int r = 0; r < len; ++r) {
        const float ksr = __shfl_sync(0xffffffffu, ks_l, par * IB + j + r);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int c = 0; c < 4; ++c) mx[c & 1] = fmaxf(mx[c & 1], valid ? sa[mt][c] * ksr : -INFINITY);
      }
      float alpha[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], 4));
        mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], 8));
        mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], 16));
        const float m_new = fmaxf(m_run[hh], mx[hh]);
        alpha[hh] = m_new == -INFINITY ? 1.f : __expf(m_run[hh] - m_new);
        m_run[hh] = m_new;
        l_run[hh] *= alpha[hh];
      }
      float pe[MT][4];  // sum over the run of P^T * v_scale
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int c = 0; c < 4; ++c) pe[mt][c] = 0.f;
      for (int r = 0; r < len; ++r) {
        const float ksr = __shfl_sync(0xffffffffu, ks_l, par * IB + j + r);
        const float vsr = __shfl_sync(0xffffffffu, vs_l, par * IB + j + r);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float m = m_run[c & 1];
            const float pr = (!valid || m == -INFINITY) ? 0.f : __expf(sa[mt][c] * ksr - m);
            l_run[c & 1] += pr;
            pe[mt][c] = fmaf(pr, vsr, pe[mt][c]);
          }
      }
#pragma unroll
      for (int mt = 0; mt < DT; ++mt) {
        o[mt][0] *= alpha[0];
        o[mt][1] *= alpha[1];
        o[mt][2] *= alpha[0];
        o[mt][3] *= alpha[1];
      }
      // ---- O^T[d][head] += V^T P^T: head dim on M, heads on N, tokens on K ----
#pragma unroll
      for (int kk = 0; kk < MT; ++kk) {
        // B fragment = P^T[token][head]: transpose the two 8x8 token halves
        const uint32_t b0 = movm_t(pack_bf16(pe[kk][0], pe[kk][1]));
        const uint32_t b1 = movm_t(pack_bf16(pe[kk][2], pe[kk][3]));
#pragma unroll
        for (int mt = 0; mt < DT; ++mt) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4_t(addr(vb, kk * 16 + (lm >> 1) * 8 + lr, mt * 16 + (lm & 1) * 8), a0, a1, a2, a3);
          mma16816_full(o[mt], a0, a1, a2, a3, b0, b1);
        }
      }
      __syncwarp();  // the stage is refilled by a later issue
      j += len;
    }
    // ---- item partial (one per request x query head x item) ----
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float l = l_run[hh];
      l += __shfl_xor_sync(0xffffffffu, l, 4);
      l += __shfl_xor_sync(0xffffffffu, l, 8);
      l += __shfl_xor_sync(0xffffffffu, l, 16);
      const int hd = 2 * tig + hh;
      if (hd < G) {
        float* pp = part + ((b * Hq + (int64_t)kvh * G + hd) * nit + k) * (D + 2);
#pragma unroll
        for (int mt = 0; mt < DT; ++mt) {
          pp[mt * 16 + grp] = o[mt][hh];
          pp[mt * 16 + grp + 8] = o[mt][2 + hh];
        }
        if (grp == 0) {
          pp[D] = m_run[hh];
          pp[D + 1] = l;
        }
      }
    }
    if (has_next) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        qa[ks][0] = qn[ks][0];
        qa[ks][1] = qn[ks][1];
      }
      meta_cur = meta_nxt;
      kvh_cur = kvh_nxt;
      meta_nxt = meta_nn;
      kvh_nxt = kvh_nn;
    }
  }
}

// ---- schedule build ------------------------------------------------------
// (1) per (request, head unit): positions sorted by (phys, position) in smem;
//     item keys = physical block of each item's middle slot; key histogram
__global__ void sched_order_kernel(const int32_t* __restrict__ table, Geom g, int64_t layer,
                                   int64_t B, int64_t p_blocks, const int32_t* __restrict__ seq_blocks,
                                   int ib, int sortn, int key_mode, int32_t* __restrict__ order,
                                   int32_t* __restrict__ item_key, int32_t* __restrict__ hist,
                                   int32_t* __restrict__ refs) {
  extern __shared__ unsigned long long keys[];
  const int64_t b = blockIdx.x;
  const int64_t hu = blockIdx.y;
  const int64_t unit = g.head_mode ? layer * g.h + hu : layer;
  int64_t nblk = seq_blocks ? (int64_t)seq_blocks[b] : p_blocks;
  nblk = nblk < 0 ? 0 : (nblk > p_blocks ? p_blocks : nblk);
  const int32_t* tab = table + unit * g.NB + b * p_blocks;
  for (int j = threadIdx.x; j < sortn; j += blockDim.x) {
    unsigned long long key = ~0ull;
    if (j < nblk) {
      int32_t ph = tab[j];
      ph = ph < 0 ? 0 : (ph >= g.NB ? (int32_t)(g.NB - 1) : ph);
      key = ((unsigned long long)(uint32_t)ph << 32) | (uint32_t)j;
      atomicAdd(&refs[hu * g.NB + ph], 1);
    }
    keys[j] = key;
  }
  __syncthreads();
  for (int kk = 2; kk <= sortn; kk <<= 1)
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < sortn; i += blockDim.x) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const unsigned long long a = keys[i], c = keys[ixj];
          if ((a > c) == ((i & kk) == 0)) {
            keys[i] = c;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  const int64_t nit = (p_blocks + ib - 1) / ib;
  int32_t* ord = order + (hu * B + b) * p_blocks;
  for (int64_t j = threadIdx.x; j < p_blocks; j += blockDim.x)
    ord[j] = j < nblk ? (int32_t)(keys[j] & 0xffffffffull) : -1;
  for (int64_t k = threadIdx.x; k < nit; k += blockDim.x) {
    int32_t key = -1;
    if (k * ib < nblk) {
      const int64_t last = min((int64_t)nblk, (k + 1) * ib) - 1;
      const int64_t pick = key_mode == 1 ? (k * ib + last) / 2 : (key_mode == 2 ? last : k * ib);
      key = (int32_t)(keys[pick] >> 32);
      atomicAdd(&hist[hu * g.NB + key], 1);
    }
    item_key[(hu * B + b) * nit + k] = key;
  }
}

// (2) exclusive scan of one head unit's key histogram -> counting-sort offsets
__global__ void sched_scan_kernel(int32_t* __restrict__ hist, int64_t NB, int32_t* __restrict__ n_items) {
  __shared__ int32_t part_sum[1024];
  int32_t* h = hist + (int64_t)blockIdx.x * NB;
  const int64_t per = (NB + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = min(NB, lo + per);
  int32_t sum = 0;
  for (int64_t i = lo; i < hi; ++i) sum += h[i];
  part_sum[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // Hillis-Steele inclusive scan
    const int32_t v = threadIdx.x >= off ? part_sum[threadIdx.x - off] : 0;
    __syncthreads();
    part_sum[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = part_sum[threadIdx.x] - sum;
  for (int64_t i = lo; i < hi; ++i) {
    const int32_t v = h[i];
    h[i] = run;
    run += v;
  }
  if (threadIdx.x == blockDim.x - 1) n_items[blockIdx.x] = part_sum[threadIdx.x];
}

// (3) scatter items to their sorted rows, gathering slot metadata
__global__ void sched_scatter_kernel(const int32_t* __restrict__ item_key,
                                     const int32_t* __restrict__ order,
                                     const int32_t* __restrict__ table,
                                     const float* __restrict__ k_scale,
                                     const float* __restrict__ v_scale, Geom g, int64_t layer,
                                     int64_t B, int64_t p_blocks, int ib,
                                     int32_t* __restrict__ hist, int32_t* __restrict__ meta,
                                     int32_t* __restrict__ sphys, float* __restrict__ sks,
                                     float* __restrict__ svs, int32_t* __restrict__ n_repeats,
                                     const int32_t* __restrict__ refs) {
  const int64_t hu = blockIdx.y;
  const int64_t unit = g.head_mode ? layer * g.h + hu : layer;
  const int64_t nit = (p_blocks + ib - 1) / ib;
  const int64_t cap = B * nit;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < cap;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int32_t key = item_key[hu * cap + x];
    if (key < 0) continue;
    const int64_t pos = hu * cap + atomicAdd(&hist[hu * g.NB + key], 1);
    meta[pos] = (int32_t)x;
    const int64_t b = x / nit, k = x % nit;
    const int32_t* ord = order + (hu * B + b) * p_blocks;
    int32_t prev = -1, reps = 0;
    for (int j = 0; j < ib; ++j) {
      const int64_t jj = k * ib + j;
      const int32_t o = jj < p_blocks ? ord[jj] : -1;
      int32_t ph = -1;
      float ksv = 0.f, vsv = 0.f;
      if (o >= 0) {
        const int64_t slot = unit * g.NB + b * p_blocks + o;
        ph = table[slot];
        ksv = k_scale[slot];
        vsv = v_scale[slot];
        // a block no other slot references is read once: flagged in the K scale's sign
        // bit (scales are >= 0) for the decode's L2 eviction policy
        const int32_t pc = ph < 0 ? 0 : (ph >= g.NB ? (int32_t)(g.NB - 1) : ph);
        if (refs[hu * g.NB + pc] == 1) ksv = -ksv;
      }
      sphys[pos * ib + j] = ph;
      sks[pos * ib + j] = ksv;
      svs[pos * ib + j] = vsv;
      if (j > 0 && ph >= 0 && ph == prev) ++reps;
      prev = ph;
    }
    if (reps && n_repeats) atomicAdd(n_repeats, reps);
  }
}

bool decode_sched_item_blocks_ok(int ib) { return ib == 8 || ib == 16; }

__global__ void remap_ids_kernel(const int32_t* __restrict__ ids, int64_t n,
                                 const int32_t* __restrict__ map, int64_t map_len,
                                 int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = ids[i];
    out[i] = (x >= 0 && x < map_len) ? map[x] : -1;
  }
}

cudaError_t launch_remap_ids(const int32_t* ids, int64_t n, const int32_t* map, int64_t map_len,
                             int32_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 4096);
  remap_ids_kernel<<<(unsigned)blocks, 256, 0, s>>>(ids, n, map, map_len, out);
  return cudaGetLastError();
}

int64_t decode_schedule_ws_ints(int64_t nh, int64_t NB, int64_t B, int64_t p_blocks, int ib) {
  return 2 * nh * NB + nh * B * ((p_blocks + ib - 1) / ib);  // hist, refs, item keys
}

cudaError_t launch_decode_schedule(const int32_t* table, const float* k_scale, const float* v_scale,
                                   const Geom& g, int64_t layer, int64_t B, int64_t p_blocks,
                                   const int32_t* seq_blocks, int ib, int32_t* order,
                                   int32_t* meta, int32_t* phys, float* ks, float* vs,
                                   int32_t* n_items, int32_t* n_repeats, int32_t* ws,
                                   cudaStream_t s) {
  const int64_t nh = g.head_mode ? g.h : 1;
  const int64_t nit = (p_blocks + ib - 1) / ib;
  int32_t* hist = ws;
  int32_t* refs = ws + nh * g.NB;
  int32_t* item_key = ws + 2 * nh * g.NB;
  cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(int32_t) * 2 * nh * g.NB, s);  // hist + refs
  if (e != cudaSuccess) return e;
  if (n_repeats && (e = cudaMemsetAsync(n_repeats, 0, sizeof(int32_t), s)) != cudaSuccess) return e;
  if (B == 0) return cudaMemsetAsync(n_items, 0, sizeof(int32_t) * nh, s);
  int sortn = 1;
  while (sortn < p_blocks) sortn <<= 1;
  const size_t smem = sizeof(unsigned long long) * sortn;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(sched_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // items are counting-sorted by the physical block of their middle slot: measured on
  // a cfg4 layer (batch 256 x 8K), middle 827-831 us vs first 847-862 vs last 853 (the
  // concurrent items' blocks stay closer together, fewer L2 re-reads); KVF_SCHED_KEY =
  // 0 / 1 / 2 selects first / middle / last (measurements)
  static const int key_mode = [] {
    const char* e = getenv("KVF_SCHED_KEY");
    return e ? atoi(e) : 1;
  }();
  sched_order_kernel<<<dim3((unsigned)B, (unsigned)nh), 512, smem, s>>>(
      table, g, layer, B, p_blocks, seq_blocks, ib, sortn, key_mode, order, item_key, hist, refs);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  sched_scan_kernel<<<(unsigned)nh, 1024, 0, s>>>(hist, g.NB, n_items);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int64_t n = B * nit;
  sched_scatter_kernel<<<dim3((unsigned)std::min<int64_t>((n + 127) / 128, 8192), (unsigned)nh), 128, 0, s>>>(
      item_key, order, table, k_scale, v_scale, g, layer, B, p_blocks, ib, hist, meta, phys, ks, vs,
      n_repeats, refs);
  return cudaGetLastError();
}

namespace {
template <int D, int T, int DW, int DNS, int IB, bool DEDUP>
cudaError_t decode_sched_t(const DecodeArgs& a, cudaStream_t s) {
  CUtensorMap km, vm;
  if (!make_map(&km, a.pool_k, a.g) || !make_map(&vm, a.pool_v, a.g)) return cudaErrorInvalidValue;
  constexpr int STAGE = 2 * (D / 64) * T * 128;
  constexpr int smem = 1024 + DW * DNS * STAGE + DW * DNS * 8;
  auto kern = decode_sched_kernel<D, T, DW, DNS, IB, DEDUP>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, DW * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t nit = (a.p_blocks + IB - 1) / IB;
  const int64_t work_max = a.B * nit * a.g.h;  // every item of every request valid
  const int64_t grid = std::min<int64_t>((int64_t)n_sm * per_sm, (work_max + DW - 1) / DW);
  if (grid < 1) return cudaSuccess;
  const SchedView& v = *a.sched;
  static const int env_minor = [] {  // KVF_SCHED_HEAD_MINOR: sweep order A/B
    const char* e = getenv("KVF_SCHED_HEAD_MINOR");
    return e ? atoi(e) : 0;
  }();
  const int head_minor = (!a.g.head_mode && env_minor) ? 1 : 0;
  // KVF_DECODE_L2: L2 eviction policy A/B (see the kernel). Measured on a cfg4 layer (batch
  // 256 x 8K, CR 2.09): no hint 822 us, evict-first for single-reference blocks 778 us,
  // + evict-last for shared blocks 771 us; DRAM reads 4.61 -> 4.18 GB (unique 4.12 GB)
  static const int l2_mode = [] {
    const char* e = getenv("KVF_DECODE_L2");
    return e ? atoi(e) : 2;
  }();
  kern<<<(unsigned)grid, DW * 32, smem, s>>>(km, vm, a.q, a.q_dtype, a.g, a.layer, a.B, a.p_blocks,
                                            a.Hq, (float)a.sm_scale, v.meta, v.phys, v.ks, v.vs,
                                            v.n_items, v.cap, (float*)a.ws, head_minor, l2_mode);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_decode_combine(a, nit, IB, s);
}

template <int D, int T>
cudaError_t decode_sched_ib(const DecodeArgs& a, cudaStream_t s) {
  // one block per warp tile; 16-token blocks: 8 KB stages, 12 warps x 2 stages.
  // Measured on B200 at batch 64 x 4K (us per layer): 8 warps x 3 stages 143.6,
  // 12 x 2 121.8, 13 x 2 138.1, 14 x 2 122.8, 9 x 3 152.0, 7 x 4 139.1; two blocks
  // per tile: 6 x 2 141.0, 4 x 3 164.4 (the warp loop is latency bound: warps per
  // SM -- balanced over the 4 schedulers -- beat deeper rings and larger tiles).
  constexpr int DW = T == 16 ? 12 : 6;
  // runs of repeated blocks (CFF, in-request sharing) take the dedup variant;
  // caches without repeats keep the leaner loop
  if (a.sched->dedup) {
    if (a.sched->ib == 16) return decode_sched_t<D, T, DW, 2, 16, true>(a, s);
    if (a.sched->ib == 8) return decode_sched_t<D, T, DW, 2, 8, true>(a, s);
  } else {
    if (a.sched->ib == 16) return decode_sched_t<D, T, DW, 2, 16, false>(a, s);
    if (a.sched->ib == 8) return decode_sched_t<D, T, DW, 2, 8, false>(a, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

bool decode_sched_shape_ok(int t, int d) { return (t == 16 || t == 32) && (d == 64 || d == 128); }

cudaError_t launch_decode_sched(const DecodeArgs& a, cudaStream_t s) {
  if (!decode_tma_supported(a) || !a.sched || !decode_sched_shape_ok(a.g.t, a.g.d))
    return cudaErrorInvalidValue;
  if (a.g.d == 128) return a.g.t == 16 ? decode_sched_ib<128, 16>(a, s) : decode_sched_ib<128, 32>(a, s);
  return a.g.t == 16 ? decode_sched_ib<64, 16>(a, s) : decode_sched_ib<64, 32>(a, s);
}

}  // namespace kvf
