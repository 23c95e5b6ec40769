// K6 main path (bf16 pools, t | 32, d in {64, 128}, G <= 8): TMA-fed
// flash-decoding over the fused cache (attention.py:58-80 generalised).
//
// CTA = (split, kv head, request), 4 warps; warp w owns 32-token tiles
// w, w+4, ... of the split and runs its own 3-stage TMA ring:
//   * block table entries and per-slot K/V scales for all its tiles are
//     fetched once up front (one lane per block), so the copy issue never
//     waits on a dependent global load;
//   * each block's head slice (t tokens x d) arrives as 128B-swizzled TMA
//     boxes {64, 1, t, 1} of the pool's (d, h, t, rows) tensor map;
//   * S^T = Q K^T and O += (P * v_scale) V run on mma.sync m16n8k16 (bf16 in,
//     fp32 accumulate) with swizzle-aware ldmatrix addressing;
//   * the 4 warp partials are merged in smem into one (o, m, l) split partial.
// K_slot = k_scale[slot] * pool_k[table[slot]]: shared fused blocks are read
// as stored, never materialised per slot.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include "kernels.h"
#include "tma_util.cuh"

namespace kvf {

using namespace tma;
namespace {
constexpr int DTT = kDecodeTileTokens;  // tokens per warp tile
constexpr int DTILES_MIN = 4;  // fewest tiles per warp per split of any config
}  // namespace

// smem layout of one stage: [tensor K|V][block of tile][d half][t rows x 128 B]
template <int D, int DW, int DNS, int DTILES>
__global__ void __launch_bounds__(DW * 32)
decode_tma_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                  const void* __restrict__ q, int q_dtype, Geom g, int64_t layer,
                  const int32_t* __restrict__ table, const float* __restrict__ k_scale,
                  const float* __restrict__ v_scale, int64_t p_blocks,
                  const int32_t* __restrict__ seq_blocks, int Hq, float sm_scale,
                  float* __restrict__ part) {
  constexpr int HALVES = D / 64;
  constexpr int KS = D / 16;
  constexpr int NE = D / 8;
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* dsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  const int t = g.t;
  const int bpt = DTT / t;                       // blocks per tile
  const int box_bytes = t * 128;                 // one (block, half) box
  const int tens_bytes = bpt * HALVES * box_bytes;
  const int stage_bytes = 2 * tens_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, tig = lane & 3;
  uint8_t* wst = dsm + (size_t)warp * DNS * stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + (size_t)DW * DNS * stage_bytes) + warp * DNS;

  const int G = Hq / g.h;
  const int64_t b = blockIdx.z;
  const int kvh = blockIdx.y;
  const int64_t split = blockIdx.x, nsplit = gridDim.x;
  const int64_t unit = g.head_mode ? layer * g.h + kvh : layer;
  const int64_t nblk = seq_blocks ? (int64_t)seq_blocks[b] : p_blocks;
  const int64_t span_blocks = (int64_t)DW * DTILES * bpt;  // blocks per split
  // block index of slot j (tile j / bpt of this warp, block j % bpt)
  auto blk_of = [&](int j) {
    const int i = j / bpt, bb = j % bpt;
    return split * span_blocks + (int64_t)(i * DW + warp) * bpt + bb;
  };
  // ---- table entries and scales of every block this warp will read ----
  int32_t phys_l = 0;
  float ks_l = 0.f, vs_l = 0.f;
  bool val_l = false;
  if (lane < DTILES * bpt) {
    const int64_t blk = blk_of(lane);
    if (blk < nblk) {
      const int64_t slot = unit * g.NB + b * p_blocks + blk;
      phys_l = table[slot];
      ks_l = k_scale[slot] * sm_scale;
      vs_l = v_scale[slot];
      val_l = true;
    }
  }
  if (lane == 0) {
    for (int s = 0; s < DNS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t rowbase = layer * g.NB;

  auto issue = [&](int i) {  // all lanes (shuffles), lane 0 issues the copies
    const int s = i % DNS;
    uint8_t* st = wst + (size_t)s * stage_bytes;
    uint32_t bytes = 0;
    int32_t ph[DTT];  // per block of the tile (bpt <= 32)
#pragma unroll 1
    for (int bb = 0; bb < bpt; ++bb) {
      ph[bb] = __shfl_sync(0xffffffffu, phys_l, i * bpt + bb);
      bytes += 2u * HALVES * box_bytes;  // invalid blocks load block 0 (finite data, p = 0)
    }
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[s], bytes);
      for (int bb = 0; bb < bpt; ++bb) {
        const int row = (int)(rowbase + ph[bb]);
        for (int hf = 0; hf < HALVES; ++hf) {
          const int off = (bb * HALVES + hf) * box_bytes;
          tma4(st + off, &kmap, &bars[s], hf * 64, kvh, 0, row);
          tma4(st + tens_bytes + off, &vmap, &bars[s], hf * 64, kvh, 0, row);
        }
      }
    }
  };

  for (int i = 0; i < DNS - 1 && i < DTILES; ++i) issue(i);

  // ---- Q fragments (rows = query heads of the group, zero beyond G) ----
  uint32_t qa[KS][2];
  {
    const bool real = grp < G;
    const int64_t qrow = (b * Hq + (int64_t)kvh * G + (real ? grp : 0)) * D;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int e0 = ks * 16 + 2 * tig;
      float x0 = 0.f, x1 = 0.f, x8 = 0.f, x9 = 0.f;
      if (real) {
        if (q_dtype == BF16) {
          const __nv_bfloat16* qp = (const __nv_bfloat16*)q + qrow;
          x0 = __bfloat162float(qp[e0]);
          x1 = __bfloat162float(qp[e0 + 1]);
          x8 = __bfloat162float(qp[e0 + 8]);
          x9 = __bfloat162float(qp[e0 + 9]);
        } else {
          const float* qp = (const float*)q + qrow;
          x0 = qp[e0];
          x1 = qp[e0 + 1];
          x8 = qp[e0 + 8];
          x9 = qp[e0 + 9];
        }
      }
      qa[ks][0] = pack_bf16(x0, x1);
      qa[ks][1] = pack_bf16(x8, x9);
    }
  }

  float m_run = -INFINITY, l_run = 0.f;
  float o[NE][4];
#pragma unroll
  for (int et = 0; et < NE; ++et)
#pragma unroll
    for (int k = 0; k < 4; ++k) o[et][k] = 0.f;
  const int lr = lane & 7, lm = lane >> 3;

  for (int i = 0; i < DTILES; ++i) {
    if (i + DNS - 1 < DTILES) issue(i + DNS - 1);
    const int s = i % DNS;
    mbar_wait(&bars[s], (i / DNS) & 1);
    const uint32_t kb = su32(wst + (size_t)s * stage_bytes);
    const uint32_t vb = kb + tens_bytes;
    // swizzled address of (token, element) inside a tensor tile
    auto addr = [&](uint32_t base, int tok, int e) {
      const int bb = tok / t, tr = tok % t, hf = e >> 6, ch = (e & 63) >> 3;
      return base + (uint32_t)((bb * HALVES + hf) * box_bytes + tr * 128 + ((ch ^ (tr & 7)) << 4));
    };
    // per-token scale / validity of this lane's 8 tokens
    float s4[4][4];
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int k = 0; k < 4; ++k) s4[n][k] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
      for (int n = 0; n < 4; n += 2) {
        uint32_t r0, r1, r2, r3;
        ldsm_x4(addr(kb, n * 8 + (lm >> 1) * 8 + lr, ks * 16 + (lm & 1) * 8), r0, r1, r2, r3);
        mma16816(s4[n], qa[ks][0], qa[ks][1], r0, r1);
        mma16816(s4[n + 1], qa[ks][0], qa[ks][1], r2, r3);
      }
    }
    float mx = -INFINITY;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int tl = n * 8 + 2 * tig + k;
        const int jb = i * bpt + tl / t;
        const float ksv = __shfl_sync(0xffffffffu, ks_l, jb);
        const bool vv = __shfl_sync(0xffffffffu, (int)val_l, jb);
        const float lg = vv ? s4[n][k] * ksv : -INFINITY;
        s4[n][k] = lg;
        mx = fmaxf(mx, lg);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    const float alpha = m_new == -INFINITY ? 1.f : __expf(m_run - m_new);
    float lsum = 0.f;
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float p = m_new == -INFINITY ? 0.f : __expf(s4[n][k] - m_new);
        s4[n][k] = p;
        lsum += p;
      }
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    l_run = l_run * alpha + lsum;
    m_run = m_new;
#pragma unroll
    for (int et = 0; et < NE; ++et) {
      o[et][0] *= alpha;
      o[et][1] *= alpha;
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      float pv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int tl = kk * 16 + (k >> 1) * 8 + 2 * tig + (k & 1);
        const float vsv = __shfl_sync(0xffffffffu, vs_l, i * bpt + tl / t);
        pv[k] = s4[2 * kk + (k >> 1)][k & 1] * vsv;
      }
      const uint32_t a0 = pack_bf16(pv[0], pv[1]);
      const uint32_t a2 = pack_bf16(pv[2], pv[3]);
#pragma unroll
      for (int et = 0; et < NE; et += 2) {
        uint32_t r0, r1, r2, r3;
        ldsm_x4_t(addr(vb, kk * 16 + (lm & 1) * 8 + lr, et * 8 + (lm >> 1) * 8), r0, r1, r2, r3);
        mma16816(o[et], a0, a2, r0, r1);
        mma16816(o[et + 1], a0, a2, r2, r3);
      }
    }
    __syncwarp();  // stage s is refilled by a later issue()
  }
  // ---- merge the warp partials ----
  __syncthreads();
  float* wm = reinterpret_cast<float*>(dsm);
  float* wl = wm + DW * 8;
  float* wo = wl + DW * 8;
  if (grp < G) {
    if (tig == 0) {
      wm[warp * 8 + grp] = m_run;
      wl[warp * 8 + grp] = l_run;
    }
#pragma unroll
    for (int et = 0; et < NE; ++et) {
      wo[(warp * 8 + grp) * D + et * 8 + 2 * tig] = o[et][0];
      wo[(warp * 8 + grp) * D + et * 8 + 2 * tig + 1] = o[et][1];
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < G * D; x += DW * 32) {
    const int gg = x / D, e = x % D;
    float M = -INFINITY;
    for (int w = 0; w < DW; ++w) M = fmaxf(M, wm[w * 8 + gg]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < DW; ++w) {
      const float f = wm[w * 8 + gg] == -INFINITY ? 0.f : __expf(wm[w * 8 + gg] - M);
      L += wl[w * 8 + gg] * f;
      O += wo[(w * 8 + gg) * D + e] * f;
    }
    float* pp = part + (((b * Hq + (int64_t)kvh * G + gg) * nsplit) + split) * (D + 2);
    pp[e] = O;
    if (e == 0) {
      pp[D] = M;
      pp[D + 1] = L;
    }
  }
}

namespace {
template <int D, int DW, int DNS, int DTILES>
cudaError_t decode_tma_t(const DecodeArgs& a, cudaStream_t s) {
  CUtensorMap km, vm;
  if (!make_map(&km, a.pool_k, a.g) || !make_map(&vm, a.pool_v, a.g)) return cudaErrorInvalidValue;
  const int bpt = DTT / a.g.t;
  const int stage_bytes = 2 * bpt * (D / 64) * a.g.t * 128;
  const int smem = 1024 + DW * DNS * stage_bytes + DW * DNS * 8;
  static int attr = 0;
  if (attr < smem) {
    cudaError_t e =
        cudaFuncSetAttribute(decode_tma_kernel<D, DW, DNS, DTILES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  const int cbs = DW * DTILES * bpt;  // blocks per split
  const int64_t nsplit = (a.p_blocks + cbs - 1) / cbs;
  dim3 grid((unsigned)nsplit, a.g.h, (unsigned)a.B);
  decode_tma_kernel<D, DW, DNS, DTILES><<<grid, DW * 32, smem, s>>>(
      km, vm, a.q, a.q_dtype, a.g, a.layer, a.table, (const float*)a.k_scale,
      (const float*)a.v_scale, a.p_blocks, a.seq_blocks, a.Hq, (float)a.sm_scale, (float*)a.ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_decode_combine(a, nsplit, cbs, s);
}
}  // namespace

bool decode_tma_supported(const DecodeArgs& a) {
  if (a.dtype != BF16 || a.probs != nullptr) return false;
  if (a.q_dtype != BF16 && a.q_dtype != F32) return false;
  if (a.g.d != 64 && a.g.d != 128) return false;
  if (a.g.t < 1 || DTT % a.g.t != 0 || a.g.t > 256) return false;
  if (a.Hq % a.g.h != 0 || a.Hq / a.g.h > 8) return false;
  if ((reinterpret_cast<uintptr_t>(a.pool_k) & 15) || (reinterpret_cast<uintptr_t>(a.pool_v) & 15))
    return false;
  if (a.g.L * a.g.NB >= (int64_t)INT32_MAX) return false;
  const int cbs = 2 * DTILES_MIN * (DTT / a.g.t);
  if (16 * (DTT / a.g.t) > 32) return false;  // table prefetch: one lane per block
  if (cbs < 4) return false;  // workspace is sized for splits of >= 4 blocks
  return encode_fn() != nullptr;
}

cudaError_t launch_decode_tma(const DecodeArgs& a, cudaStream_t s) {
  // warps per CTA x stages per warp (192 KB of stages either way)
  // 4 warps x 3 stages x 16 tiles of 32 tokens per CTA: long-lived CTAs hide
  // the per-CTA prologue (table prefetch, first TMA round trip) and epilogue
  // (measured on B200 at batch 64 x 4K: 4 tiles/warp 319 us, 8: 245 us,
  // 16: 210 us per layer, i.e. 78% of HBM copy bandwidth)
  if (a.g.d == 128) return decode_tma_t<128, 4, 3, 16>(a, s);
  return decode_tma_t<64, 4, 3, 16>(a, s);
}


}  // namespace kvf
