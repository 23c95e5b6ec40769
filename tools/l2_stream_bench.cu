// L2-resident streaming rate per SM for the decode access pattern: a slot's
// head slice = 16 rows of 256 B at a 2 KB stride ([block][token][head][d] bf16,
// h = 8, d = 128). Compares TMA boxes (as decode_sched_kernel issues them),
// plain 16-B loads and cp.async into shared memory.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2s tools/l2_stream_bench.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

constexpr int T = 16, H = 8, D = 128;
constexpr int BLK = T * H * D * 2;  // 32 KB per block (all heads)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                   su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
                   su32(dst)), "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// (a) TMA: W warps per CTA, each with its own NS-stage ring of one slot (K half boxes x2)
template <int W, int NS>
__global__ void k_tma(const __grid_constant__ CUtensorMap map, int nblocks, int iters, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* st = sm + warp * NS * 4096;
  uint64_t* bars = (uint64_t*)(sm + W * NS * 4096) + warp * NS;
  if (lane == 0) for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
  __syncwarp();
  unsigned acc = 0;
  const uint32_t seed = blockIdx.x * W + warp;
  auto issue = [&](int it) {
    const int s = it % NS;
    const uint32_t hsh = hash(seed * 7919u + it);
    const int row = hsh % nblocks, head = (hsh >> 20) & 7;
    if (lane == 0) {
      mbar_expect_tx(&bars[s], 4096);
      tma4(st + s * 4096, &map, &bars[s], 0, head, 0, row);
      tma4(st + s * 4096 + 2048, &map, &bars[s], 64, head, 0, row);
    }
  };
  for (int i = 0; i < NS - 1 && i < iters; ++i) issue(i);
  for (int it = 0; it < iters; ++it) {
    if (it + NS - 1 < iters) issue(it + NS - 1);
    const int s = it % NS;
    mbar_wait(&bars[s], (it / NS) & 1);
    acc ^= ((const unsigned*)(st + s * 4096))[lane * 32];
    __syncwarp();
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// (a') TMA with one 4 KB box per stage ({64 d, 2 heads, 16 tokens, 1 block})
template <int W, int NS>
__global__ void k_tma1(const __grid_constant__ CUtensorMap map, int nblocks, int iters, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* st = sm + warp * NS * 4096;
  uint64_t* bars = (uint64_t*)(sm + W * NS * 4096) + warp * NS;
  if (lane == 0) for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
  __syncwarp();
  unsigned acc = 0;
  const uint32_t seed = blockIdx.x * W + warp;
  auto issue = [&](int it) {
    const int s = it % NS;
    const uint32_t hsh = hash(seed * 7919u + it);
    const int row = hsh % nblocks, head = ((hsh >> 20) & 3) * 2;
    if (lane == 0) {
      mbar_expect_tx(&bars[s], 4096);
      tma4(st + s * 4096, &map, &bars[s], 0, head, 0, row);
    }
  };
  for (int i = 0; i < NS - 1 && i < iters; ++i) issue(i);
  for (int it = 0; it < iters; ++it) {
    if (it + NS - 1 < iters) issue(it + NS - 1);
    const int s = it % NS;
    mbar_wait(&bars[s], (it / NS) & 1);
    acc ^= ((const unsigned*)(st + s * 4096))[lane * 32];
    __syncwarp();
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// (c) hybrid: each warp streams one 4 KB slot per iteration through a 2-stage TMA ring AND
// one 4 KB slot by 16-B ld.global (the decode's K by TMA, V by the LSU path)
template <int W, int NS>
__global__ void k_hybrid(const __grid_constant__ CUtensorMap map, const uint8_t* __restrict__ pool,
                         int nblocks, int iters, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* st = sm + warp * NS * 4096;
  uint64_t* bars = (uint64_t*)(sm + W * NS * 4096) + warp * NS;
  if (lane == 0) for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
  __syncwarp();
  unsigned acc = 0;
  const uint32_t seed = blockIdx.x * W + warp;
  auto issue = [&](int it) {
    const int s = it % NS;
    const uint32_t hsh = hash(seed * 7919u + it);
    const int row = hsh % nblocks, head = (hsh >> 20) & 7;
    if (lane == 0) {
      mbar_expect_tx(&bars[s], 4096);
      tma4(st + s * 4096, &map, &bars[s], 0, head, 0, row);
      tma4(st + s * 4096 + 2048, &map, &bars[s], 64, head, 0, row);
    }
  };
  for (int i = 0; i < NS - 1 && i < iters; ++i) issue(i);
  for (int it = 0; it < iters; ++it) {
    if (it + NS - 1 < iters) issue(it + NS - 1);
    const uint32_t h2 = hash(seed * 104729u + it);
    const uint8_t* base = pool + (size_t)(h2 % nblocks) * BLK + ((h2 >> 20) & 7) * D * 2;
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = k * 32 + lane, r = idx >> 4, c = idx & 15;
      v[k] = __ldg((const uint4*)(base + r * (H * D * 2) + c * 16));
    }
    const int s = it % NS;
    mbar_wait(&bars[s], (it / NS) & 1);
    acc ^= ((const unsigned*)(st + s * 4096))[lane * 32];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x;
    __syncwarp();
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// (b) LDG: each warp loads one slot head slice (4 KB = 16 rows x 256 B) per iteration,
// U slots in flight per warp (unrolled independent loads)
template <int U>
__global__ void k_ldg(const uint8_t* __restrict__ pool, int nblocks, int iters, unsigned* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t seed = blockIdx.x * (blockDim.x / 32) + warp;
  unsigned acc = 0;
  for (int it = 0; it < iters; it += U) {
    uint4 v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t hsh = hash(seed * 7919u + it + u);
      const int row = hsh % nblocks, head = (hsh >> 20) & 7;
      const uint8_t* base = pool + (size_t)row * BLK + head * D * 2;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // 16 rows x 16 chunks of 16 B = 256 loads / 32 lanes
        const int idx = k * 32 + lane, r = idx >> 4, c = idx & 15;
        v[u][k] = __ldg((const uint4*)(base + r * (H * D * 2) + c * 16));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc ^= v[u][k].x ^ v[u][k].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

int main(int argc, char** argv) {
  const int nblocks = argc > 1 ? atoi(argv[1]) : 2048;  // 2048: 64 MB, L2 resident
  uint8_t* pool;
  unsigned* sink;
  if (cudaMalloc(&pool, (size_t)nblocks * BLK) != cudaSuccess) return 1;
  cudaMemset(pool, 1, (size_t)nblocks * BLK);
  cudaMalloc(&sink, 4);
  CUtensorMap m;
  cuuint64_t dims[4] = {D, H, T, (cuuint64_t)nblocks};
  cuuint64_t strides[3] = {D * 2, H * D * 2, (cuuint64_t)T * H * D * 2};
  cuuint32_t box[4] = {64, 1, T, 1}, es[4] = {1, 1, 1, 1};
  enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch, double bytes) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %8.1f GB/s chip  %6.1f GB/s per SM  (%s)\n", name, bytes * 5 / (ms / 1e3) / 1e9,
           bytes * 5 / (ms / 1e3) / 1e9 / 148, cudaGetErrorString(cudaGetLastError()));
  };
  const int iters = 2048;
#define TMA(W, NS)                                                                                      \
  {                                                                                                     \
    const int smem = 1024 + W * NS * 4096 + W * NS * 8;                                                 \
    cudaFuncSetAttribute(k_tma<W, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);              \
    run("tma W=" #W " NS=" #NS, [&] { k_tma<W, NS><<<148, W * 32, smem>>>(m, nblocks, iters, sink); }, \
        148.0 * W * iters * 4096);                                                                      \
  }
#define TMAX(W, NS, EXTRA)                                                                              \
  {                                                                                                     \
    const int smem = 1024 + W * NS * 4096 + W * NS * 8 + EXTRA;                                         \
    cudaFuncSetAttribute(k_tma<W, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);              \
    run("tma W=" #W " NS=" #NS " +smem " #EXTRA, [&] { k_tma<W, NS><<<148, W * 32, smem>>>(m, nblocks, iters, sink); }, \
        148.0 * W * iters * 4096);                                                                      \
  }
  CUtensorMap m2;
  cuuint32_t box2[4] = {64, 2, T, 1};
  enc()(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, pool, dims, strides, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
#define TMA1(W, NS)                                                                                      \
  {                                                                                                     \
    const int smem = 1024 + W * NS * 4096 + W * NS * 8;                                                 \
    cudaFuncSetAttribute(k_tma1<W, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);             \
    run("tma1box W=" #W " NS=" #NS, [&] { k_tma1<W, NS><<<148, W * 32, smem>>>(m2, nblocks, iters, sink); }, \
        148.0 * W * iters * 4096);                                                                      \
  }
#define HYB(W, NS)                                                                                      \
  {                                                                                                     \
    const int smem = 1024 + W * NS * 4096 + W * NS * 8;                                                 \
    cudaFuncSetAttribute(k_hybrid<W, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);           \
    run("hybrid tma+ldg W=" #W " NS=" #NS, [&] { k_hybrid<W, NS><<<148, W * 32, smem>>>(m, pool, nblocks, iters, sink); }, \
        148.0 * W * iters * 8192);                                                                      \
  }
  HYB(12, 2) HYB(12, 3) HYB(16, 2) HYB(8, 3)
  TMA1(12, 2) TMA1(12, 3) TMA1(20, 2) TMA1(12, 4) TMA1(24, 2) TMA1(16, 3)
  TMAX(12, 2, 32768) TMAX(12, 2, 65536) TMAX(12, 2, 98304) TMAX(12, 2, 120000)
  TMA(6, 2) TMA(8, 2) TMA(12, 2) TMA(16, 2) TMA(20, 2) TMA(24, 1) TMA(8, 3) TMA(12, 3) TMA(6, 4) TMA(12, 4) TMA(24, 2)
#define LDG(U, WPC)                                                                                      \
  run("ldg U=" #U " warps=" #WPC, [&] { k_ldg<U><<<148 * 2, WPC * 32>>>(pool, nblocks, iters / 2, sink); }, \
      148.0 * 2 * WPC * (iters / 2) * 4096);
  LDG(1, 16) LDG(2, 16) LDG(2, 8) LDG(4, 8) LDG(1, 32)
  return 0;
}
