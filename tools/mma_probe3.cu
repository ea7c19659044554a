// mma_probe3.cu -- tensor-pipe cost of one 128x128 weight tile the way the decode kernel issues it:
// kind::f16 = 8 back-to-back MMAs (K = 16) reading a fresh 64-column W^T slot from TMEM, kind::i8 =
// 4 MMAs (K = 32) reading a fresh 32-column slot; one tcgen05.commit per tile; N = 16 or 32.
// Slots rotate over NW, accumulators over 2 blocks.  Reports SM cycles per tile.
#include <cstdio>

#include "ptx.cuh"

using namespace tl;

__device__ __forceinline__ uint64_t sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int KIND, int N, int NW>
__global__ void tile_kernel(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (warp == 0 && elect_one()) {
    constexpr uint32_t cols = KIND ? 32 : 64;
    constexpr uint32_t idesc = KIND ? ((2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24))
                                    : ((1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24));
    const uint64_t bd = sw128(smem_u32(sm));
    int g = 0;
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + 448 + (t & 1) * 32;
      const uint32_t aw = tmem + g * cols;
      if constexpr (KIND) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(aw + j * 8), "l"(bd + (uint64_t)(2 * j)), "r"(idesc), "r"(1u));
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(aw + j * 8), "l"(bd + (uint64_t)((j >> 2) * 128 + (j & 3) * 2)), "r"(idesc), "r"(1u));
      }
      tc_commit(&bar);
      if (++g == NW) g = 0;
    }
  }
  __syncwarp();
  if (warp == 0) mbar_wait(&bar, (uint32_t)(tiles - 1) & 1);
  tc_fence_before();
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int KIND, int N, int NW>
void run(long long* d) {
  auto k = tile_kernel<KIND, N, NW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 + 1024);
  const int tiles = 4096;
  k<<<148, 128, 8192 + 1024>>>(tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s N=%d NW=%d: %.1f cycles per 128x128 tile  %s\n", KIND ? "kind::i8 " : "kind::f16", N, NW,
         (double)mx / tiles, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 4096);
  // commits wait only at the end: this is the pipe's own rate (the tile's MMAs back to back)
  run<0, 16, 5>(d);
  run<0, 32, 5>(d);
  run<0, 16, 1>(d);
  run<1, 16, 7>(d);
  run<1, 32, 7>(d);
  run<1, 16, 1>(d);
  return 0;
}
