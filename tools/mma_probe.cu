// mma_probe.cu -- cycles per tcgen05.mma.cta_group::1.kind::f16 (M=128, K=16) for
// A from TMEM ("TS") vs A from shared memory ("SS"), for several N.
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

__global__ void mma_kernel(int N, int ts, int reps, int nd, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A: 128 rows x 128 B (16 KB), B: 256 rows x 128 B (32 KB)
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
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
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t abase = smem_u32(sm), bbase = smem_u32(sm + 16384);
    uint64_t bd[4], ad[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      bd[j] = sw128(bbase + j * 32);
      ad[j] = sw128(abase + j * 32);
    }
    long long t0 = clock64();
    if (elect_one()) {
      for (int r = 0; r < reps; r += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (ts) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + (j % nd) * N),
                "r"(tmem + 256 + j * 8), "l"(bd[j & 3]), "r"(idesc), "r"(1u));
          } else {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (j % nd) * N),
                "l"(ad[j & 3]), "l"(bd[j & 3]), "r"(idesc), "r"(1u));
          }
        }
      }
      tc_commit(&bar);
    }
    __syncwarp();
    long long t1 = clock64();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024);
  for (int ts = 1; ts >= 0; --ts)
    for (int N : {16, 32, 64, 128})
      for (int nd : {1, 2, 4, 8}) {
        if (nd * N > 256) continue;
        const int reps = 4096;
        const int grid = 148;
        mma_kernel<<<grid, 128, 49152 + 1024>>>(N, ts, reps, nd, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%s N=%3d independent accumulators=%d: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n",
               ts ? "TS" : "SS", N, nd, (double)h[0] / reps, (double)h[1] / reps,
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
      }
  return 0;
}
