// tmem_probe.cu -- on-chip bandwidth of the decode kernel's W^T traffic: 16 warps storing 16-column
// chunks into tensor memory (tcgen05.st.32x32b.x16, 2 KB per warp-instruction), alone and with one
// thread concurrently issuing TS-form kind::f16 MMAs that read the stored columns (8 per 64-column
// slot, as the decode kernel).  Reports SM-wide bytes per cycle.
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

__global__ void __launch_bounds__(640, 1) probe(int iters, int with_mma, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4096 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
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
  long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (warp >= 4) {
    // 16 writer warps: warp w writes lane quarter (w & 3), 16-column chunk (w >> 2) of a 64-column
    // slot; slots rotate over 4 (columns 0..255)
    const int dw = warp - 4;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = 0x3c003c00u + i;
    for (int it = 0; it < iters; ++it) {
      const uint32_t a = tmem + lane_off + (it & 3) * 64 + (dw >> 2) * 16;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
          : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else if (warp == 1 && with_mma) {
    if (elect_one()) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t bd = sw128(smem_u32(sm));
      // one 8-MMA tile per 4 writer iterations (= one 64-column slot written), A from the slots
      for (int it = 0; it < iters / 4; ++it) {
        const uint32_t aw = tmem + (it & 3) * 64;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
              "r"(aw + j * 8), "l"(bd + (uint64_t)((j >> 2) * 128 + (j & 3) * 2)), "r"(idesc), "r"(1u));
      }
      tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  long long t1 = clock64();
  long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) {
    out[blockIdx.x] = t1 - t0;
    out[148 + blockIdx.x] = g1 - g0;
  }
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 296);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  const int iters = 4096;
  for (int with_mma = 0; with_mma < 2; ++with_mma) {
    probe<<<148, 640, 8192>>>(iters, with_mma, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[296];
    cudaMemcpy(h, d, 8 * 296, cudaMemcpyDeviceToHost);
    long long mx = 0, gx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    for (int i = 148; i < 296; ++i) gx = h[i] > gx ? h[i] : gx;
    printf("max clock64 cycles %lld, globaltimer %lld ns\n", mx, gx);
    const double bytes = 16.0 * iters * 2048.0;  // 16 warps x iters x 2 KB
    printf("STTM %s: %.1f B/clk/SM written (%.0f cycles per 32 KB W^T tile)  %s\n",
           with_mma ? "+ TS MMAs reading it" : "alone", bytes / mx, 32768.0 / (bytes / mx),
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  }
  return 0;
}
