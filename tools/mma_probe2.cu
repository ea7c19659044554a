// mma_probe2.cu -- tcgen05.mma (kind::f16, K=16) dispatch rate vs M (64/128), N (16..256),
// CTAs per SM (1/2, each owning 512/cps TMEM columns) and issuing warps per CTA (1/2, each into
// its own accumulators).  Reports the SM-wide cycles per MMA: if two issuers halve it, the
// single-thread floor is an issue-side latency, not tensor-pipe occupancy.
#include <cstdio>
#include <cstdlib>

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

// kind: 0 = kind::f16 (K = 16), 1 = kind::i8 (K = 32); fresh: the TS A operand cycles over 32
// different 8-column TMEM chunks (as the decode kernel's W^T slots), else one fixed chunk
__global__ void mma_kernel(int M, int N, int reps, int ncols, int issuers, int ts, long long* out, int kind = 0,
                           int fresh = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A: 128 rows x 128 B, B: 256 rows x 128 B
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&slot, ncols);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (warp < issuers) {
    const uint32_t idesc = kind ? ((2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
                                : ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24));
    const uint32_t abase = smem_u32(sm), bbase = smem_u32(sm + 16384);
    // accumulator region of this issuer: N columns; A (TS) operand: 8 columns after all accumulators
    const uint32_t acc = tmem + warp * N;
    const uint32_t aop = tmem + issuers * N + warp * 8;
    if (elect_one()) {
      for (int r = 0; r < reps; r += 4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t bd = sw128(bbase + j * 32);
          if (ts && kind) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(acc),
                "r"(fresh ? tmem + 256 + ((r + j) & 31) * 8 : aop), "l"(bd), "r"(idesc), "r"(1u));
          } else if (ts) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(acc),
                "r"(fresh ? tmem + 256 + ((r + j) & 31) * 8 : aop), "l"(bd), "r"(idesc), "r"(1u));
          } else {
            const uint64_t ad = sw128(abase + j * 32);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc),
                "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
          }
        }
      }
      tc_commit(&bar[warp]);
    }
    __syncwarp();
    mbar_wait(&bar[warp], 0);
  }
  tc_fence_before();
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) tmem_dealloc(tmem, ncols);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 4096);
  const int smem = 49152 + 1024;
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // fresh-A TS operands (the decode kernel's case): kind::f16 vs kind::i8, one issuer, 1 CTA/SM
  for (int kind = 0; kind < 2; ++kind)
    for (int fresh = 0; fresh < 2; ++fresh)
      for (int N : {16, 32, 64, 128}) {
        const int reps = 2048;
        mma_kernel<<<148, 128, smem>>>(128, N, reps, 512, 1, 1, d, kind, fresh);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("TS %s M=128 N=%3d A=%s: %.1f cycles per MMA (%.1f weights/clk)  %s\n", kind ? "i8 " : "f16", N,
               fresh ? "fresh" : "fixed", (double)mx / reps, (kind ? 4096.0 : 2048.0) * reps / mx,
               e == cudaSuccess ? "ok" : cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
      }
  if (getenv("PROBE_ALL") == nullptr) return 0;
  for (int ts = 1; ts >= 0; --ts)
    for (int M : {128, 64})
      for (int N : {16, 32, 64, 128, 256})
        for (int cps : {1, 2})
          for (int iss : {1, 2}) {
            const int ncols = 512 / cps;
            if (iss * N + iss * 8 > ncols) continue;
            const int reps = 2048;
            const int grid = 148 * cps;
            mma_kernel<<<grid, 128, smem>>>(M, N, reps, ncols, iss, ts, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[296];
            cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            const double per = (double)mx / ((double)reps * iss * cps);
            printf("%s M=%3d N=%3d ctas/SM=%d issuers/CTA=%d: %.1f SM-cycles per MMA (%.0f MAC/clk/SM)  %s\n",
                   ts ? "TS" : "SS", M, N, cps, iss, per, (double)M * N * 16 / per,
                   e == cudaSuccess ? "ok" : cudaGetErrorString(e));
            if (e != cudaSuccess) return 1;
          }
  return 0;
}
