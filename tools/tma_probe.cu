// tma_probe.cu -- how fast can one CTA per SM stream HBM through cp.async.bulk?
// Each CTA streams its own contiguous range of a large buffer through an NS-stage smem
// ring; consumers only wait for the data and release the stage.  Variants: bytes per
// stage, bulk copies per stage (chunks), number of issuing lanes, CTAs per SM.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace tl;

template <int NS>
__global__ void stream_kernel(const uint8_t* src, size_t bytes_per_cta, int stage_bytes, int chunks, int issuers,
                              unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * stage_bytes);
  uint64_t* empty = full + NS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * bytes_per_cta;
  const int T = (int)(bytes_per_cta / stage_bytes);
  const int chunk = stage_bytes / chunks;
  long long t0 = clock64();
  if (warp == 0) {
    const uint64_t pol = policy_evict_first();
    for (int t = 0; t < T; ++t) {
      const int s = t % NS;
      if (t >= NS) mbar_wait(&empty[s], ((t / NS) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], stage_bytes);
      __syncwarp();
      for (int c = lane; c < chunks; c += 32) {
        if (lane < issuers || issuers >= 32)
          tma_bulk_g2s(sm + s * stage_bytes + c * chunk, base + (size_t)t * stage_bytes + c * chunk, chunk, &full[s],
                       pol);
      }
      if (issuers < 32 && chunks > issuers) {
        // remaining chunks by lane 0
        if (lane == 0)
          for (int c = 32; c < chunks; ++c)
            tma_bulk_g2s(sm + s * stage_bytes + c * chunk, base + (size_t)t * stage_bytes + c * chunk, chunk,
                         &full[s], pol);
      }
      __syncwarp();
    }
  } else {
    for (int t = 0; t < T; ++t) {
      const int s = t % NS;
      mbar_wait(&full[s], (t / NS) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  const size_t total = (size_t)2 << 30;  // 2 GiB
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 4096 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int stage, chunks, issuers, ctas_per_sm; };
  std::vector<Cfg> cfgs = {{8192, 1, 1, 1}, {8192, 4, 4, 1},   {8192, 8, 8, 1},   {16384, 1, 1, 1},
                           {16384, 8, 8, 1}, {32768, 1, 1, 1}, {32768, 16, 16, 1}, {8192, 1, 1, 2},
                           {8192, 1, 1, 4}, {4096, 1, 1, 1},  {2048, 1, 1, 1},   {16384, 1, 1, 2}};
  for (auto c : cfgs) {
    const int grid = 148 * c.ctas_per_sm;
    size_t per = total / grid;
    per -= per % c.stage;
    const int NS = 8;
    const int smem = NS * c.stage + 2 * NS * 8 + 64;
    cudaFuncSetAttribute(stream_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      stream_kernel<8><<<grid, 160, smem>>>(buf, per, c.stage, c.chunks, c.issuers, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaError_t err = cudaGetLastError();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stage=%6d chunks=%2d issuers=%2d ctas/SM=%d smem=%6d : %.1f GB/s %s\n", c.stage, c.chunks, c.issuers,
           c.ctas_per_sm, smem, (double)per * grid / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
