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

template <int NS>
static void run(uint8_t* buf, size_t total, unsigned long long* cyc, int stage, int chunks, int ctas_per_sm,
                cudaEvent_t e0, cudaEvent_t e1) {
  const int grid = 148 * ctas_per_sm;
  size_t per = total / grid;
  per -= per % stage;
  const int smem = NS * stage + 2 * NS * 8 + 64;
  if (smem > 227 * 1024) return;
  cudaFuncSetAttribute(stream_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    stream_kernel<NS><<<grid, 160, smem>>>(buf, per, stage, chunks, chunks, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  printf("NS=%2d stage=%6d chunks=%d ctas/SM=%d smem=%6d in-flight/SM=%6d : %.1f GB/s %s\n", NS, stage, chunks,
         ctas_per_sm, smem, NS * stage * ctas_per_sm, (double)per * grid / (best * 1e-3) / 1e9,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
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
  for (int stage : {2560, 6656, 12544, 16896, 13312}) {
    for (int chunks : {1, 2}) {
      run<8>(buf, total, cyc, stage, chunks, 1, e0, e1);
      run<16>(buf, total, cyc, stage, chunks, 1, e0, e1);
      run<24>(buf, total, cyc, stage, chunks, 1, e0, e1);
      run<32>(buf, total, cyc, stage, chunks, 1, e0, e1);
    }
  }
  return 0;
}
