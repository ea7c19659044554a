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

// the decode kernel's consumer pattern: R tiles per stage, 4 groups x 4 warps, group g takes tiles
// g, g+4, ... and each of its warps waits for the tile's stage and arrives on the stage's empty
// barrier once per TILE (4*R arrivals per stage); `mode` 1: one arrival per group per tile (R*4/4)
template <int NS>
__global__ void group_kernel(const uint8_t* src, size_t bytes_per_cta, int stage_bytes, int R, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * stage_bytes);
  uint64_t* empty = full + NS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mode ? R : 4 * R);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * bytes_per_cta;
  const int Q = (int)(bytes_per_cta / stage_bytes);  // stages
  const int T = Q * R;                                // tiles
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int q = 0; q < Q; ++q) {
        const int s = q % NS;
        if (q >= NS) mbar_wait(&empty[s], ((q / NS) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        tma_bulk_g2s(sm + s * stage_bytes, base + (size_t)q * stage_bytes, stage_bytes, &full[s], pol);
      }
    }
  } else if (warp >= 4 && warp < 20) {
    const int g = (warp - 4) >> 2;
    for (int t = g; t < T; t += 4) {
      const int q = t / R, s = q % NS;
      mbar_wait(&full[s], (q / NS) & 1);
      if (mode) {
        named_bar_sync(1 + g, 128);
        if ((warp & 3) == 0 && lane == 0) mbar_arrive(&empty[s]);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
  }
  __syncthreads();
}

template <int NS>
static void run_group(uint8_t* buf, size_t total, int stage, int R, int mode, cudaEvent_t e0, cudaEvent_t e1) {
  const int grid = 148;
  size_t per = total / grid;
  per -= per % stage;
  const int smem = NS * stage + 2 * NS * 8 + 64;
  cudaFuncSetAttribute(group_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    group_kernel<NS><<<grid, 640, smem>>>(buf, per, stage, R, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("groups NS=%d stage=%d R=%d mode=%d per-CTA %zu KB: %.1f GB/s %s\n", NS, stage, R, mode, per >> 10,
         (double)per * grid / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

// short streams as the decode kernel sees them: per-CTA ranges of 128 KB ... 4 MB (148 CTAs), 12 KB
// stages x 11 (u1..u3-like) and 16 KB x 10 (u8-like); the slope between sizes removes launch costs
static void short_streams(uint8_t* buf, unsigned long long* cyc, cudaEvent_t e0, cudaEvent_t e1) {
  for (int stage : {12288, 16384})
    for (size_t per : {(size_t)128 << 10, (size_t)256 << 10, (size_t)512 << 10, (size_t)1 << 20, (size_t)4 << 20}) {
      const size_t total = per * 148;
      if (stage == 12288) run<11>(buf, total, cyc, stage, 1, 1, e0, e1);
      else run<10>(buf, total, cyc, stage, 1, 1, e0, e1);
      printf("   ^ per-CTA stream %zu KB\n", per >> 10);
    }
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
  if (getenv("PROBE_GROUPS")) {
    for (size_t per : {(size_t)256 << 10, (size_t)4 << 20})
      for (int mode : {0, 1}) {
        run_group<11>(buf, per * 148, 12288, 6, mode, e0, e1);  // u1-like: 6 tiles of 2 KB per stage
        run_group<11>(buf, per * 148, 12288, 2, mode, e0, e1);  // u3-like: 2 tiles of 6 KB
        run_group<10>(buf, per * 148, 16384, 1, mode, e0, e1);  // u8-like: 1 tile of 16 KB
      }
    return 0;
  }
  if (getenv("PROBE_SHORT")) {
    short_streams(buf, cyc, e0, e1);
    return 0;
  }
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
