// gather.cu -- SURVEY §8(f) row f3: the gathered-output column-sharded matmul over NVLink peer memory
// (peer.cuh has the fused epilogue).  Kernels here: the replicate-and-signal kernel for the families
// whose epilogue is not fused (CUDA-core GEMV, prefill GEMM) and the consumer-side flag wait.
#include <cstdlib>

#include "paths.cuh"

namespace tl {

// Replicates Y [M, N] (row stride ldy, fp16/bf16 bits) into every peer's gathered buffer, 16 bytes per
// thread per row segment, then signals like the fused epilogue.  Launched after the matmul in stream
// order (so every element of Y is final).
__global__ void __launch_bounds__(256) gather_push_kernel(PeerOut po, const uint16_t* __restrict__ Y, int64_t ldy,
                                                          int M, int N) {
  const int vpr = N / 8;  // 16-byte vectors per row (N % 128 == 0)
  const int64_t total = (int64_t)M * vpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / vpr;
    const int v = (int)(i - m * vpr);
    const int64_t off = m * ldy + (int64_t)v * 8;
    const uint4 x = *reinterpret_cast<const uint4*>(Y + off);
    for (int q = 0; q < po.n; ++q) *reinterpret_cast<uint4*>(po.y[q] + off) = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) peer_signal(po, gridDim.x);
}

tl_status gather_push(const PeerOut& po, const __half* Y, int64_t ldy, int64_t M, int64_t N, cudaStream_t st) {
  const int64_t vecs = M * (N / 8);
  int blocks = (int)((vecs + 255) / 256);
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  gather_push_kernel<<<blocks, 256, 0, st>>>(po, reinterpret_cast<const uint16_t*>(Y), ldy, (int)M, (int)N);
  return check_launch("gather_push_kernel");
}

// One thread per other rank spins (acquire, system scope) until that rank's arrival counter reaches
// `epoch` (wrap-safe), with a bound: after timeout_ns the kernel traps, so a missing peer surfaces as
// a launch failure instead of a hang.
__global__ void gather_wait_kernel(const uint32_t* flags, int nranks, int self, uint32_t epoch, long long timeout_ns) {
  const int q = threadIdx.x;
  if (q >= nranks || q == self) return;
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q) : "memory");
    if ((int32_t)(v - epoch) >= 0) break;
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) __trap();
    __nanosleep(64);
  }
}

}  // namespace tl

using namespace tl;

extern "C" tl_status tl_gather_wait(const uint32_t* flags, int32_t nranks, int32_t self, uint32_t epoch,
                                    void* stream) {
  if (nranks < 1 || nranks > kMaxPeers + 1 || self < 0 || self >= nranks)
    return fail(TL_EINVAL_SHAPE, "tl_gather_wait: nranks=%d self=%d (1 <= nranks <= %d)", nranks, self,
                kMaxPeers + 1);
  if (!flags) return fail(TL_ENULL, "tl_gather_wait: NULL flags");
  if (nranks == 1) return TL_OK;
  const char* e = getenv("TL_GATHER_TIMEOUT_MS");
  const long long ms = e ? atoll(e) : 10000;
  gather_wait_kernel<<<1, 32, 0, as_stream(stream)>>>(flags, nranks, self, epoch, ms * 1000000ll);
  return check_launch("gather_wait_kernel");
}
