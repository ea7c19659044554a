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

// ---- row-parallel (K-sharded) variant: NVLink reduce-scatter over peer memory (row f3) ----------
namespace tl {

// One thread per pending signal: +1 (release, system scope) on every peer's arrival flag for this
// rank, after all prior work of the stream (kernel boundary) -- "my partial is complete".
__global__ void signal_peers_kernel(PeerOut po) {
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int i = 0; i < po.n; ++i) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(po.flag[i]) : "memory");
  }
}

// Y[m, c] = sum_{q = 0 .. P-1} parts[q][m, c] in fp32, in rank order (deterministic), rounded once;
// 8 columns (16 bytes) per thread per row, grid-stride.  parts[q] are peer-mapped addresses of the
// ranks' partials at this rank's column block (row stride ldp).
template <bool BF>
__global__ void __launch_bounds__(256) reduce_scatter_kernel(PeerParts pp, int M, int N, int64_t ldp,
                                                             uint16_t* __restrict__ Y, int64_t ldy) {
  const int vpr = N / 8;
  const int64_t total = (int64_t)M * vpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / vpr;
    const int v = (int)(i - m * vpr);
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int q = 0; q < pp.n; ++q) {
      const uint4 x = __ldcv(reinterpret_cast<const uint4*>(pp.p[q] + m * ldp + (int64_t)v * 8));
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[2 * j] += Act<BF>::to_float((uint16_t)(w[j] & 0xFFFFu));
        acc[2 * j + 1] += Act<BF>::to_float((uint16_t)(w[j] >> 16));
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      o[j] = (uint32_t)Act<BF>::from_float(acc[2 * j]) | ((uint32_t)Act<BF>::from_float(acc[2 * j + 1]) << 16);
    *reinterpret_cast<uint4*>(Y + m * ldy + (int64_t)v * 8) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace tl

extern "C" tl_status tl_signal_peers(uint32_t* const* flag_peers, int32_t npeers, void* stream) {
  if (npeers < 0 || npeers > kMaxPeers) return fail(TL_EINVAL_SHAPE, "npeers=%d outside [0, %d]", npeers, kMaxPeers);
  if (npeers == 0) return TL_OK;
  if (!flag_peers) return fail(TL_ENULL, "tl_signal_peers: NULL flag array");
  PeerOut po{};
  for (int i = 0; i < npeers; ++i) {
    if (!flag_peers[i]) return fail(TL_ENULL, "tl_signal_peers: NULL flag %d", i);
    if (reinterpret_cast<uintptr_t>(flag_peers[i]) & 3u) return fail(TL_EALIGN, "flag %d not 4-byte aligned", i);
    po.flag[i] = flag_peers[i];
  }
  po.n = npeers;
  signal_peers_kernel<<<1, 32, 0, as_stream(stream)>>>(po);
  return check_launch("signal_peers_kernel");
}

extern "C" tl_status tl_reduce_scatter_peer(tl_atype a, const void* const* parts, int32_t nranks, int64_t M,
                                            int64_t N, int64_t ldp, void* Y, int64_t ldy, void* stream) {
  if (a != TL_ACT_F16 && a != TL_ACT_BF16) return fail(TL_EUNSUPPORTED, "partials are fp16 or bf16 (atype %d)", (int)a);
  if (nranks < 1 || nranks > kMaxPeers + 1) return fail(TL_EINVAL_SHAPE, "nranks=%d outside [1, %d]", nranks, kMaxPeers + 1);
  if (M < 0 || N <= 0 || N % 8 || ldp < N || ldy < N || ldp % 8 || ldy % 8)
    return fail(TL_EINVAL_SHAPE, "M=%lld N=%lld ldp=%lld ldy=%lld (N, ldp, ldy multiples of 8, ld >= N)",
                (long long)M, (long long)N, (long long)ldp, (long long)ldy);
  if (M == 0) return TL_OK;
  if (!parts || !Y) return fail(TL_ENULL, "tl_reduce_scatter_peer: NULL pointer");
  PeerParts pp{};
  for (int q = 0; q < nranks; ++q) {
    if (!parts[q]) return fail(TL_ENULL, "tl_reduce_scatter_peer: NULL partial %d", q);
    if (!aligned16(parts[q])) return fail(TL_EALIGN, "partial %d not 16-byte aligned", q);
    pp.p[q] = reinterpret_cast<const uint16_t*>(parts[q]);
  }
  pp.n = nranks;
  if (!aligned16(Y)) return fail(TL_EALIGN, "Y not 16-byte aligned");
  const int64_t vecs = M * (N / 8);
  int blocks = (int)((vecs + 255) / 256);
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (a == TL_ACT_BF16)
    reduce_scatter_kernel<true><<<blocks, 256, 0, as_stream(stream)>>>(pp, (int)M, (int)N, ldp,
                                                                       reinterpret_cast<uint16_t*>(Y), ldy);
  else
    reduce_scatter_kernel<false><<<blocks, 256, 0, as_stream(stream)>>>(pp, (int)M, (int)N, ldp,
                                                                        reinterpret_cast<uint16_t*>(Y), ldy);
  return check_launch("reduce_scatter_kernel");
}
