// peer.cuh -- SURVEY §8(f) row f3: the gathered-output variant of the column-sharded matmul with the
// all-gather fused into the epilogue.  Output column n depends only on W[:, n], so
// rank r computes its column block [n0, n1) alone; instead of an all-gather after the matmul, the
// epilogue stores every finished Y element into the local gathered buffer AND into each peer's
// gathered buffer over NVLink (peer-mapped device addresses), and the CTA that finishes last
// releases one arrival flag per peer at system scope.  The consumer waits on its flags
// (tl_gather_wait) before it reads the gathered Y.
#pragma once

#include <cstdint>

namespace tl {

constexpr int kMaxPeers = 7;  // an 8-GPU NVSwitch box: up to 7 other ranks

struct PeerOut {
  unsigned short* y[kMaxPeers];  // peer i's gathered Y at THIS rank's column offset (row stride = ldy)
  uint32_t* flag[kMaxPeers];     // peer i's arrival counter for this rank (+1 per call)
  uint32_t* done;                // local CTA-arrival counter of this launch (workspace, self-resetting)
  int n;                         // number of peers (0: plain local output)
  int signal;                    // 1 on the launch that completes the call (tc2 chunks M by 128)
};

// row-parallel reduce-scatter: the ranks' partials at this rank's column block (peer-mapped)
struct PeerParts {
  const uint16_t* p[kMaxPeers + 1];
  int n;
};

// Replicate one output element / 4 consecutive elements into every peer's gathered buffer.
__device__ __forceinline__ void peer_store(const PeerOut& po, int64_t off, unsigned short v) {
  for (int i = 0; i < po.n; ++i) po.y[i][off] = v;
}
__device__ __forceinline__ void peer_store4(const PeerOut& po, int64_t off, uint2 v) {
  for (int i = 0; i < po.n; ++i) *reinterpret_cast<uint2*>(po.y[i] + off) = v;
}

// Called by ONE thread of each CTA after a CTA-wide barrier that follows every Y store of the CTA
// (so the barrier orders all of them before this thread's release).  Each CTA makes its stores
// visible at system scope and arrives on the local counter (acq_rel, system scope); the last of
// the `grid` CTAs resets the counter and releases +1 on every peer's flag for this rank.  The
// release is cumulative: every CTA's peer stores happen-before it.
__device__ __forceinline__ void peer_signal(const PeerOut& po, unsigned grid) {
  if (po.n == 0) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (!po.signal) return;
  uint32_t prev;
  asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(po.done) : "memory");
  if (prev == grid - 1) {
    *po.done = 0;  // the next launch is ordered after this one by the stream
    for (int i = 0; i < po.n; ++i)
      asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(po.flag[i]) : "memory");
  }
}

}  // namespace tl
