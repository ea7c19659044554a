// dequant.cuh -- the tl_dequant test-hook kernel, instantiated per format (build/gen/deq_*.cu).
#pragma once
#include "api_util.cuh"

namespace tl {

// ---------------------------------------------------------------------------------
// dequant hook: thread per (tile, column); the column run's segment words are loaded with
// the same 16-byte vectors and unpacked with the same pair_value<> the tensor-core
// dequant warps use, then scaled EXACTLY in fp32.
template <class F>
__global__ void dequant_kernel(const uint8_t* __restrict__ wt, const __half* __restrict__ scales,
                               const __half* __restrict__ zeros, float* __restrict__ out, int64_t K, int64_t N,
                               int G, uint32_t magic) {
  const int64_t KT = K / kBK;
  const int64_t tile = blockIdx.x;
  const int nl = threadIdx.x;
  const int64_t nt = tile / KT, kt = tile % KT;
  const int64_t n = nt * kBN + nl;
  const uint8_t* tb = wt + tile * (int64_t)tile_bytes(F::bits);
  uint32_t words[4 * F::bits];
#pragma unroll
  for (int s = 0; s < F::nseg; ++s) {
    const int w = seg_width(F::bits, s), base = seg_base(F::bits, s);
#pragma unroll
    for (int v = 0; v < w; ++v) {
      const uint4 x = ld_nc_v4(tb + 2048 * base + (v * 128 + nl) * 16);
      words[4 * base + 4 * v + 0] = x.x;
      words[4 * base + 4 * v + 1] = x.y;
      words[4 * base + 4 * v + 2] = x.z;
      words[4 * base + 4 * v + 3] = x.w;
    }
  }
  PairConsts pc;
  pc.magic = magic;
  int gcur = -1;
  float s = 0.f;
  static_for<0, 64>([&](auto I) {
    constexpr int i = decltype(I)::value;
    const int64_t k = kt * kBK + 2 * i;
    const int g = (int)(k / G);
    if (g != gcur) {
      gcur = g;
      s = __half2float(scales[(int64_t)g * N + n]);
      float z = 0.f;
      if (F::kind == kUint && zeros) z = __half2float(zeros[(int64_t)g * N + n]);
      if (F::kind == kInt) z = (float)(1 << (F::bits - 1));
      make_pair_consts<F>(pc, z);
    }
    const float2 v = __half22float2(pair_value<F, i>(words, pc));
    out[k * N + n] = v.x * s;          // (value - z) * s is exact in fp32 (reading R9)
    out[(k + 1) * N + n] = v.y * s;
  });
}

template <class F>
void launch_dequant(const uint8_t* wt, const __half* scales, const __half* zeros, float* out, int64_t K, int64_t N,
                    int G, unsigned tiles, cudaStream_t st) {
  dequant_kernel<F><<<tiles, kBN, 0, st>>>(wt, scales, zeros, out, K, N, G, 0x64006400u);
}

}  // namespace tl
