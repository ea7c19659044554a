// dequant.cuh -- the tl_dequant test-hook kernel, instantiated per format (build/gen/deq_*.cu).
#pragma once
#include "api_util.cuh"

namespace tl {

// ---------------------------------------------------------------------------------
// dequant hook: thread per (tile, column); the column's words are loaded with the same 16-byte
// vectors and unpacked with the same extract_pair<> the kernels use, then scaled EXACTLY in fp32:
//   ints:   (x & mask) | 0x6400 = 1024 + u*2^P;  HFMA2(x, 2^-P, -(2^(10-P) + z)) = u - z exactly
//   floats: the field placement is value(code) * 2^(bias-15) exactly; * 2^(15-bias) in fp32
template <class F>
__global__ void dequant_kernel(const uint8_t* __restrict__ wt, const __half* __restrict__ scales,
                               const __half* __restrict__ zeros, float* __restrict__ out, int64_t K, int64_t N,
                               int G) {
  const int64_t KT = K / kBK;
  const int64_t tile = blockIdx.x;
  const int nl = threadIdx.x;
  const int64_t nt = tile / KT, kt = tile % KT;
  const int64_t n = nt * kBN + nl;
  const uint8_t* tb = wt + tile * (int64_t)tile_bytes(F::bits);
  uint32_t words[4 * F::bits];
#pragma unroll
  for (int v = 0; v < F::bits; ++v) {
    const uint4 x = ld_nc_v4(tb + (v * 128 + nl) * 16);
    words[4 * v + 0] = x.x;
    words[4 * v + 1] = x.y;
    words[4 * v + 2] = x.z;
    words[4 * v + 3] = x.w;
  }
  static_for<0, 2>([&](auto HH) {
    constexpr int h = decltype(HH)::value;
    uint32_t bw[2 * F::bits];
#pragma unroll
    for (int j = 0; j < 2 * F::bits; ++j) bw[j] = words[tile_word(h, j)];
    static_for<0, 32>([&](auto I) {
      constexpr int i = decltype(I)::value;
      constexpr PairPlan pp = kPlan<F::kind, F::bits, F::exp>.pr[i];
      const int64_t k = kt * kBK + 2 * (32 * h + i);
      const int64_t g = k / G;
      const float s = __half2float(scales[g * N + n]);
      float2 v;
      if constexpr (F::kind != kFloat) {
        float z = (float)(1 << (F::bits - 1));
        if constexpr (F::kind == kUint) z = zeros ? __half2float(zeros[g * N + n]) : 0.f;
        const __half c = __float2half_rn(-(float)(1 << (10 - pp.P)) - z);  // integer < 2048: exact
        const uint32_t x = extract_pair<F, i>(bw, 0x64006400u);
        v = __half22float2(__hfma2(u32_as_h2(x), u32_as_h2(h2_pow2_neg<pp.P>()), __halves2half2(c, c)));
      } else {
        const uint32_t x = extract_pair<F, i>(bw, 0u);
        const float2 r = __half22float2(u32_as_h2(x));
        constexpr float up = (float)(1 << (15 - F::bias));
        v = make_float2(r.x * up, r.y * up);
      }
      out[k * N + n] = v.x * s;          // (value - z) * s is exact in fp32 (reading R9)
      out[(k + 1) * N + n] = v.y * s;
    });
  });
}

template <class F>
void launch_dequant(const uint8_t* wt, const __half* scales, const __half* zeros, float* out, int64_t K, int64_t N,
                    int G, unsigned tiles, cudaStream_t st) {
  dequant_kernel<F><<<tiles, kBN, 0, st>>>(wt, scales, zeros, out, K, N, G);
}

}  // namespace tl
