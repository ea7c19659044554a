// prefill.cuh -- the large-M (prefill) regime: "For the prefill stage,
// quantized weights are decoded to float16, and computations are performed using standard
// f16xf16 matrix multiplication kernels, as computation becomes the bottleneck at this stage"
// (swept at 4096 / 8192 / 12288 tokens).
//
// B200 form: the weight is decoded in column chunks of Nc columns into an fp16 W^T[Nc, K] buffer
// of the caller's workspace (Nc chosen so the chunk, <= 64 MB, stays in the 126 MB L2 between the
// decode and the GEMM that reads it), then a plain cuBLAS f16 x f16 GEMM with fp32 accumulation
// produces Y[:, chunk].  The decode kernel here is this library's: thread = one
// column of a 128 x 128 tile, the layout-v2 extraction + HFMA2 (u - z exactly, as tc2) + HMUL2
// by the group scale (one fp16 rounding, reading R9), and 16-byte stores of the column's 128
// contiguous k values.
#pragma once

#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

// W^T[n0 + n, k] (row stride K) for the n-tiles [nt0, nt0 + ntiles) and every k-tile
template <class F, bool BF>
__global__ void __launch_bounds__(128) dq16_kernel(const uint8_t* __restrict__ wt, const __half* __restrict__ scales,
                                                   const __half* __restrict__ zeros, __half* __restrict__ out,
                                                   int N, int K, int G, int nt0, uint32_t magic) {
  constexpr int B = F::bits;
  const int KT = K / kBK;
  const int kt = blockIdx.x % KT;
  const int ntl = blockIdx.x / KT;
  const int nt = nt0 + ntl;
  const int n = threadIdx.x;
  const int col = nt * kBN + n;
  const uint8_t* tb = wt + ((int64_t)nt * KT + kt) * tile_bytes(B);
  uint32_t words[4 * B];
#pragma unroll
  for (int v = 0; v < B; ++v) {
    const uint4 x = ld_nc_v4(tb + (v * 128 + n) * 16);
    words[4 * v + 0] = x.x;
    words[4 * v + 1] = x.y;
    words[4 * v + 2] = x.z;
    words[4 * v + 3] = x.w;
  }
  __half* dst = out + (int64_t)(ntl * kBN + n) * K + kt * kBK;
  static_for<0, 4>([&](auto CC) {
    constexpr int c = decltype(CC)::value;  // 32-k sub-piece
    constexpr int h = c >> 1;
    const int64_t row = (int64_t)(kt * kBK + c * 32) / G;
    const uint32_t sb = __half_as_ushort(scales[row * N + col]);
    const __half2 s2 = u32_as_h2(sb | (sb << 16));
    const float sf = Act<BF>::to_float(sb);
    uint32_t cp[10];
    if constexpr (F::kind != kFloat) {
      uint32_t zneg;
      if constexpr (F::kind == kUint) {
        const uint32_t zb = zeros ? Act<BF>::neg_zero_h(__half_as_ushort(zeros[row * N + col])) : 0x8000u;
        zneg = zb | (zb << 16);
      } else {
        constexpr uint32_t zb = 0x8000u | ((uint32_t)(B - 1 + 15) << 10);  // -2^(b-1)
        zneg = zb | (zb << 16);
      }
      static_for<0, 10>([&](auto PP) {
        constexpr int P = decltype(PP)::value;
        if constexpr (plan_has_p<F>(P)) {
          constexpr uint32_t k = 0x8000u | ((uint32_t)(25 - P) << 10);  // fp16 -2^(10-P)
          cp[P] = h2_as_u32(__hadd2(u32_as_h2(zneg), u32_as_h2(k | (k << 16))));
        }
      });
    }
    uint32_t bw[2 * B];
#pragma unroll
    for (int j = 0; j < 2 * B; ++j) bw[j] = words[tile_word(h, j)];
    uint32_t r[16];
    static_for<0, 16>([&](auto II) {
      constexpr int ii = decltype(II)::value;
      constexpr int i = (c & 1) * 16 + ii;
      __half2 v;  // exact
      if constexpr (F::kind != kFloat) {
        constexpr int P = kPlan<F::kind, F::bits, F::exp>.pr[i].P;
        const uint32_t x = extract_pair<F, i>(bw, magic);
        v = __hfma2(u32_as_h2(x), u32_as_h2(h2_pow2_neg<P>()), u32_as_h2(cp[P]));
      } else {
        constexpr uint32_t e = (uint32_t)(30 - F::bias) << 10;  // 2^(15-bias)
        const uint32_t x = extract_pair<F, i>(bw, 0u);
        v = __hmul2(u32_as_h2(x), u32_as_h2(e | (e << 16)));
      }
      if constexpr (!BF) {
        r[ii] = h2_as_u32(__hmul2(v, s2));
      } else {
        const float2 f = __half22float2(v);
        const __nv_bfloat162 b = __floats2bfloat162_rn(f.x * sf, f.y * sf);
        r[ii] = *reinterpret_cast<const uint32_t*>(&b);
      }
    });
    uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) d4[q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
  });
}

template <class F>
tl_status launch_dq16(const uint8_t* wt, const __half* scales, const __half* zeros, __half* out, int N, int K, int G,
                      int nt0, int ntiles, bool bf, cudaStream_t st) {
  if (bf) dq16_kernel<F, true><<<ntiles * (K / kBK), 128, 0, st>>>(wt, scales, zeros, out, N, K, G, nt0, 0x64006400u);
  else dq16_kernel<F, false><<<ntiles * (K / kBK), 128, 0, st>>>(wt, scales, zeros, out, N, K, G, nt0, 0x64006400u);
  return check_launch("dq16_kernel");
}

}  // namespace tl
