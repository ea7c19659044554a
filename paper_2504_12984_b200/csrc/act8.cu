// act8.cu -- SURVEY §8 row f4: int8 activations (A8Wx) and microscaling (MX) scales.
//
// PAPER.md:518 "operand A can have data types with 32, 16, or 8 bits ... Standard data types such as
// float32, float16, and int8 are supported"; "we also support bfloat16 and int8".
// Reading R24: an int8 activation is the integer it encodes; the product is the same plain definition
// Y[m,n] = fp16(sum_k A[m,k] * w[k,n]) with fp32 accumulation.  Every int8 value is an fp16 integer
// (|a| <= 128 < 2^11), so the staging kernel below converts A EXACTLY into an fp16 copy in the
// workspace and the fp16 kernel families run unchanged on it (row f4).
//
// PAPER.md:585 "Microscaling data types can be thought as a more fine-grained quantization thus we
// could also support it".  Reading R25: an MX block is a group of 32 weights along K sharing one
// E8M0 scale 2^(e-127) (the element formats fp4 e2m1, fp6 e2m3 / e3m2 and fp8 e4m3 are kernel
// formats; MXINT8 is int8 with an implicit 2^-6, passed as exp_adjust = -6).  tl_mx_scales_to_f16
// converts the E8M0 codes once, at weight-preparation time, into the library's fp16 group scales
// (G = 32), exactly whenever 2^(e-127+exp_adjust) is an fp16 number (2^-24 .. 2^15); every other
// code -- and the E8M0 NaN code 0xFF -- becomes an fp16 NaN, so an out-of-range block poisons its
// outputs instead of silently saturating.
#include <cuda_fp16.h>

#include "api_util.cuh"

namespace tl {

// One thread converts 16 consecutive int8 of a row into 16 fp16 (one 16-byte load, two 16-byte
// stores).  PDL: the launch may overlap the previous kernel's tail; A is read after
// griddepcontrol.wait.  The dependent matmul reads the staged copy after its own wait.
__global__ void __launch_bounds__(256) a8_stage_kernel(const int8_t* __restrict__ A, int64_t lda, int M, int K,
                                                       __half* __restrict__ out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int vec_per_row = K / 16;
  const int64_t total = (int64_t)M * vec_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / vec_per_row;
    const int v = (int)(i - m * vec_per_row);
    const uint4 x = *reinterpret_cast<const uint4*>(A + m * lda + (int64_t)v * 16);
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint32_t h[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int lo = (int)(int8_t)(w[j] >> (16 * q));
        const int hi = (int)(int8_t)(w[j] >> (16 * q + 8));
        const __half2 p = __halves2half2(__int2half_rn(lo), __int2half_rn(hi));  // exact: |v| <= 128
        h[j * 2 + q] = *reinterpret_cast<const uint32_t*>(&p);
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(out + m * (int64_t)K + (int64_t)v * 16);
    dst[0] = make_uint4(h[0], h[1], h[2], h[3]);
    dst[1] = make_uint4(h[4], h[5], h[6], h[7]);
  }
}

tl_status stage_a8(const int8_t* A, int64_t lda, int64_t M, int64_t K, __half* out, cudaStream_t st) {
  const int64_t vecs = M * (K / 16);
  int blocks = (int)((vecs + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, a8_stage_kernel, A, lda, (int)M, (int)K, out);
  if (e != cudaSuccess) return fail(TL_ECUDA, "a8_stage_kernel launch: %s", cudaGetErrorString(e));
  return check_launch("a8_stage_kernel");
}

// E8M0 code e -> fp16 2^(e - 127 + adj) when representable (normal 2^-14..2^15, subnormal down to
// 2^-24), else NaN.  Built from the fp16 bit pattern directly (no float rounding involved).
__global__ void mx_scales_kernel(const uint8_t* __restrict__ e8m0, int64_t count, int adj,
                                 unsigned short* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = e8m0[i];
    const int x = e - 127 + adj;  // the scale is 2^x
    unsigned short h;
    if (e == 0xFF || x > 15 || x < -24) h = 0x7E00u;                 // NaN
    else if (x >= -14) h = (unsigned short)((x + 15) << 10);          // normal: biased exponent x + 15
    else h = (unsigned short)(1u << (x + 24));                        // subnormal: 2^x = m * 2^-24
    out[i] = h;
  }
}

// E8M0 code e -> bf16 2^(e - 127 + adj): bf16 has E8M0's 8 exponent bits, so every finite code is
// exact when adj = 0 (e = 0 gives the bf16 subnormal 2^-127); out of range (|x| beyond
// 2^-133 .. 2^127) or the NaN code 0xFF -> NaN.
__global__ void mx_scales_bf16_kernel(const uint8_t* __restrict__ e8m0, int64_t count, int adj,
                                      unsigned short* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = e8m0[i];
    const int x = e - 127 + adj;  // the scale is 2^x
    unsigned short h;
    if (e == 0xFF || x > 127 || x < -133) h = 0x7FC0u;                 // NaN
    else if (x >= -126) h = (unsigned short)((x + 127) << 7);            // normal: biased exponent x + 127
    else h = (unsigned short)(1u << (x + 133));                          // subnormal: 2^x = m * 2^-133
    out[i] = h;
  }
}

}  // namespace tl

using namespace tl;

extern "C" tl_status tl_mx_scales_to_bf16(const uint8_t* e8m0, int64_t count, int32_t exp_adjust, void* scales_bf16,
                                          void* stream) {
  if (count < 0) return fail(TL_EINVAL_SHAPE, "count=%lld < 0", (long long)count);
  if (count == 0) return TL_OK;
  if (!e8m0 || !scales_bf16) return fail(TL_ENULL, "tl_mx_scales_to_bf16: NULL pointer");
  if (exp_adjust < -64 || exp_adjust > 64) return fail(TL_EINVAL_SHAPE, "exp_adjust=%d outside [-64, 64]", exp_adjust);
  int blocks = (int)((count + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  mx_scales_bf16_kernel<<<blocks, 256, 0, as_stream(stream)>>>(e8m0, count, exp_adjust,
                                                               reinterpret_cast<unsigned short*>(scales_bf16));
  return check_launch("mx_scales_bf16_kernel");
}

extern "C" tl_status tl_mx_scales_to_f16(const uint8_t* e8m0, int64_t count, int32_t exp_adjust, void* scales_f16,
                                         void* stream) {
  if (count < 0) return fail(TL_EINVAL_SHAPE, "count=%lld < 0", (long long)count);
  if (count == 0) return TL_OK;
  if (!e8m0 || !scales_f16) return fail(TL_ENULL, "tl_mx_scales_to_f16: NULL pointer");
  if (exp_adjust < -64 || exp_adjust > 64) return fail(TL_EINVAL_SHAPE, "exp_adjust=%d outside [-64, 64]", exp_adjust);
  int blocks = (int)((count + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  mx_scales_kernel<<<blocks, 256, 0, as_stream(stream)>>>(e8m0, count, exp_adjust,
                                                         reinterpret_cast<unsigned short*>(scales_f16));
  return check_launch("mx_scales_kernel");
}
