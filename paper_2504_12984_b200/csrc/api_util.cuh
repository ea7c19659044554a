// api_util.cuh -- host-side validation and error reporting shared by the C-ABI entry points.
#pragma once

#include <cstdarg>
#include <cstdio>

#include "../../include/tilus_b200.h"
#include "dispatch.cuh"

namespace tl {

void set_error(const char* fmt, ...);  // thread-local message for tl_last_error()

inline tl_status fail(tl_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return st;
}

inline tl_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TL_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return TL_OK;
}

// Is `w` one of the 37 kernel formats (reading R4)?
inline bool wtype_ok(tl_wtype w) {
  return dispatch_format(w.kind, w.bits, w.kind == 2 ? w.exp_bits : 0, [](auto) {}) &&
         (w.kind == 2 ? (w.man_bits == w.bits - 1 - w.exp_bits) : (w.exp_bits == 0 && w.man_bits == 0));
}

inline tl_status check_wtype(tl_wtype w) {
  if (!wtype_ok(w))
    return fail(TL_EINVAL_DTYPE, "weight type kind=%d bits=%d e=%d m=%d is not a kernel format", w.kind, w.bits,
                w.exp_bits, w.man_bits);
  return TL_OK;
}

inline tl_status check_kn(int64_t K, int64_t N) {
  if (K <= 0 || N <= 0 || K % kBK || N % kBN)
    return fail(TL_EINVAL_SHAPE, "K=%lld, N=%lld must be positive multiples of 128", (long long)K, (long long)N);
  if (K > (1ll << 20) || N > (1ll << 20)) return fail(TL_EINVAL_SHAPE, "K or N above 2^20");
  return TL_OK;
}

inline tl_status check_group(int64_t K, int32_t G) {
  const bool ok = G > 0 && K % G == 0 && (G == 32 || G == 64 || G % 128 == 0);
  if (!ok) return fail(TL_EINVAL_GROUP, "group %d must divide K=%lld and be 32, 64 or a multiple of 128", G, (long long)K);
  return TL_OK;
}

// Per-(kernel, device) one-time preparation: opts `fn` into `smem_bytes` of dynamic
// shared memory on the CURRENT device and returns its resident CTAs per SM there (occupancy).
// Function attributes are per device context, so the cache is keyed on (fn, device); it is
// guarded by a mutex (the C ABI is thread-safe).  Returns 0 on a CUDA error (tl_last_error set).
int prepare_kernel(const void* fn, int smem_bytes, int threads);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace tl
