// prefill.cu -- host side of the large-M path (prefill.cuh): per-chunk decode to fp16 + cuBLAS
// f16 x f16 GEMM with fp32 accumulation.  cuBLAS is used only for the plain dense
// GEMM; the decode is this library's kernel.
#include <cublas_v2.h>

#include <map>
#include <mutex>

#include "paths.cuh"
#include "prefill.cuh"

namespace tl {

template <class F>
tl_status launch_dq16(const uint8_t* wt, const __half* scales, const __half* zeros, __half* out, int N, int K, int G,
                      int nt0, int ntiles, bool bf, cudaStream_t st);
#define TL_EXTERN_DQ16(K, B, E)                                                                            \
  extern template tl_status launch_dq16<Fmt<K, B, E>>(const uint8_t*, const __half*, const __half*, __half*, int, \
                                                      int, int, int, int, bool, cudaStream_t);
TL_FOR_EACH_FORMAT(TL_EXTERN_DQ16)
#undef TL_EXTERN_DQ16

constexpr size_t kCublasWs = 32u << 20;     // cuBLAS workspace (set explicitly: no allocation, graph-capturable)
constexpr size_t kChunkBytes = 64u << 20;   // decoded W^T chunk (stays in the 126 MB L2 for the GEMM)

static int64_t chunk_cols(int64_t N, int64_t K) {
  int64_t nc = (int64_t)(kChunkBytes / (2 * (size_t)K)) / kBN * kBN;
  if (nc < kBN) nc = kBN;
  return nc < N ? nc : N;
}

size_t prefill_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  (void)M;
  return kCublasWs + (size_t)chunk_cols(N, K) * (size_t)K * 2 + 256;
}

static std::mutex g_cublas_mu;
static std::map<int, cublasHandle_t> g_cublas;

tl_status prefill_matmul(tl_wtype w, int64_t M, int64_t N, int64_t K, int32_t G, const __half* A, int64_t lda,
                         const uint8_t* wt, const __half* scales, const __half* zeros, __half* Y, int64_t ldy,
                         uint8_t* ws, bool bf, cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(TL_ECUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(g_cublas_mu);
  cublasHandle_t h;
  auto it = g_cublas.find(dev);
  if (it == g_cublas.end()) {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return fail(TL_ECUDA, "cublasCreate failed");
    g_cublas[dev] = h;
  } else {
    h = it->second;
  }
  uint8_t* cws = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
  __half* wbuf = reinterpret_cast<__half*>(cws + kCublasWs);
  if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS || cublasSetWorkspace(h, cws, kCublasWs) != CUBLAS_STATUS_SUCCESS)
    return fail(TL_ECUDA, "cublasSetStream / cublasSetWorkspace failed");
  const int64_t nc_max = chunk_cols(N, K);
  const float alpha = 1.f, beta = 0.f;
  for (int64_t n0 = 0; n0 < N; n0 += nc_max) {
    const int64_t nc = (N - n0) < nc_max ? (N - n0) : nc_max;
    tl_status s = TL_EUNSUPPORTED;
    dispatch_format(w.kind, w.bits, w.kind == 2 ? w.exp_bits : 0, [&](auto f) {
      using F = decltype(f);
      s = launch_dq16<F>(wt, scales, zeros, wbuf, (int)N, (int)K, G, (int)(n0 / kBN), (int)(nc / kBN), bf, st);
    });
    if (s != TL_OK) return s;
    // Y^T[n0:n0+nc, :M] = (W^T chunk [nc, K]) x A^T  (column-major view of the row-major arrays)
    const cudaDataType_t dt = bf ? CUDA_R_16BF : CUDA_R_16F;
    const cublasStatus_t r = cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)nc, (int)M, (int)K, &alpha, wbuf, dt,
                                          (int)K, A, dt, (int)lda, &beta, Y + n0, dt, (int)ldy, CUBLAS_COMPUTE_32F,
                                          CUBLAS_GEMM_DEFAULT);
    if (r != CUBLAS_STATUS_SUCCESS) return fail(TL_ECUDA, "cublasGemmEx failed (%d)", (int)r);
  }
  return TL_OK;
}

}  // namespace tl
