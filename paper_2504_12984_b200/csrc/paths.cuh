// paths.cuh -- internal interface between the C-ABI layer (api.cu) and the kernel
// families (gemv.cu: CUDA-core decode path; tc.cu: tcgen05 tensor-core path).
#pragma once

#include "api_util.cuh"
#include "peer.cuh"

namespace tl {

struct GemvParams {
  int M, N, K, G;
  const __half* A;
  int64_t lda;
  const uint8_t* wt;
  const __half* scales;
  const __half* zeros;
  __half* Y;
  int64_t ldy;
  float* partial;  // [grid][2][M][128] fp32 stream-K partial tiles
  int* sem;        // [N/128] self-resetting tile semaphores
  int units;       // (N/128) * (K/128)
  uint32_t magic;  // 0x64006400 (see PairConsts::magic)
};

tl_status gemv_dispatch(tl_wtype w, const GemvParams& p, int grid_req, cudaStream_t st);
bool gv1_eligible(int64_t M, int64_t K, int32_t G);
tl_status gv1_matmul(tl_wtype w, int64_t N, int64_t K, int32_t G, const __half* A, const uint8_t* wt,
                     const __half* scales, const __half* zeros, __half* Y, float* partial, int* sem, int grid_req,
                     bool static_weights, cudaStream_t st);
size_t gemv_workspace_bytes(int64_t M, int64_t N, int64_t K);

// CTAs the GEMV workspace holds partial slots for (the grid is clamped to it)
constexpr int kGemvMaxCtas = 148 * 8;
// internal status (never returned through the ABI): the decode kernel's ring does not fit
constexpr tl_status TL_ENOFIT = (tl_status)100;
size_t tc_workspace_bytes(int64_t M, int64_t N, int64_t K);
tl_status tc_matmul(tl_wtype w, int64_t M, int64_t N, int64_t K, int32_t G, const __half* A, int64_t lda,
                    const uint8_t* wt, const __half* scales, const __half* zeros, __half* Y, int64_t ldy,
                    float* partial, int* sem, int grid_req, bool bf, const PeerOut* po, cudaStream_t st);
size_t prefill_workspace_bytes(int64_t M, int64_t N, int64_t K);
tl_status prefill_matmul(tl_wtype w, int64_t M, int64_t N, int64_t K, int32_t G, const __half* A, int64_t lda,
                         const uint8_t* wt, const __half* scales, const __half* zeros, __half* Y, int64_t ldy,
                         uint8_t* ws, bool bf, cudaStream_t st);
bool tcd_eligible(int64_t M, int32_t G);
int splitk_grid(int work, int sms, bool expensive_partials);
size_t tcd_workspace_bytes(int64_t M, int64_t N, int64_t K);
tl_status tcd_matmul(tl_wtype w, int64_t M, int64_t N, int64_t K, int32_t G, const __half* A, int64_t lda,
                     const uint8_t* wt, const __half* scales, const __half* zeros, __half* Y, int64_t ldy,
                     float* partial, int* sem, int grid_req, bool static_weights, bool bf, const PeerOut* po,
                     cudaStream_t st);
// row f3 (gather.cu): replicate a finished local Y [M, N] (row stride ldy) into the peers' gathered
// buffers and signal them -- the path for the kernel families without a fused epilogue
tl_status gather_push(const PeerOut& po, const __half* Y, int64_t ldy, int64_t M, int64_t N, cudaStream_t st);

// row f4 (act8.cu): exact int8 -> fp16 staging of A; the staged copy sits behind the fp16 workspace
tl_status stage_a8(const int8_t* A, int64_t lda, int64_t M, int64_t K, __half* out, cudaStream_t st);
inline size_t a8_staging_offset(size_t f16_workspace_bytes) { return (f16_workspace_bytes + 255) & ~(size_t)255; }

}  // namespace tl
