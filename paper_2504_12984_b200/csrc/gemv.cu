// gemv.cu -- format dispatch of the CUDA-core path; the kernels are in gemv.cuh and are
// instantiated one format per translation unit (build/gen/gemv_*.cu) so they compile in parallel.
#include "paths.cuh"

namespace tl {

template <class F>
tl_status launch_gemv(const GemvParams& p, int grid_req, cudaStream_t st);

tl_status gemv_dispatch(tl_wtype w, const GemvParams& p, int grid_req, cudaStream_t st) {
  tl_status r = TL_EUNSUPPORTED;
  dispatch_format(w.kind, w.bits, w.kind == 2 ? w.exp_bits : 0, [&](auto f) {
    using F = decltype(f);
    r = launch_gemv<F>(p, grid_req, st);
  });
  return r;
}

size_t gemv_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  // partial slots for at most kGemvMaxCtas CTAs (the launch clamps its grid to it), 2 slots each,
  // + one semaphore per n-tile
  const int64_t grid = kGemvMaxCtas;
  return (size_t)(grid * 2 * (M > 16 ? 16 : M) * kBN * 4) + (size_t)((N / kBN) * 4) + 256;
}

}  // namespace tl
