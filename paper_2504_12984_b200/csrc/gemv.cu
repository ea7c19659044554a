// gemv.cu -- format dispatch of the CUDA-core path; the kernels are in gemv.cuh and are
// instantiated one format per translation unit (build/gen/gemv_*.cu) so they compile in parallel.
#include <cstdlib>

#include "gv1.cuh"
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

template <class F>
tl_status launch_gv1(const Gv1Params& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st);
#define TL_EXTERN_GV1(K, B, E)                                                                                 \
  extern template tl_status launch_gv1<Fmt<K, B, E>>(const Gv1Params&, const CUtensorMap*, int, uint32_t, cudaStream_t);
TL_FOR_EACH_FORMAT(TL_EXTERN_GV1)
#undef TL_EXTERN_GV1
tl_status make_tmap_side(CUtensorMap* m, const __half* X, int64_t N, int64_t K, int32_t G, int R);

bool gv1_eligible(int64_t M, int64_t K, int32_t G) { return M == 1 && G % kBK == 0 && K * 2 <= 65536; }

// CUDA-core decode GEMV for M = 1 (gv1.cuh)
tl_status gv1_matmul(tl_wtype w, int64_t N, int64_t K, int32_t G, const __half* A, const uint8_t* wt,
                     const __half* scales, const __half* zeros, __half* Y, float* partial, int* sem, int grid_req,
                     bool static_weights, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms > 160) sms = 160;
  Gv1Params p{};
  p.N = (int)N;
  p.K = (int)K;
  p.G = G;
  p.units = (int)((N / kBN) * (K / kBK));
  p.wt = wt;
  p.A = A;
  p.scales = scales;
  p.zeros = zeros;
  p.Y = Y;
  p.partial = partial;
  p.sem = sem;
  p.static_w = static_weights ? 1 : 0;
  {
    const char* v = getenv("TL_GV1_DBG");
    p.dbg = v ? atoi(v) : 0;
  }
  int grid = grid_req > 0 ? grid_req : splitk_grid((int)(N / kBN), sms, false);
  if (grid > 160) grid = 160;
  if (grid > p.units) grid = p.units;
  const uint32_t wb = (uint32_t)tile_bytes(w.bits);
  const int R = gv1_tiles_per_stage(w.bits);
  p.stage_bytes = ((uint32_t)R * wb + side_bytes(R) + 127) & ~127u;
  const uint32_t KT = (uint32_t)(K / kBK);
  const uint32_t fixed = 128 + (uint32_t)K * 2 + KT * 4 + kGv1Groups * kBN * 4 + 1024;
  if (fixed + 3u * p.stage_bytes > 227u * 1024u) return TL_ENOFIT;
  int ns = (int)((227u * 1024u - fixed) / p.stage_bytes);
  if (ns > 32) ns = 32;
  p.ns = ns;
  p.stash_off = ((uint32_t)ns * p.stage_bytes + 127) & ~127u;
  p.sums_off = p.stash_off + (uint32_t)K * 2;
  p.red_off = (p.sums_off + KT * 4 + 127) & ~127u;
  p.bar_off = (p.red_off + kGv1Groups * kBN * 4 + 15) & ~15u;
  const uint32_t smem = p.bar_off + (2 * ns + 1) * 8 + 32 + 128;
  if (smem > 227 * 1024) return TL_ENOFIT;
  CUtensorMap tmap[2];
  tl_status s = make_tmap_side(&tmap[0], scales, N, K, G, R);
  if (s != TL_OK) return s;
  if ((s = make_tmap_side(&tmap[1], zeros ? zeros : scales, N, K, G, R)) != TL_OK) return s;
  s = TL_EUNSUPPORTED;
  dispatch_format(w.kind, w.bits, w.kind == 2 ? w.exp_bits : 0, [&](auto f) {
    using F = decltype(f);
    s = launch_gv1<F>(p, tmap, grid, smem, st);
  });
  return s;
}

size_t gemv_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  // partial slots for at most kGemvMaxCtas CTAs (the launch clamps its grid to it), 2 slots each,
  // + one semaphore per n-tile
  const int64_t grid = kGemvMaxCtas;
  return (size_t)(grid * 2 * (M > 16 ? 16 : M) * kBN * 4) + (size_t)((N / kBN) * 4) + 256;
}

}  // namespace tl
