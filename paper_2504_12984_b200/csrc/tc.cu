// tc.cu -- host side of the tensor-core paths (decode tcd.cuh, batched tc2.cuh): shared-memory
// carve-up, the TMA tensor map of the activations, m-chunking (MMA N <= 128) and the per-format
// dispatch.  The kernels are instantiated one format per translation unit (build/gen/tcd_*.cu,
// build/gen/tc2_*.cu).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "tc2.cuh"
#include "tcd.cuh"

namespace tl {

template <class F>
tl_status launch_tc2(const Tc2Params& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st);


template <class F>
tl_status launch_tcd(const TcdParams& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st);

// the kernels are instantiated one format per generated translation unit (build.py): keep this
// one from instantiating all 37 formats' kernels again
#define TL_EXTERN_TC(K, B, E)                                                                              \
  extern template tl_status launch_tc2<Fmt<K, B, E>>(const Tc2Params&, const CUtensorMap*, int, uint32_t,   \
                                                     cudaStream_t);                                       \
  extern template tl_status launch_tcd<Fmt<K, B, E>>(const TcdParams&, const CUtensorMap*, int, uint32_t,   \
                                                     cudaStream_t);
TL_FOR_EACH_FORMAT(TL_EXTERN_TC)
#undef TL_EXTERN_TC

static tl_status make_tmap_a(CUtensorMap* m, const __half* A, int64_t M, int64_t K, int64_t lda, int NB);

long long* g_trace = nullptr;  // debug: clock64 stamps of CTA 0 (TL_TRACE=1)

bool tcd_eligible(int64_t M, int32_t G) { return M >= 1 && M <= kTcdNB && G >= kBK; }

static int env_dbg(const char* name) {
  const char* v = getenv(name);
  return v ? atoi(v) : 0;
}

// decode tensor-core path (tcd.cuh): the weight tile and its scale / zero slices ride in one TMA stage
tl_status tcd_matmul(tl_wtype w, int64_t M, int64_t N, int64_t K, int32_t G, const __half* A, int64_t lda,
                     const uint8_t* wt, const __half* scales, const __half* zeros, __half* Y, int64_t ldy,
                     float* partial, int* sem, int grid_req, bool static_weights, bool bf, const PeerOut* po,
                     cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms > 160) sms = 160;
  TcdParams p{};
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.G = G;
  p.units = (int)((N / kBN) * (K / kBK));
  p.wt = wt;
  p.A = A;
  p.lda = lda;
  p.scales = scales;
  p.zeros = zeros;
  p.Y = Y;
  p.ldy = ldy;
  p.partial = partial;
  p.sem = sem;
  p.dbg = env_dbg("TL_TCD_DBG");
  p.static_w = static_weights ? 1 : 0;
  p.bf = bf ? 1 : 0;
  if (po) p.po = *po;
  p.magic = 0x64006400u;
  if (getenv("TL_TRACE")) {
    static int launches = 0;  // two trace buffers, alternating per launch (back-to-back overlap)
    if (!g_trace) cudaMalloc(&g_trace, 2 * 16 * 256 * sizeof(long long));
    p.trace = g_trace + (launches++ & 1) * 16 * 256;
  }
  int grid = grid_req > 0 ? grid_req : splitk_grid((int)(N / kBN), sms, false);
  if (grid > 160) grid = 160;
  if (grid > p.units) grid = p.units;
  // decode (M = 1) with the activation row resident in shared memory (TcdCfg<1>): K*2 <= 64 KB
  p.rot = (M <= 1 && K * 2 <= 65536) ? 1 : 0;
  const uint32_t wb = (uint32_t)tile_bytes(w.bits);
  const int R = tcd_tiles_per_stage(w.bits);
  p.R = R;
  p.stage_bytes = ((uint32_t)R * (wb + 512) + 127) & ~127u;  // R weight tiles | R scale rows | R zero rows
  const uint32_t red = (uint32_t)((M <= 1 && K * 2 <= 65536) ? TcdCfg<1>::NG : TcdCfg<kTcdNB>::NG) * (uint32_t)M * kBN * 4;
  const uint32_t opb = (uint32_t)((M <= 1 && K * 2 <= 65536) ? TcdCfg<1>::NOP : TcdCfg<kTcdNB>::NOP) * kTcdOpBytes;
  const uint32_t stash = p.rot ? (uint32_t)(K * 2) : 0u;
  const uint64_t fixed = 1024 /*align*/ + (uint64_t)opb + stash + red + 2048 /*barriers, tmem slot, flags*/;
  if (fixed + 3ull * p.stage_bytes > 227u * 1024u)
    return TL_ENOFIT;  // caller falls back to the batched path
  int ns = (int)((227u * 1024u - fixed) / p.stage_bytes);
  if (ns > 32) ns = 32;
  if (env_dbg("TL_TCD_NS") > 0 && env_dbg("TL_TCD_NS") < ns) ns = env_dbg("TL_TCD_NS");
  p.ns = ns;
  p.op_off = ((uint32_t)ns * p.stage_bytes + 1023) & ~1023u;
  p.stash_off = p.op_off + opb;
  p.red_off = p.stash_off + ((stash + 127) & ~127u);
  p.bar_off = (p.red_off + red + 15) & ~15u;
  const uint32_t smem =
      p.bar_off + (2 * ns + 2 * kTcdMaxNOP + 2 * kTcdMaxNW + 2 * kTcdMaxNACC + 1) * 8 + 32 + 1024;
  if (smem > 227 * 1024) return TL_ENOFIT;
  CUtensorMap tmap;
  tl_status s = make_tmap_a(&tmap, A, M, K, lda, kTcdNB);
  if (s != TL_OK) return s;
  s = TL_EUNSUPPORTED;
  dispatch_format(w.kind, w.bits, w.kind == 2 ? w.exp_bits : 0, [&](auto f) {
    using F = decltype(f);
    s = launch_tcd<F>(p, &tmap, grid, smem, st);
  });
  return s;
}

size_t tcd_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  (void)M;
  (void)N;
  (void)K;
  return (size_t)160 * 2 * kTcdNB * 128 * 4;
}

constexpr int kTcMaxCtas = 160;

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Split-K grid (row a2 / a10; measured): `work` = independent output blocks
// (n-tiles for tcd, n-pairs for tc2), `sms` = SMs.  When a whole multiple S >= 2 of the blocks fits
// the SMs, every block is split into exactly S CTAs (ranges aligned to block boundaries: each
// stream-K reduction has S equal contributors that finish together); when there are more
// blocks than SMs, the grid is the smallest that gives every CTA the same number of WHOLE blocks
// if that loses little, else one CTA per SM (stream-K).  `expensive_partials`: the batched
// kernel's fp32 partial tiles are up to 128 KB per CTA, the decode kernel's 0.5-8 KB.
int splitk_grid(int work, int sms, bool expensive_partials) {
  if (work <= 0) return 1;
  if (work <= sms) {
    const int S = sms / work;
    if (expensive_partials) return S * work;                  // aligned splits always win (tc2)
    return (S >= 2 && S * work * 100 >= 85 * sms) ? S * work : sms;  // tcd: only near-full grids
  }
  const int per = (work + sms - 1) / sms;  // whole blocks per CTA
  const int g = (work + per - 1) / per;
  return (expensive_partials && work % per == 0) ? g : sms;
}

size_t tc_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  (void)N;
  (void)K;
  const int nb = round_up((int)(M < 128 ? M : 128), 16);
  return (size_t)kTcMaxCtas * 2 /*slots*/ * 2 /*n-pair tiles*/ * nb * 128 * 4;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// A [M, K] fp16 row-major (row stride lda elements): boxes of 64 k x NB rows, 128B swizzle,
// rows >= M zero-filled by the TMA unit.
static tl_status make_tmap_a(CUtensorMap* m, const __half* A, int64_t M, int64_t K, int64_t lda, int NB) {
  auto enc = get_encode();
  if (!enc) return fail(TL_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)(lda * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)NB};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(A), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TL_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TL_OK;
}

// The [K/G, N] scale / zero array as a 3-D tensor {128 columns, K/G rows, N/128 n-tiles}
// (strides N*2 and 256 bytes): boxes {128, R, 1} = the rows of R consecutive k-tiles of one n-tile
// (common.cuh side_row_off).  Rows past K/G are zero-filled.
tl_status make_tmap_side(CUtensorMap* m, const __half* X, int64_t N, int64_t K, int32_t G, int R) {
  auto enc = get_encode();
  if (!enc) return fail(TL_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)kBN, (cuuint64_t)(K / G), (cuuint64_t)(N / kBN)};
  cuuint64_t strides[2] = {(cuuint64_t)(N * 2), (cuuint64_t)(kBN * 2)};
  cuuint32_t box[3] = {(cuuint32_t)kBN, (cuuint32_t)R, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(X), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TL_ECUDA, "cuTensorMapEncodeTiled (scales) failed (%d)", (int)r);
  return TL_OK;
}

tl_status tc_matmul(tl_wtype w, int64_t M, int64_t N, int64_t K, int32_t G, const __half* A, int64_t lda,
                    const uint8_t* wt, const __half* scales, const __half* zeros, __half* Y, int64_t ldy,
                    float* partial, int* sem, int grid_req, bool bf, const PeerOut* po, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms > kTcMaxCtas) sms = kTcMaxCtas;
  for (int64_t m0 = 0; m0 < M; m0 += 128) {
    const int mc = (int)((M - m0) < 128 ? (M - m0) : 128);
    Tc2Params p{};
    p.M = mc;
    p.N = (int)N;
    p.K = (int)K;
    p.G = G;
    p.NB = round_up(mc, 16);
    p.NT = (int)(N / kBN);
    p.units = (int)(((N / kBN + 1) / 2) * (K / kBK));  // (n-pair, k-tile) units
    p.wt = wt;
    p.scales = scales;
    p.zeros = zeros;
    p.Y = Y + m0 * ldy;
    p.ldy = ldy;
    p.partial = partial;
    p.sem = sem;
    p.magic = 0x64006400u;
    p.dbg = env_dbg("TL_TC2_DBG");
    p.bf = bf ? 1 : 0;
    if (po) {
      p.po = *po;
      for (int i = 0; i < po->n; ++i) p.po.y[i] = po->y[i] + m0 * ldy;
      p.po.signal = (m0 + 128 >= M) ? 1 : 0;  // the last chunk's launch signals the whole call
    }
    // stage: [activation boxes NB x 256 B (1024-aligned, 128B swizzle) | weight tile 2p | weight tile 2p+1]
    const uint32_t wb = (uint32_t)tile_bytes(w.bits);
    p.w_off_in_stage = (uint32_t)p.NB * 256;
    p.stage_bytes = (p.w_off_in_stage + 2 * wb + 1023) & ~1023u;
    const uint32_t budget = 227 * 1024 - 1024 - 512;
    int ns = 16;
    while (ns > 2 && (uint32_t)ns * p.stage_bytes > budget) --ns;
    p.ns = ns;
    const uint32_t smem = ns * p.stage_bytes + (2 * ns + 2 * kTc2Groups + 2) * 8 + 32 + 1024;
    if (smem > 227 * 1024)
      return fail(TL_EUNSUPPORTED, "tensor-core tile does not fit shared memory (ns=%d stage=%u smem=%u)", ns,
                  p.stage_bytes, smem);
    CUtensorMap tmap;
    tl_status s = make_tmap_a(&tmap, A + m0 * lda, mc, K, lda, p.NB);
    if (s != TL_OK) return s;
    int grid = grid_req > 0 ? grid_req : splitk_grid((p.NT + 1) / 2, sms, true);
    if (grid > kTcMaxCtas) grid = kTcMaxCtas;
    if (grid > p.units) grid = p.units;
    // distributed stream-K reduction (tc2.cuh): only for the aligned splits (grid = S x n-pairs, so
    // every CTA's range lies inside one n-pair and its S contributors start together) and when every
    // CTA is resident at once (one CTA per SM).  Measured: u3 M = 128 qkv 42.6 -> 39.9 us, o 37.9 ->
    // 33.7, down 69.3 -> 64.2; with unaligned ranges the contributors' waits chain (148 CTAs on qkv:
    // 57 -> 223 us), hence the guard.  TL_TC2_DIST=0 keeps the last-arriver reduction.
    {
      int sm_count = 148;
      cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
      const char* d = getenv("TL_TC2_DIST");
      const int npairs = (p.NT + 1) / 2;
      p.dist = (grid <= sm_count && grid % npairs == 0 && (d == nullptr || atoi(d) != 0)) ? 1 : 0;
    }
    s = TL_EUNSUPPORTED;
    dispatch_format(w.kind, w.bits, w.kind == 2 ? w.exp_bits : 0, [&](auto f) {
      using F = decltype(f);
      s = launch_tc2<F>(p, &tmap, grid, smem, st);
    });
    if (s != TL_OK) return s;
  }
  return TL_OK;
}

}  // namespace tl

// debug hook (not part of the public ABI): copy the CTA-0 pipeline stamps to the host
extern "C" int tl__debug_trace(long long* host) {
  if (!tl::g_trace) return -1;
  return (int)cudaMemcpy(host, tl::g_trace, 2 * 16 * 256 * sizeof(long long), cudaMemcpyDeviceToHost);
}
