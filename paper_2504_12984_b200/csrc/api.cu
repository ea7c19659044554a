// api.cu -- C-ABI entry points of the hot path: validation, the
// GEMV / tensor-core dispatch (row a2), workspace layout, the
// host-buffer end-to-end call and the error strings.
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "api_util.cuh"
#include "paths.cuh"

namespace tl {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int prepare_kernel(const void* fn, int smem_bytes, int threads) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> occ;  // (kernel, device) -> CTAs per SM
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    set_error("cudaGetDevice failed");
    return 0;
  }
  std::lock_guard<std::mutex> lk(mu);
  auto it = occ.find({fn, dev});
  if (it != occ.end()) return it->second;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess) {
    set_error("cudaFuncSetAttribute(MaxDynamicSharedMemorySize=%d) failed on device %d", smem_bytes, dev);
    return 0;
  }
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem_bytes) != cudaSuccess || n < 1) n = 1;
  occ[{fn, dev}] = n;
  return n;
}

// M from which decode-to-fp16 + cuBLAS GEMM beats the fused batched kernel (measured, DESIGN.md
// "Dispatch")
constexpr int64_t kPrefillM = 512;
static bool prefill_wins(int64_t M, int64_t N);

// Workspace: [semaphores: 64 KiB][partials ...]
constexpr size_t kSemBytes = 64 * 1024;

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// Path choice (row a2).  PAPER.md:546 used CUDA cores for 1-15 tokens and tensor
// cores from 16 on an L40S; on B200 the crossover is lower and is set
// from the measured sweep.
static bool prefill_wins(int64_t M, int64_t N) {
  // measured (profiles/r2_prefill.txt): on a wide layer (gate_up, N = 57344) the fused batched
  // kernel keeps ~1015 TFLOP/s up to M ~ 1.5k, decode + cuBLAS wins from 2048; on narrower layers
  // (N <= 16384: qkv, o, down) the batched kernel fills the machine worse and decode + GEMM wins
  // from M = 512
  return M >= 2048 || (M >= kPrefillM && N <= 16384);
}

static int choose_path(tl_wtype w, int64_t M, int64_t N, int32_t G) {
  const int forced = env_int("TL_FORCE_PATH", 0);
  if (forced >= TL_PATH_GEMV && forced <= TL_PATH_PREFILL) return forced;
  (void)w;
  // measured on B200: the tensor-core decode kernel (tcd) for M <= 16 with a group
  // that is a multiple of 128 (it beats the CUDA-core GEMV from M = 1), the CUDA-core GEMV for the
  // remaining decode shapes (G = 32, 64), the tcgen05 GEMM above M = 16
  if (tcd_eligible(M, G)) return TL_PATH_TCD;
  if (prefill_wins(M, N)) return TL_PATH_PREFILL;
  if (M <= 1) return TL_PATH_GEMV;
  return TL_PATH_TC;
}

}  // namespace tl

using namespace tl;

extern "C" {

const char* tl_status_str(tl_status s) {
  switch (s) {
    case TL_OK: return "TL_OK";
    case TL_EINVAL_DTYPE: return "TL_EINVAL_DTYPE";
    case TL_EINVAL_SHAPE: return "TL_EINVAL_SHAPE";
    case TL_EINVAL_GROUP: return "TL_EINVAL_GROUP";
    case TL_EALIGN: return "TL_EALIGN";
    case TL_EZEROS: return "TL_EZEROS";
    case TL_EWORKSPACE: return "TL_EWORKSPACE";
    case TL_EUNSUPPORTED: return "TL_EUNSUPPORTED";
    case TL_ECUDA: return "TL_ECUDA";
    case TL_ENULL: return "TL_ENULL";
  }
  return "TL_UNKNOWN";
}

const char* tl_last_error(void) { return g_err; }

size_t tl_matmul_workspace_bytes(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group) {
  if (a == TL_ACT_I8) {
    // row f4: the fp16 workspace, then the exact fp16 copy of A (act8.cu)
    const size_t f16 = tl_matmul_workspace_bytes(w, TL_ACT_F16, M, N, K, group);
    return M > 0 && K > 0 ? a8_staging_offset(f16) + (size_t)M * (size_t)K * 2 : f16;
  }
  (void)w;
  (void)group;
  if (a != TL_ACT_F16 && a != TL_ACT_BF16) return 0;
  if (M <= 0 || N <= 0 || K <= 0) return kSemBytes;
  size_t g = gemv_workspace_bytes(M, N, K);
  size_t t = tc_workspace_bytes(M, N, K);
  size_t ts = tcd_workspace_bytes(M, N, K);
  if (ts > t) t = ts;
  if (prefill_wins(M, N) || env_int("TL_FORCE_PATH", 0) == TL_PATH_PREFILL) {
    const size_t pf = prefill_workspace_bytes(M, N, K);
    if (pf > t) t = pf;
  }
  return kSemBytes + (g > t ? g : t);
}

tl_status tl_matmul_plan(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group,
                         int32_t* path_out, int32_t* splits_out) {
  if (a == TL_ACT_I8) a = TL_ACT_F16;  // int8 activations run the fp16 families on the staged copy
  if (a != TL_ACT_F16 && a != TL_ACT_BF16) return fail(TL_EUNSUPPORTED, "unknown activation type %d", (int)a);
  (void)K;
  int path = choose_path(w, M, N, group);
  if (a == TL_ACT_BF16 && path == TL_PATH_GEMV) path = tcd_eligible(M, group) ? TL_PATH_TCD : TL_PATH_TC;
  if (path == TL_PATH_TCD && !tcd_eligible(M, group)) path = TL_PATH_TC;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms > 160) sms = 160;
  int splits = 0;
  if (path == TL_PATH_TCD) splits = splitk_grid((int)(N / kBN), sms, false);
  if (path == TL_PATH_TC) splits = splitk_grid((int)((N / kBN + 1) / 2), sms, true);
  if (path_out) *path_out = path;
  if (splits_out) *splits_out = splits;
  return TL_OK;
}

}  // extern "C"

// The body of tl_matmul_ex; `po` (row f3, peer.cuh) non-NULL = gathered output: every finished
// element of Y is also stored into the peers' gathered buffers and the peers are signalled.
static tl_status matmul_core(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group, const void* A,
                             int64_t lda, const void* w_t, const void* scales, const void* zeros, void* Y, int64_t ldy,
                             void* workspace, size_t workspace_bytes, int32_t path, int32_t splits, uint32_t flags,
                             const PeerOut* po, void* stream) {
  tl_status st;
  if ((st = check_wtype(w)) != TL_OK) return st;
  if (a != TL_ACT_F16 && a != TL_ACT_BF16 && a != TL_ACT_I8)
    return fail(TL_EUNSUPPORTED, "unknown activation type %d", (int)a);
  const bool bf = a == TL_ACT_BF16;
  if (flags & ~TL_FLAG_STATIC_WEIGHTS) return fail(TL_EINVAL_SHAPE, "unknown flags 0x%x", flags);
  if (path < TL_PATH_AUTO || path > TL_PATH_PREFILL) return fail(TL_EUNSUPPORTED, "unknown path %d", path);
  if (splits < 0) return fail(TL_EINVAL_SHAPE, "splits=%d < 0", splits);
  if ((st = check_kn(K, N)) != TL_OK) return st;
  if ((st = check_group(K, group)) != TL_OK) return st;
  if (M < 0) return fail(TL_EINVAL_SHAPE, "M=%lld < 0", (long long)M);
  if (M == 0) return TL_OK;
  if (M > (1 << 20)) return fail(TL_EINVAL_SHAPE, "M above 2^20");
  if (!A || !w_t || !scales || !Y) return fail(TL_ENULL, "tl_matmul: NULL pointer");
  if (zeros && w.kind != 0) return fail(TL_EZEROS, "zero points are for uint formats only (reading R6)");
  if (lda < K || ldy < N) return fail(TL_EINVAL_SHAPE, "lda=%lld < K or ldy=%lld < N", (long long)lda, (long long)ldy);
  const int64_t a_esize = a == TL_ACT_I8 ? 1 : 2;
  if (!aligned16(A) || !aligned16(w_t) || !aligned16(scales) || !aligned16(Y) || (zeros && !aligned16(zeros)) ||
      (lda * a_esize) % 16 || (ldy * 2) % 16)
    return fail(TL_EALIGN, "pointers and row strides must be 16-byte aligned");
  const size_t need = tl_matmul_workspace_bytes(w, a, M, N, K, group);
  if (!workspace || workspace_bytes < need)
    return fail(TL_EWORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
  if (!aligned16(workspace)) return fail(TL_EALIGN, "workspace must be 16-byte aligned");
  if (a == TL_ACT_I8) {
    // row f4 (reading R24): stage A exactly as fp16 behind the fp16 workspace, then the fp16 path
    const size_t f16 = tl_matmul_workspace_bytes(w, TL_ACT_F16, M, N, K, group);
    __half* staged = reinterpret_cast<__half*>(reinterpret_cast<uint8_t*>(workspace) + a8_staging_offset(f16));
    if ((st = stage_a8(reinterpret_cast<const int8_t*>(A), lda, M, K, staged, as_stream(stream))) != TL_OK) return st;
    return matmul_core(w, TL_ACT_F16, M, N, K, group, staged, K, w_t, scales, zeros, Y, ldy, workspace,
                       a8_staging_offset(f16), path, splits, flags, po, stream);
  }
  if (path == TL_PATH_AUTO) path = choose_path(w, M, N, group);
  // the CUDA-core kernels are fp16-only: bf16 requests run on the tensor-core families
  if (bf && path == TL_PATH_GEMV) path = tcd_eligible(M, group) ? TL_PATH_TCD : TL_PATH_TC;
  if (path == TL_PATH_TCD && !tcd_eligible(M, group)) path = TL_PATH_TC;
  if (po && path != TL_PATH_TCD && path != TL_PATH_TC) {
    // families without a fused epilogue: the local result, then one replicate-and-signal kernel
    st = matmul_core(w, a, M, N, K, group, A, lda, w_t, scales, zeros, Y, ldy, workspace, workspace_bytes, path,
                     splits, flags, nullptr, stream);
    if (st != TL_OK) return st;
    return gather_push(*po, reinterpret_cast<const __half*>(Y), ldy, M, N, as_stream(stream));
  }
  int* sem = reinterpret_cast<int*>(workspace);
  float* partial = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(workspace) + kSemBytes);
  cudaStream_t s = as_stream(stream);
  if (path == TL_PATH_PREFILL) {
    if (workspace_bytes < kSemBytes + prefill_workspace_bytes(M, N, K))
      return fail(TL_EWORKSPACE, "the prefill path needs %zu workspace bytes",
                  kSemBytes + prefill_workspace_bytes(M, N, K));
    return prefill_matmul(w, M, N, K, group, reinterpret_cast<const __half*>(A), lda,
                          reinterpret_cast<const uint8_t*>(w_t), reinterpret_cast<const __half*>(scales),
                          reinterpret_cast<const __half*>(zeros), reinterpret_cast<__half*>(Y), ldy,
                          reinterpret_cast<uint8_t*>(workspace) + kSemBytes, bf, s);
  }
  if (path == TL_PATH_GEMV && gv1_eligible(M, K, group) && env_int("TL_OLD_GEMV", 0) == 0) {
    tl_status r = gv1_matmul(w, N, K, group, reinterpret_cast<const __half*>(A), reinterpret_cast<const uint8_t*>(w_t),
                             reinterpret_cast<const __half*>(scales), reinterpret_cast<const __half*>(zeros),
                             reinterpret_cast<__half*>(Y), partial, sem, splits,
                             (flags & TL_FLAG_STATIC_WEIGHTS) != 0, s);
    if (r != TL_ENOFIT) return r;
  }
  if (path == TL_PATH_GEMV) {
    if (M > 16) {
      // the CUDA-core path handles up to 16 rows per launch
      for (int64_t m0 = 0; m0 < M; m0 += 16) {
        const int64_t mm = (M - m0) < 16 ? (M - m0) : 16;
        st = tl_matmul_ex(w, a, mm, N, K, group, reinterpret_cast<const __half*>(A) + m0 * lda, lda, w_t, scales,
                          zeros, reinterpret_cast<__half*>(Y) + m0 * ldy, ldy, workspace, workspace_bytes,
                          TL_PATH_GEMV, splits, flags, stream);
        if (st != TL_OK) return st;
      }
      return TL_OK;
    }
    GemvParams p{};
    p.M = (int)M;
    p.N = (int)N;
    p.K = (int)K;
    p.G = group;
    p.A = reinterpret_cast<const __half*>(A);
    p.lda = lda;
    p.wt = reinterpret_cast<const uint8_t*>(w_t);
    p.scales = reinterpret_cast<const __half*>(scales);
    p.zeros = reinterpret_cast<const __half*>(zeros);
    p.Y = reinterpret_cast<__half*>(Y);
    p.ldy = ldy;
    p.partial = partial;
    p.sem = sem;
    p.units = (int)((N / kBN) * (K / kBK));
    p.magic = 0x64006400u;
    return gemv_dispatch(w, p, splits > 0 ? splits : env_int("TL_GRID", 0), s);
  }
  if (path == TL_PATH_TCD) {
    tl_status r = tcd_matmul(w, M, N, K, group, reinterpret_cast<const __half*>(A), lda,
                             reinterpret_cast<const uint8_t*>(w_t), reinterpret_cast<const __half*>(scales),
                             reinterpret_cast<const __half*>(zeros), reinterpret_cast<__half*>(Y), ldy, partial, sem,
                             splits, (flags & TL_FLAG_STATIC_WEIGHTS) != 0, bf, po, s);
    if (r != TL_ENOFIT) return r;
    // the decode kernel's stage ring does not fit shared memory for this shape: batched path
    path = TL_PATH_TC;
  }
  if (path == TL_PATH_TC) {
    return tc_matmul(w, M, N, K, group, reinterpret_cast<const __half*>(A), lda,
                     reinterpret_cast<const uint8_t*>(w_t), reinterpret_cast<const __half*>(scales),
                     reinterpret_cast<const __half*>(zeros), reinterpret_cast<__half*>(Y), ldy, partial, sem,
                     splits, bf, po, s);
  }
  return fail(TL_EUNSUPPORTED, "unknown path %d", path);
}

extern "C" {

tl_status tl_matmul_ex(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group, const void* A,
                       int64_t lda, const void* w_t, const void* scales, const void* zeros, void* Y, int64_t ldy,
                       void* workspace, size_t workspace_bytes, int32_t path, int32_t splits, uint32_t flags,
                       void* stream) {
  return matmul_core(w, a, M, N, K, group, A, lda, w_t, scales, zeros, Y, ldy, workspace, workspace_bytes, path,
                     splits, flags, nullptr, stream);
}

tl_status tl_matmul_gathered(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group, const void* A,
                             int64_t lda, const void* w_t, const void* scales, const void* zeros, void* Y,
                             int64_t ldy, void* const* Y_peers, uint32_t* const* flag_peers, int32_t npeers,
                             void* workspace, size_t workspace_bytes, uint32_t flags, void* stream) {
  if (npeers < 0 || npeers > kMaxPeers) return fail(TL_EINVAL_SHAPE, "npeers=%d outside [0, %d]", npeers, kMaxPeers);
  if (npeers == 0)
    return matmul_core(w, a, M, N, K, group, A, lda, w_t, scales, zeros, Y, ldy, workspace, workspace_bytes,
                       TL_PATH_AUTO, 0, flags, nullptr, stream);
  if (!Y_peers || !flag_peers) return fail(TL_ENULL, "tl_matmul_gathered: NULL peer arrays");
  PeerOut po{};
  for (int i = 0; i < npeers; ++i) {
    if (!Y_peers[i] || !flag_peers[i]) return fail(TL_ENULL, "tl_matmul_gathered: NULL peer pointer %d", i);
    if (!aligned16(Y_peers[i]) || (reinterpret_cast<uintptr_t>(flag_peers[i]) & 3u))
      return fail(TL_EALIGN, "peer %d: Y must be 16-byte and the flag 4-byte aligned", i);
    po.y[i] = reinterpret_cast<unsigned short*>(Y_peers[i]);
    po.flag[i] = flag_peers[i];
  }
  po.n = npeers;
  po.signal = 1;
  if (M == 0) return TL_OK;  // nothing to send: callers do not wait for an empty call
  if (workspace && workspace_bytes >= kSemBytes && aligned16(workspace))
    po.done = reinterpret_cast<uint32_t*>(workspace) + kSemBytes / 4 - 1;  // last semaphore word
  return matmul_core(w, a, M, N, K, group, A, lda, w_t, scales, zeros, Y, ldy, workspace, workspace_bytes,
                     TL_PATH_AUTO, 0, flags, &po, stream);
}

tl_status tl_matmul(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group, const void* A,
                    int64_t lda, const void* w_t, const void* scales, const void* zeros, void* Y, int64_t ldy,
                    void* workspace, size_t workspace_bytes, void* stream) {
  return tl_matmul_ex(w, a, M, N, K, group, A, lda, w_t, scales, zeros, Y, ldy, workspace, workspace_bytes,
                      TL_PATH_AUTO, 0, 0u, stream);
}

tl_status tl_matmul_batch_hostio(tl_atype a, int32_t count, const tl_batch_item* items, const void* A_host,
                                 void* A_dev, void* Y_dev, void* Y_host, uint32_t flags, void* stream) {
  if (count < 0) return fail(TL_EINVAL_SHAPE, "count=%d < 0", count);
  if (count == 0) return TL_OK;
  if (a != TL_ACT_F16 && a != TL_ACT_BF16 && a != TL_ACT_I8)
    return fail(TL_EUNSUPPORTED, "unknown activation type %d", (int)a);
  if (!items || !A_host || !A_dev || !Y_dev || !Y_host) return fail(TL_ENULL, "tl_matmul_batch_hostio: NULL pointer");
  const size_t ae = a == TL_ACT_I8 ? 1 : 2;
  size_t a_bytes = 0, y_bytes = 0;
  for (int i = 0; i < count; ++i) {
    if (items[i].M < 0 || items[i].N <= 0 || items[i].K <= 0)
      return fail(TL_EINVAL_SHAPE, "item %d: M=%lld N=%lld K=%lld", i, (long long)items[i].M, (long long)items[i].N,
                  (long long)items[i].K);
    a_bytes += (size_t)(items[i].M * items[i].K) * ae;
    y_bytes += (size_t)(items[i].M * items[i].N) * 2;
  }
  cudaStream_t s = as_stream(stream);
  if (cudaMemcpyAsync(A_dev, A_host, a_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return fail(TL_ECUDA, "H2D copy of the activations failed");
  size_t ao = 0, yo = 0;
  for (int i = 0; i < count; ++i) {
    const tl_batch_item& it = items[i];
    tl_status st = tl_matmul_ex(it.w, a, it.M, it.N, it.K, it.group, reinterpret_cast<uint8_t*>(A_dev) + ao, it.K,
                                it.w_t, it.scales, it.zeros, reinterpret_cast<uint8_t*>(Y_dev) + yo, it.N, it.workspace,
                                it.workspace_bytes, TL_PATH_AUTO, 0, flags, stream);
    if (st != TL_OK) return st;
    ao += (size_t)(it.M * it.K) * ae;
    yo += (size_t)(it.M * it.N) * 2;
  }
  if (cudaMemcpyAsync(Y_host, Y_dev, y_bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return fail(TL_ECUDA, "D2H copy of the outputs failed");
  return TL_OK;
}

tl_status tl_matmul_hostio(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group,
                           const void* A_host, void* A_dev, const void* w_t, const void* scales, const void* zeros,
                           void* Y_dev, void* Y_host, void* workspace, size_t workspace_bytes, uint32_t flags,
                           void* stream) {
  if (M == 0) return TL_OK;
  if (a != TL_ACT_F16 && a != TL_ACT_BF16 && a != TL_ACT_I8)
    return fail(TL_EUNSUPPORTED, "unknown activation type %d", (int)a);
  if (!A_host || !A_dev || !Y_dev || !Y_host) return fail(TL_ENULL, "tl_matmul_hostio: NULL pointer");
  cudaStream_t s = as_stream(stream);
  const size_t a_bytes = (size_t)(M * K) * (a == TL_ACT_I8 ? 1 : 2);
  if (cudaMemcpyAsync(A_dev, A_host, a_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return fail(TL_ECUDA, "H2D copy of A failed");
  tl_status st = tl_matmul_ex(w, a, M, N, K, group, A_dev, K, w_t, scales, zeros, Y_dev, N, workspace,
                              workspace_bytes, TL_PATH_AUTO, 0, flags, stream);
  if (st != TL_OK) return st;
  if (cudaMemcpyAsync(Y_host, Y_dev, (size_t)(M * N * 2), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return fail(TL_ECUDA, "D2H copy of Y failed");
  return TL_OK;
}

}  // extern "C"
