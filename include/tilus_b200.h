/*
 * tilus_b200.h -- C ABI of the B200-native A16Wx low-bit-weight matmul.
 *
 * The operation is the paper's "C_{M,N} = A_{M,K} x B_{K,N}, where A and B are
 * float16 and int6", generalised to every weight format of
 * PAPER.md:162 (uint1..8, int2..8 -- int1 is an extension --, float3..8 with any
 * exponent/mantissa split), with group-wise fp16 scales along K and, for
 * unsigned formats, zero points (north star; readings R6-R8):
 *
 *     w[k,n] = (value(q[k,n]) - z[k/G, n]) * s[k/G, n]        (z = 0 unless uint)
 *     Y[m,n] = fp16( sum_k A[m,k] * w[k,n] )   accumulated in fp32
 *
 * The weights reach the library as the paper's compact bitstream
 * (LSB-first, row-major [K,N], reading R1/R2), are re-laid
 * out ONCE by tl_transform_weights (the "Change Layout" pre-processing step of
 * PAPER.md:187 / PAPER.md:409-416) and then consumed by tl_matmul on every
 * call.  The transformed layout is opaque and versioned (tl_format_version).
 *
 * Conventions (all functions):
 *   - extern "C", never throw, never synchronise the host.  Thread-safe: per-device kernel
 *     attributes are set once per (kernel, device) under a lock; the error message is
 *     thread-local.
 *   - Every pointer argument is a DEVICE pointer unless its name ends in _host.
 *   - The caller owns every buffer (including the workspace); the library never
 *     allocates on the hot path, so calls are CUDA-graph capturable.
 *   - All argument checks run on the host before any launch; a non-OK status
 *     means nothing was enqueued.  After launching, cudaGetLastError() is
 *     mapped to TL_ECUDA.  Asynchronous device faults surface at the caller's
 *     next synchronisation.  tl_last_error() returns a thread-local message.
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *     default stream).
 *   - Pointers and row strides must be 16-byte aligned.
 *   - Shape support: K % 128 == 0, N % 128 == 0; group G divides K and is one of
 *     32, 64, 128 or a multiple of 128 (G == K is per-channel).  M >= 0; M == 0 is
 *     a no-op returning TL_OK.
 */
#ifndef TILUS_B200_H_
#define TILUS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Weight element type: the 4-byte dtype code of SPEC.md:276 (kind, bits, exp, man).
 * kind 0 = uint, 1 = int (two's complement), 2 = float (bias 2^(E-1)-1, subnormals,
 * no Inf/NaN -- reading R3).  Kernel formats: bits 1..8; float needs bits >= 3,
 * 1 <= exp <= 4, man = bits-1-exp >= 0 (reading R4) -- 37 formats in all. */
typedef struct {
  uint8_t kind;
  uint8_t bits;
  uint8_t exp_bits;
  uint8_t man_bits;
} tl_wtype;

/* Activation type: the dtype of A, of the scales, of the zero points and of Y (PAPER.md:170
 * "A ... float16"; "we also support bfloat16").  bf16 runs on the
 * tensor-core families (decode, batched, prefill); a TL_PATH_GEMV request with bf16 runs on the
 * decode / batched tensor-core kernel instead.  The dequantized weight is exact in fp16 and is
 * rounded once to bf16 where the MMA / GEMM operand is bf16 (reading R9). */
/* TL_ACT_I8 ("operand A can have data types with 32, 16, or 8 bits",
 * PAPER.md:527 "we also support ... int8"; reading R24): A is int8 [M,K] (lda in elements = bytes,
 * a multiple of 16); scales, zeros and Y are fp16.  Each int8 is the integer it encodes, so the
 * result is the same definition Y = fp16(sum_k A[m,k] * w[k,n]).  The library stages A exactly as
 * fp16 in the tail of the workspace (tl_matmul_workspace_bytes(.., TL_ACT_I8, ..) includes it) and
 * runs the fp16 families on the copy. */
typedef enum { TL_ACT_F16 = 0, TL_ACT_BF16 = 1, TL_ACT_I8 = 2 } tl_atype;

typedef enum {
  TL_OK = 0,
  TL_EINVAL_DTYPE = 1,  /* weight format not one of the 37 kernel formats      */
  TL_EINVAL_SHAPE = 2,  /* K, N not multiples of 128, negative M, bad strides   */
  TL_EINVAL_GROUP = 3,  /* G does not divide K or is not 32/64/128/128*j        */
  TL_EALIGN = 4,        /* pointer or stride not 16-byte aligned                */
  TL_EZEROS = 5,        /* zeros given for a non-uint format                    */
  TL_EWORKSPACE = 6,    /* workspace missing or smaller than required           */
  TL_EUNSUPPORTED = 7,  /* valid request outside what this build implements     */
  TL_ECUDA = 8,         /* a CUDA runtime call or launch failed                 */
  TL_ENULL = 9          /* a required pointer is NULL                           */
} tl_status;

/* Which kernel family tl_matmul uses (CUDA cores for few tokens, tensor cores for
 * more; on B200 the choice is re-measured):
 *   TL_PATH_GEMV  CUDA-core GEMV / skinny GEMM (FHFMA, fp32 accumulation), any M (16 rows per launch)
 *   TL_PATH_TC    tcgen05 GEMM, dequantized W^T in tensor memory, batch as MMA-N (any M)
 *   TL_PATH_TCD   tcgen05 decode kernel for M <= 16 and group a multiple of 128: W^T unpacked into
 *                 tensor memory as exact fp16 values, scale / zero point applied per tile in fp32,
 *                 launched with programmatic dependent launch (see TL_FLAG_STATIC_WEIGHTS).  Falls
 *                 back to TL_PATH_TC outside that range.
 *   TL_PATH_PREFILL  large M: the weight decoded to fp16 in L2-sized column chunks
 *                 of the workspace by this library's kernel, then a cuBLAS f16 x f16 GEMM with fp32
 *                 accumulation per chunk.  The workspace then holds up to 32 MB + 64 MB.
 * TL_PATH_AUTO: the measured dispatch rule. */
typedef enum { TL_PATH_AUTO = 0, TL_PATH_GEMV = 1, TL_PATH_TC = 2, TL_PATH_TCD = 3, TL_PATH_PREFILL = 4 } tl_path;

/* tl_matmul_ex / tl_matmul_hostio flags.
 *   TL_FLAG_STATIC_WEIGHTS  w_t, scales and zeros are not written by any kernel that may still be
 *     running on `stream` when this call is enqueued (e.g. resident model weights prepared long
 *     before).  The decode kernel (TL_PATH_TCD) is launched with programmatic dependent launch: its
 *     CTAs may start while the previous kernel in the stream is finishing.  With this flag its
 *     weight / scale / zero stream starts at once, overlapping that tail; A, Y and the workspace
 *     are touched only after griddepcontrol.wait (the previous grid completed, its writes
 *     visible).  Without the flag every read waits, so a transform or scale-producing kernel may
 *     directly precede the matmul: PTX guarantees the visibility of a prerequisite grid's writes
 *     only after griddepcontrol.wait. */
#define TL_FLAG_STATIC_WEIGHTS 1u

/* ---- sizes --------------------------------------------------------------- */

/* ceil(K*N*bits/8): bytes of the compact bitstream. */
size_t tl_packed_bytes(tl_wtype w, int64_t K, int64_t N);

/* Bytes of the transformed weight.  Equal to tl_packed_bytes for every legal
 * shape: the transform permutes bits and adds no padding (PAPER.md:187,
 * "u8[K/BK, N/BN, BK*BN*b/8]").  Returns 0 for an illegal shape. */
size_t tl_transformed_bytes(tl_wtype w, int64_t K, int64_t N);

/* Version of the opaque transformed layout; bumps whenever the layout changes. */
uint32_t tl_format_version(void);

/* ---- one-time weight preparation ------------------------------------------ */

/* Pack one code per byte (codes[K*N], row-major, each < 2^bits) into the compact
 * LSB-first bitstream (readings R1/R2).  bitstream must hold
 * tl_packed_bytes(w,K,N) bytes.  Codes are taken modulo 2^bits. */
tl_status tl_pack(tl_wtype w, int64_t K, int64_t N, const uint8_t* codes, uint8_t* bitstream,
                  void* stream);

/* Inverse of tl_pack (test hook): codes[K*N], one per byte. */
tl_status tl_unpack(tl_wtype w, int64_t K, int64_t N, const uint8_t* bitstream, uint8_t* codes,
                    void* stream);

/* The paper's "Change Layout" step: re-lay the
 * bitstream out into 128x128 tiles whose bytes are in the order the kernels'
 * threads load and unpack them.  w_t must hold
 * tl_transformed_bytes(w,K,N) bytes and must not alias bitstream. */
tl_status tl_transform_weights(tl_wtype w, int64_t K, int64_t N, const uint8_t* bitstream,
                               void* w_t, void* stream);

/* Exact inverse of tl_transform_weights (test hook). */
tl_status tl_untransform_weights(tl_wtype w, int64_t K, int64_t N, const void* w_t,
                                 uint8_t* bitstream, void* stream);

/* ---- the hot path ------------------------------------------------------------ */

/* Workspace bytes tl_matmul needs for this problem (split-K partials and tile semaphores): the
 * global workspace of the paper's runtime, which kernels request via AllocateGlobal
 * (PAPER.md:439-440), here owned by the caller so calls stay graph-capturable.
 * The workspace must be ZERO-FILLED once when allocated; the kernels leave every semaphore at zero
 * again when they finish, so it can be reused by any later call on the same stream without
 * clearing.  Returns 0 for an unknown activation type. */
size_t tl_matmul_workspace_bytes(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group);

/* Y[M,N] (row stride ldy elements) = A[M,K] (row stride lda elements) x dequant(w_t): the paper's
 * C = A x B with fp32 accumulation cast to the activation type.
 * A, scales and Y have type `a` (for TL_ACT_I8: A int8, scales / zeros / Y fp16).  scales: [K/G, N] row-major.  zeros: [K/G, N] with integer
 * values, uint formats only, or NULL (z = 0).  Enqueued on `stream`; no flags: every read is
 * ordered after the previous kernel in the stream. */
tl_status tl_matmul(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group, const void* A,
                    int64_t lda, const void* w_t, const void* scales, const void* zeros, void* Y,
                    int64_t ldy, void* workspace, size_t workspace_bytes, void* stream);

/* As tl_matmul with an explicit kernel family (tl_path), split-K grid (0 = auto; requests above
 * the CTA count the workspace is sized for are clamped to it) and flags (TL_FLAG_*); used by the
 * bench, the dispatch sweep and the tests. */
tl_status tl_matmul_ex(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group,
                       const void* A, int64_t lda, const void* w_t, const void* scales,
                       const void* zeros, void* Y, int64_t ldy, void* workspace, size_t workspace_bytes,
                       int32_t path, int32_t splits, uint32_t flags, void* stream);

/* End-to-end variant for host buffers: copies A_host [M,K] (pinned recommended)
 * into the device staging buffer A_dev, runs tl_matmul into Y_dev and copies
 * Y_dev back into Y_host [M,N], all on `stream` (no host sync).  Weights,
 * scales and zeros stay resident on the device (flags as tl_matmul_ex). */
tl_status tl_matmul_hostio(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group,
                           const void* A_host, void* A_dev, const void* w_t, const void* scales,
                           const void* zeros, void* Y_dev, void* Y_host, void* workspace,
                           size_t workspace_bytes, uint32_t flags, void* stream);

/* One matmul of a batched host-buffer call (tl_matmul_batch_hostio): the weight of one linear layer and
 * its own batch M, as tl_matmul's arguments (device pointers). */
typedef struct {
  tl_wtype w;
  int32_t group;
  int64_t M, N, K;
  const void* w_t;
  const void* scales;
  const void* zeros;        /* NULL unless uint with zero points */
  void* workspace;          /* tl_matmul_workspace_bytes(w, a, M, N, K, group) bytes, zero-filled once; */
  size_t workspace_bytes;   /* items may share one workspace (they run in stream order) */
} tl_batch_item;

/* End-to-end call for several matmuls whose activations arrive in ONE host buffer and whose outputs
 * return in ONE host buffer (e.g. the linear layers of a decode step): one host->device copy of
 * A_host (the items' A [M_i, K_i] row-major, concatenated in item order, each block starting at a
 * multiple of 16 bytes -- automatic, since K % 128 == 0) into A_dev, the items' matmuls on `stream`
 * in order (TL_PATH_AUTO, `flags` as tl_matmul_ex; consecutive decode launches overlap through
 * programmatic dependent launch), Y_i into Y_dev (concatenated likewise), and one device->host copy
 * of Y_dev into Y_host.  A_dev / Y_dev hold sum_i M_i K_i and sum_i M_i N_i elements of type `a`
 * (int8 A for TL_ACT_I8).  No host synchronisation.  Errors as tl_matmul_ex for the first failing
 * item (items before it are enqueued), TL_EINVAL_SHAPE for count < 0, TL_ENULL for NULL buffers. */
tl_status tl_matmul_batch_hostio(tl_atype a, int32_t count, const tl_batch_item* items, const void* A_host,
                                 void* A_dev, void* Y_dev, void* Y_host, uint32_t flags, void* stream);

/* Which family (tl_path) and split-K grid (CTAs; 0 = the CUDA-core path's occupancy-sized grid)
 * tl_matmul would use for this problem on the current device (for the bench and the dispatch
 * sweep).  The rule is DESIGN.md "Dispatch". */
tl_status tl_matmul_plan(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group,
                         int32_t* path_out, int32_t* splits_out);

/* ---- row f3: gathered output over NVLink peer memory --------------------------------------------- */

/* Column-sharded matmul with the all-gather FUSED into the epilogue (north star
 * (5); output column n depends only on W[:, n], so a column shard computes alone).
 * Rank r owns columns [n0, n1) of an [M, N_total] layer; every rank holds a gathered buffer
 * Yg[M, N_total] (row stride ldy) and a flag array flags[nranks] (uint32, zero-initialised, never
 * reset).  This call computes the rank's shard exactly like tl_matmul (A, w_t, scales, zeros are the
 * shard's; N = n1 - n0) into Y = &Yg_local[0, n0], and the kernel's epilogue also stores every
 * finished element into each peer's gathered buffer: Y_peers[i] = device address, mapped into this
 * process (CUDA IPC / peer access over NVLink), of &Yg_peer_i[0, n0] with the same ldy.  When the
 * last element is stored, the kernel releases +1 (system scope) on flag_peers[i] = &flags_peer_i[r].
 * The fused epilogue runs in the decode and batched tensor-core kernels; the other families compute
 * locally and then replicate with one copy-and-signal kernel.  Y_peers / flag_peers are HOST arrays
 * of npeers <= 7 device pointers (npeers = 0: a plain tl_matmul).  Ordering contract: the caller
 * must not start call e+1 into a peer's buffer before that peer has consumed call e (alternate two
 * gathered buffers, or rely on the layer dependency).  M == 0 sends and signals nothing.  Errors as
 * tl_matmul_ex, plus TL_EINVAL_SHAPE for npeers outside [0, 7], TL_ENULL / TL_EALIGN for peer
 * pointers (Y 16-byte, flag 4-byte aligned). */
tl_status tl_matmul_gathered(tl_wtype w, tl_atype a, int64_t M, int64_t N, int64_t K, int32_t group,
                             const void* A, int64_t lda, const void* w_t, const void* scales,
                             const void* zeros, void* Y, int64_t ldy, void* const* Y_peers,
                             uint32_t* const* flag_peers, int32_t npeers, void* workspace,
                             size_t workspace_bytes, uint32_t flags, void* stream);

/* Consumer side of tl_matmul_gathered: enqueue on `stream` a wait until every other rank q != self
 * has completed `epoch` gathered calls into this rank (flags[q] >= epoch, wrap-safe; flags is this
 * rank's own device array [nranks]).  Kernels enqueued after it on `stream` see the peers' stores.
 * The wait is bounded (TL_GATHER_TIMEOUT_MS, default 10000): a peer that never arrives makes the
 * wait kernel trap (a CUDA launch failure at the next synchronisation) instead of hanging.
 * TL_EINVAL_SHAPE unless 1 <= nranks <= 8 and 0 <= self < nranks; TL_ENULL for NULL flags. */
tl_status tl_gather_wait(const uint32_t* flags, int32_t nranks, int32_t self, uint32_t epoch, void* stream);

/* Row-parallel (K-sharded) variant of row f3.  Rank r holds the K rows [k0, k1) of the weight (k0, k1
 * multiples of 128 and of the group) and computes, with tl_matmul on A[:, k0:k1], a PARTIAL
 * P_r[M, N_total] = A[:, k0:k1] x dequant(W[k0:k1, :]) in the activation type.  After its matmul a
 * rank calls tl_signal_peers (release +1, system scope, on flags_q[r] of every peer q, ordered after
 * the stream's prior work); every rank then waits for the others (tl_gather_wait on its own flags)
 * and reduces its column block [n0, n1) over NVLink:
 *   Y[m, c] = fp16( sum_{q = 0 .. nranks-1} P_q[m, n0 + c] )  in fp32, in rank order (deterministic).
 * parts[q] (HOST array of nranks device pointers, peer-mapped) = &P_q[0, n0], row stride ldp; Y =
 * the rank's output block [M, N = n1 - n0] (row stride ldy).  N, ldp, ldy multiples of 8; pointers
 * 16-byte aligned; a in {TL_ACT_F16, TL_ACT_BF16}.  The partials are rounded once to the activation
 * type before the sum (reading R26).  The caller must not overwrite P_r for call e+1 before every
 * peer has reduced call e (alternate two partial buffers).  Errors: TL_EINVAL_SHAPE, TL_ENULL,
 * TL_EALIGN, TL_EUNSUPPORTED (other activation types). */
tl_status tl_signal_peers(uint32_t* const* flag_peers, int32_t npeers, void* stream);
tl_status tl_reduce_scatter_peer(tl_atype a, const void* const* parts, int32_t nranks, int64_t M, int64_t N,
                                 int64_t ldp, void* Y, int64_t ldy, void* stream);

/* Microscaling scales ("Microscaling data types can be thought as
 * a more fine-grained quantization thus we could also support it"; reading R25).  An MX weight is a
 * kernel format (fp4 e2m1, fp6 e2m3 / e3m2, fp8 e4m3, or int8 for MXINT8) with ONE E8M0 scale per
 * block of 32 weights along K: pass group = 32 to tl_matmul with the fp16 scales this call writes.
 * e8m0[count] (device, any layout -- conventionally [K/32, N]) holds exponent codes e; scales_f16
 * [count] (device) receives 2^(e - 127 + exp_adjust) as fp16 (exp_adjust = -6 for MXINT8, whose
 * elements carry an implicit 2^-6; 0 otherwise).  Exact whenever the value is an fp16 number
 * (2^-24 .. 2^15); outside that range, and for the E8M0 NaN code 0xFF, the scale is an fp16 NaN (the
 * block's outputs become NaN rather than silently wrong).  One-time weight preparation, enqueued on
 * `stream`.  TL_EINVAL_SHAPE for count < 0 or |exp_adjust| > 64, TL_ENULL for NULL pointers. */
tl_status tl_mx_scales_to_f16(const uint8_t* e8m0, int64_t count, int32_t exp_adjust, void* scales_f16,
                              void* stream);

/* The same conversion into bf16 scales, for bf16 activations (scales have the activation type): bf16
 * carries E8M0's 8 exponent bits, so with exp_adjust = 0 every code except the NaN code 0xFF is
 * exact (e = 0 is the bf16 subnormal 2^-127); values outside 2^-133 .. 2^127 and 0xFF become NaN.
 * Errors as tl_mx_scales_to_f16. */
tl_status tl_mx_scales_to_bf16(const uint8_t* e8m0, int64_t count, int32_t exp_adjust, void* scales_bf16,
                               void* stream);

/* Test hook: out[K,N] fp32 = (value(q) - z) * s, computed exactly in fp32 from
 * the TRANSFORMED weight (reading R9: exact, so it is bit-comparable with the
 * oracle's dequant). */
tl_status tl_dequant(tl_wtype w, int64_t K, int64_t N, int32_t group, const void* w_t,
                     const void* scales, const void* zeros, float* out, void* stream);

/* ---- errors -------------------------------------------------------------- */
const char* tl_status_str(tl_status s);
const char* tl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TILUS_B200_H_ */
