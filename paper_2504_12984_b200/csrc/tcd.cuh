// tcd.cuh -- decode-batch tensor-core path (M <= 16, group a multiple of 128): SURVEY §8(a)
// rows a3-a11 for the HBM-bound regime ("for small batch sizes the primary
// bottleneck is loading weights from global memory to registers").
//
// Swap-AB tcgen05.mma.cta_group::1.kind::f16: M_mma = 128 weight columns (the dequantized W^T
// tile, written to TENSOR MEMORY with tcgen05.st -- the "TS" form), N_mma = 16 batch rows (the
// activation operand, 128B-swizzled K-major in shared memory, rows >= M zero-filled by the TMA
// unit), fp32 accumulation in TMEM.  The per-weight work is the unpack alone:
//
//  * integer codes (layout v2, common.cuh): one LOP3 per pair (more for the few "spare" codes)
//    places the code at bits [P, P+b) of each half under the fp16 magic 0x6400 (1024 + u*2^P),
//    and one HFMA2 with the per-tile constant -(2^(10-P) + z) yields u - z EXACTLY in fp16, so the
//    MMA accumulates D = sum_k A[m,k] (u[k,n] - z) with no further conversion; ints are stored
//    offset-binary (zero point 2^(b-1));
//  * float codes are placed on the fp16 sign / exponent / mantissa fields (value * 2^(bias-15),
//    exact) by the LOP3s alone;
//  * the group scale is applied once per (tile, column, batch row) in fp32:
//        Y[m,n] += s[g,n] * D[n,m]      (floats: s[g,n] * 2^(15-bias) * D[n,m]).
//
// A ring stage holds R consecutive packed weight tiles (2048*b B each, ONE cp.async.bulk,
// PAPER.md:148-151 step (1)) and their scale and zero-point row slices (256 B each, 8-byte cp.async
// by warp 3 completing on the same stage barrier); the activation operand has its own ring.
// Roles (128 + 128*NG threads):
//   warp 0       weight-stream TMA producer (one elected thread)
//   warp 1       TMEM allocator + MMA issuer (one elected thread)
//   warp 2       activation operand: M > 1 a TMA producer (2-D tensor map); M = 1 the operand
//                WRITER (A[0, :] resident in shared memory, one row per tile, see TcdCfg)
//   warp 3       scale / zero stager (cp.async into the stage's side area)
//   warps 4..    NG dequant groups of 4 warps (warp%4 = TMEM lane quarter = 32 columns); group
//                g handles tiles t = g, g+NG, ... of the CTA's stream-K range: unpack into its
//                W^T slot, hand it to the MMA, then -- TcdCfg::Lag group-iterations late, so it never
//                waits for its own MMA -- read the tile's accumulator and apply the fp32 fixup.
// Stream-K: the linear unit space u = nt*KT + kt is cut into `grid` contiguous
// ranges; n-tiles shared by several CTAs are reduced in fixed CTA order (reading R12).
#pragma once

#include <cuda.h>

#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

struct TcdParams {
  int M, N, K, G;
  int units;
  int ns;                          // TMA ring stages
  int R;                           // tiles per stage (consecutive units: one contiguous weight copy)
  uint32_t stage_bytes;            // [R weight tiles | R scale row slices | R zero row slices]
  uint32_t stash_off;              // decode: A[0, 0:K] resident in shared memory (K*2 bytes)
  int rot;                         // 1: decode configuration TcdCfg<1> (M = 1, K*2 <= 64 KB)
  int bf;                          // 1: bf16 activations / scales / zeros / Y (Act<true>)
  uint32_t op_off, red_off, bar_off;  // operand ring [NOP][4 KB] (1024-aligned), reduction, barriers
  const uint8_t* wt;
  const __half* A;
  int64_t lda;
  const __half* scales;
  const __half* zeros;
  __half* Y;
  int64_t ldy;
  float* partial;  // [grid][2][16][128] fp32
  int* sem;
  long long* trace;  // optional [grid][16] %globaltimer stamps (TL_TRACE)
  uint32_t magic;  // 0x64006400, a kernel argument so that AND-mask + OR-magic fuse into ONE LOP3
                   // (LOP3 takes one immediate; the magic must live in a register)
  int static_w;  // TL_FLAG_STATIC_WEIGHTS: the weight stream may start before griddepcontrol.wait
  PeerOut po;  // row f3: gathered output fused into the epilogue (peer.cuh); po.n == 0: local only
  int dbg;  // experiment knobs (TL_TCD_DBG; device-side ones only with -DTCD_TRACE): 1 skip MMAs, 16 skip fixups, 64 stream only, 1024 no scale stager,
            // 4 skip unpack/STTM, 8 skip scale/zero copies, 128 no PDL (host)
};

constexpr int kTcdNG = 4;                       // dequant groups
// TMEM budget (512 columns) per batch tile MT:
//  * MT == 16: NW = 5 W^T slots (64 columns each) + 12 accumulators of 16 columns (one per tile in
//    flight, slot t % 12), fixups lag 2 group iterations (the accumulator of tile t - NACC must be
//    read by its group before that group arrives for tile t: 4*lag < NACC);
//  * MT == 1 (decode): the activation row of tile t is placed in operand row t % 16 (TMA box
//    starting at row -(t % 16); the other rows are zero-filled), so tile t's result lands in
//    accumulator COLUMN t % 16 and 16 consecutive tiles share one 16-column block: the first MMA of
//    tile 16e (accumulate = 0) clears block e % 2, the others accumulate.  Two blocks (32 columns)
//    leave room for NW = 7 W^T slots, so the dequant groups are not throttled by the slot ring.
//    NACC is then only the ring of "MMA(t) complete" barriers.  The activation row A[0, :] is
//    resident in shared memory (one bulk copy) and warp 2 WRITES each tile's operand: slot t % 8
//    gets A[0, kt*128 : kt*128+128] in row t % 16 and the row it held for tile t - 8 zeroed --
//    256 + 256 bytes of st.shared per tile instead of a 4 KB TMA box (the stream of small TMA
//    copies, not HBM, was the decode kernel's throughput limit).
template <int MT>
struct TcdCfg {
  static constexpr bool kRot = MT == 1;                  // row rotation (decode)
#ifndef TCD_NW_ROT
#define TCD_NW_ROT 5
#endif
#ifndef TCD_NG_ROT
#define TCD_NG_ROT 4
#endif
  static constexpr int NG = kRot ? TCD_NG_ROT : 4;       // dequant groups of 4 warps
  static constexpr int Threads = 128 + NG * 128;
  static constexpr int NW = kRot ? (TCD_NW_ROT > NG ? TCD_NW_ROT : NG + 1) : 5;  // W^T slots
  static constexpr int NACC = kRot ? 16 : 12;            // completion barriers (= accumulators if !kRot)
  static constexpr int Lag = kRot ? 2 : NACC / 4 - 1;    // fixup lag (group iterations)
  static constexpr uint32_t AccCol = 64 * NW;            // first accumulator column
  // activation operand ring: slot t % NOP is refilled once MMA(t - NOP) completed, so the
  // operand of tile t is in flight for NOP tiles (an L2 round trip); NOP <= NACC keeps the
  // completion-barrier parity unambiguous
  // decode: NOP slots; with 16, slot t % 16 always holds row t % 16 (never zeroed again).  Measured
  // 8 vs 16: the same time on every 70B layer (DESIGN.md §6 experiments), so the default keeps the
  // smaller ring (32 KB more for weight stages).
#ifndef TCD_NOP_ROT
#define TCD_NOP_ROT 8
#endif
  static constexpr int NOP = kRot ? TCD_NOP_ROT : 8;
  static_assert(NOP <= NACC, "operand ring vs completion ring");
  static_assert(AccCol + (kRot ? 32 : NACC * 16) <= 512, "TMEM split");
  static_assert(NACC % 4 == 0 && Lag >= 1 && Lag <= 2 && NG * Lag < NACC, "fixup lag");
  static_assert(kRot || NACC % NG == 0, "per-tile accumulators: the fixup of tile t - NACC is its group's");
};
constexpr int kTcdMaxNW = 7, kTcdMaxNACC = 16;  // shared-memory sizing of the barrier arrays
constexpr int kTcdThreads = 128 + kTcdNG * 128;
constexpr int kTcdNB = 16;                      // MMA N (batch rows, zero-padded)
constexpr uint32_t kTcdOpBytes = kTcdNB * 256;  // 16 rows x 128 k fp16, two 64-k SW128 blocks
constexpr int kTcdMaxNOP = 16;                  // activation operand ring slots (max over configs)

__device__ __forceinline__ void tcd_sttm_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ uint32_t tcd_ldtm_x1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return r;
}
// D[tmem] (+)= A[tmem] * B[smem], kind::f16
__device__ __forceinline__ void tcd_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// shared-memory matrix descriptor: K-major, 128B swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t tcd_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// the 4b words of column n of a transformed tile in shared memory (b 16-byte loads)
template <int B>
__device__ __forceinline__ void tcd_load_words(uint32_t wtile, int n, uint32_t* words) {
#pragma unroll
  for (int v = 0; v < B; ++v) {
    const uint4 x = lds128(wtile + (v * 128 + n) * 16);
    words[4 * v + 0] = x.x;
    words[4 * v + 1] = x.y;
    words[4 * v + 2] = x.z;
    words[4 * v + 3] = x.w;
  }
}

// is P the field position of some pair of the format's plan (ints)?
template <class F>
__host__ __device__ constexpr bool plan_uses_p(int P) {
  for (int i = 0; i < 32; ++i)
    if (kPlan<F::kind, F::bits, F::exp>.pr[i].P == P) return true;
  return false;
}

// Pipeline tracing (tools/trace_tcd.py, tools/trace_pdl.py): compiled in only with -DTCD_TRACE,
// so the production kernel carries no trace branches.
#ifdef TCD_TRACE
#define TCD_TRACE_ON 1
#else
#define TCD_TRACE_ON 0
#endif
__device__ __forceinline__ void tcd_stamp(const TcdParams& p, int i) {
  if (TCD_TRACE_ON && p.trace != nullptr) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * 16 + i] = t;
  }
}
__device__ __forceinline__ void tcd_tstamp(const TcdParams& p, int idx) {  // clock64 of CTA 0
  if (TCD_TRACE_ON && p.trace != nullptr && blockIdx.x == 0) p.trace[idx] = clock64();
}

// per-iteration clock64 stamps of CTA 0, group 0, warp 0, lane 0: [iter][8] at 2400
__device__ __forceinline__ void tcd_istamp(const TcdParams& p, int dw, int lane, uint32_t kk, int i) {
  if (TCD_TRACE_ON && p.trace != nullptr && blockIdx.x == 0 && dw == 0 && lane == 0 && kk < 40)
    p.trace[2400 + kk * 8 + i] = clock64();
}

// tiles per weight stage: ~12 KB of packed weights per stage (the cp.async.bulk ring streams at
// full HBM rate only with stages of ~12 KB and more, tools/tma_probe.cu)
#ifndef TCD_STAGE_UNITS
#define TCD_STAGE_UNITS 6
#endif
__host__ __device__ constexpr int tcd_tiles_per_stage(int b) { return (TCD_STAGE_UNITS + b - 1) / b; }

template <class F, int MT, bool BF>
__global__ void __launch_bounds__(TcdCfg<MT>::Threads, 1) tcd_kernel(const __grid_constant__ CUtensorMap tmapA, TcdParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr bool kInt = F::kind != kFloat;  // integer codes: magic form + HFMA2 (u - z)
  constexpr uint32_t WB = tile_bytes(F::bits);
  constexpr int kR = tcd_tiles_per_stage(F::bits);
  using Cfg = TcdCfg<MT>;
  constexpr int NG = Cfg::NG, NACC = Cfg::NACC, kTcdNW = Cfg::NW;
  constexpr uint32_t kTcdAccCol = Cfg::AccCol;
  constexpr int kTcdNOP = Cfg::NOP;
  const int NS = p.ns;
  const uint32_t SB = p.stage_bytes;
  const uint32_t st_u = smem_u32(smem);
  float* red = reinterpret_cast<float*>(smem + p.red_off);  // [NG][M][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* full_tma = bars;                    // [NS] stage landed
  uint64_t* empty_tma = bars + NS;              // [NS] group read the stage
  uint64_t* full_op = bars + 2 * NS;            // [NOP] activation operand landed
  uint64_t* empty_op = full_op + kTcdMaxNOP;    // [NOP] (unused: the operand slot is freed by MMA completion)
  uint64_t* full_w = empty_op + kTcdMaxNOP;  // [NW] W^T slot written
  uint64_t* empty_w = full_w + kTcdMaxNW;  // [NW] MMA done with the W^T slot
  // [NACC] "MMA(t) complete" (one tcgen05.commit per tile, slot t % NACC).  It also frees the W^T
  // slot and the operand slot of tile t.  No accumulator-empty barrier is needed: the fixup of
  // tile t - NACC is done by the same group (NACC % NG == 0) before it arrives on full_w for t.
  // Every waiter for MMA(j) provably waits before MMA(j + NACC) can complete (parity is safe).
  uint64_t* full_acc = empty_w + kTcdMaxNW;
  uint64_t* empty_acc = full_acc + kTcdMaxNACC;  // [NACC] accumulator read back
  uint64_t* stash_bar = empty_acc + kTcdMaxNACC; // decode: A[0, :] landed in the stash
  uint32_t* tslot_ptr = reinterpret_cast<uint32_t*>(stash_bar + 1);
  int* flag = reinterpret_cast<int*>(tslot_ptr + 4);

  const int KT = p.K / kBK;
  const int grid = gridDim.x;
  const int cta = blockIdx.x;
  const int u0 = (int)((int64_t)cta * p.units / grid);
  const int u1 = (int)((int64_t)(cta + 1) * p.units / grid);
  const int T = u1 - u0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool has_zeros = F::kind == kUint && p.zeros != nullptr;

  if (threadIdx.x == 0) {
    tcd_stamp(p, 0);
    if (TCD_TRACE_ON && p.trace) p.trace[blockIdx.x * 16 + 10] = T;
    for (int s = 0; s < NS; ++s) {
      // the weight TMA (arrive + tx) and warp 3's 32 cp.async lanes (1024: timing experiment, no stager)
      mbar_init(&full_tma[s], (TCD_TRACE_ON && (p.dbg & 1024)) ? 1 : 1 + 32);
      mbar_init(&empty_tma[s], 4 * kR);  // every tile of the stage: its group's 4 warps
    }
    mbar_init(stash_bar, 1);
    for (int i = 0; i < kTcdNOP; ++i) {
      mbar_init(&empty_op[i], 1);
      mbar_init(&full_op[i], 1);
    }
    for (int i = 0; i < kTcdNW; ++i) {
      mbar_init(&full_w[i], 4);
      mbar_init(&empty_w[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&full_acc[i], 1);
      mbar_init(&empty_acc[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tslot_ptr, 512);
    tmem_relinquish();
  }
  if constexpr (Cfg::kRot) {
    // decode: every operand row starts at zero; the writer only ever touches one row per tile
    uint4* z = reinterpret_cast<uint4*>(smem + p.op_off);
    for (int i = threadIdx.x; i < kTcdNOP * (int)kTcdOpBytes / 16; i += Cfg::Threads) z[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
  }
  const uint32_t op_u = st_u + p.op_off;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot_ptr;
  if (threadIdx.x == 0) tcd_stamp(p, 1);
  // Programmatic dependent launch: with TL_FLAG_STATIC_WEIGHTS the weight stream (warp 0) depends on
  // nothing a kernel still running in the stream writes, so it starts right away; otherwise warp 0
  // too waits for the previous grid (which may have produced the weights / scales: only
  // griddepcontrol.wait makes its writes visible).  Every other warp waits before it reads A or
  // touches Y / the workspace.
  if (warp == 0) {
    if (!p.static_w) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else if (warp == 3) {
    if (!p.static_w) asm volatile("griddepcontrol.wait;" ::: "memory");  // scales / zeros
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 64) tcd_stamp(p, 11);
  }

  if (warp == 0 || warp == 2) {
    // ------------------------------ TMA producers ------------------------------
    // warp 0: the stage = packed weight tile + its scale / zero-point row slices (HBM streams,
    // gated only by the stage ring); warp 2: the activation operand of the tile (two 64-k x 16-row
    // boxes from L2, 128B-swizzled by the TMA unit, rows >= M zero-filled), gated by the operand
    // ring that the MMA releases.  Separate issuers keep the weight stream from ever waiting on
    // the MMA.
    if (elect_one()) {
      const uint64_t pol_first = policy_evict_first();
      const uint64_t pol_last = policy_evict_last();
      int nt = u0 / KT, kt = u0 - (u0 / KT) * KT;
      if (warp == 0) {
        // stage q = tiles [q*R, q*R + R) of the CTA's range: ONE bulk copy of their contiguous
        // packed bytes (consecutive units are adjacent in the n-tile-major layout).  Large stages:
        // the streaming rate of cp.async.bulk rings grows with the bytes per stage (measured,
        // tools/tma_probe.cu), so small-b tiles are grouped.  Scales / zero points are not in the
        // stage: the dequant threads load their own (2 bytes each), 16 tiles ahead.
        const uint32_t bar0 = smem_u32(full_tma);
        const uint8_t* src = p.wt + (int64_t)u0 * WB;
        int s = 0;
        uint32_t ph = 0;
        constexpr int R = kR;
        for (int t0 = 0, q = 0; t0 < T; t0 += R, ++q) {
          const int n_t = min(R, T - t0);
          if (q >= NS) {
            if (TCD_TRACE_ON && (p.dbg & 512)) mbar_wait(&empty_tma[s], ph ^ 1);
            else mbar_wait_sleepy(&empty_tma[s], ph ^ 1);
          }
          if (t0 < 64) tcd_tstamp(p, 2720 + t0);
          const uint32_t st = st_u + s * SB, bar = bar0 + 8 * s;
          mbar_arrive_expect_tx_u32(bar, (uint32_t)n_t * WB);
          tma_bulk_g2s_cta(st, src, (uint32_t)n_t * WB, bar, pol_first);
          if (t0 == 0) tcd_stamp(p, 2);
          if (t0 + n_t == T) tcd_stamp(p, 3);
          src += (int64_t)n_t * WB;
          if (++s == NS) {
            s = 0;
            ph ^= 1;
          }
        }
      } else if constexpr (!Cfg::kRot) {
        prefetch_tmap(&tmapA);
        int o = 0;
        for (int t = 0; t < T; ++t) {
          // operand slot t % NOP is free once MMA(t - NOP) completed (mma_done slot (t - NOP) % NACC)
          if (t >= kTcdNOP) mbar_wait(&full_acc[(t - kTcdNOP) % NACC], (uint32_t)((t - kTcdNOP) / NACC) & 1);
          uint8_t* opp = smem + p.op_off + o * kTcdOpBytes;
          mbar_arrive_expect_tx(&full_op[o], kTcdOpBytes);
          tma_load_2d(opp, &tmapA, kt * kBK, 0, &full_op[o], pol_last);
          tma_load_2d(opp + kTcdNB * 128, &tmapA, kt * kBK + 64, 0, &full_op[o], pol_last);
          if (++kt == KT) kt = 0;
          if (++o == kTcdNOP) o = 0;
        }
      }
    }
    if constexpr (Cfg::kRot) {
      if (warp == 2) {
        // ---- decode operand writer (whole warp): A[0, :] arrived in the stash (prologue); slot
        // o = t % 8 gets A[0, kt*128 .. +128) in row r = t % 16 (128B-swizzled K-major: two 64-k
        // blocks of 16 rows x 128 B; 16-byte chunk c of row r at chunk c ^ (r % 8)) and the row it
        // held for tile t - 8, (r + 8) % 16, zeroed.  Lane l moves k = 4l .. 4l+3.
        if (lane == 0) {  // after griddepcontrol.wait: A is the previous grid's output
          mbar_arrive_expect_tx(stash_bar, (uint32_t)p.K * 2u);
          tma_bulk_g2s(smem + p.stash_off, p.A, (uint32_t)p.K * 2u, stash_bar, policy_evict_last());
        }
        mbar_wait(stash_bar, 0);
        const uint8_t* stash = smem + p.stash_off;
        const int kb = lane >> 4, c = (lane & 15) >> 1, half = lane & 1;
        int kt = u0 - (u0 / KT) * KT;
        int o = 0;
        for (int t = 0; t < ((TCD_TRACE_ON && (p.dbg & 64)) ? 0 : T); ++t) {
          if (t >= kTcdNOP) mbar_wait(&full_acc[(t - kTcdNOP) % NACC], (uint32_t)((t - kTcdNOP) / NACC) & 1);
          const uint2 v = *reinterpret_cast<const uint2*>(stash + kt * 256 + lane * 8);
          const int r = t & 15, rz = (t + 8) & 15;
          uint8_t* slot = smem + p.op_off + o * kTcdOpBytes + kb * (kTcdNB * 128);
          *reinterpret_cast<uint2*>(slot + r * 128 + ((c ^ (r & 7)) << 4) + half * 8) = v;
          if constexpr (kTcdNOP != 16)  // with 16 slots, slot t % 16 only ever holds row t % 16
            *reinterpret_cast<uint2*>(slot + rz * 128 + ((c ^ (rz & 7)) << 4) + half * 8) = make_uint2(0u, 0u);
          fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
          __syncwarp();
          if (lane == 0) mbar_arrive(&full_op[o]);
          if (++kt == KT) kt = 0;
          if (++o == kTcdNOP) o = 0;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (one thread) ------------------------------
    // the dequant group has already seen the tile's activation operand land (full_op) before it
    // arrives on full_w, so the issuer waits only for the W^T slot and the accumulator
    if (!(TCD_TRACE_ON && (p.dbg & 64)) && elect_one()) {
      const uint32_t idesc =
          (1u << 4) | Act<BF>::idesc_ab | ((uint32_t)(kTcdNB >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      int o = 0, g = 0, a = 0;
      uint32_t kk = 0, ka = 0;  // t / NW, t / NACC
      for (int t = 0; t < T; ++t) {
        mbar_wait(&full_w[g], kk & 1);
        if (t < 64) tcd_tstamp(p, 2976 + 3 * t);
        if (t < 64) tcd_tstamp(p, 2977 + 3 * t);
        tc_fence_after();
        const uint64_t bd = tcd_sw128_desc(op_u + o * kTcdOpBytes);
        // accumulator: decode -> block (t / 16) % 2, cleared by the first MMA of tile 16e only;
        // otherwise accumulator t % NACC, cleared by the tile's first MMA
        const uint32_t d = Cfg::kRot ? tmem + kTcdAccCol + ((t >> 4) & 1) * kTcdNB : tmem + kTcdAccCol + a * kTcdNB;
        const uint32_t first = Cfg::kRot ? ((t & 15) == 0 ? 0u : 1u) : 0u;
        const uint32_t aw = tmem + g * 64;
        if (!(TCD_TRACE_ON && (p.dbg & 1)))
#pragma unroll
        for (int j = 0; j < 8; ++j)
          tcd_mma_ts(d, aw + j * 8, bd + (uint64_t)((j >> 2) * (kTcdNB * 128 / 16) + (j & 3) * 2), idesc,
                     j > 0 ? 1u : first);
        tc_commit(&full_acc[a]);  // "MMA(t) complete": frees W^T slot t%NW, operand slot t%NOP, fills acc t%NACC
        if (t < 64) tcd_tstamp(p, 2978 + 3 * t);
        if (t == T - 1) tcd_stamp(p, 8);
        if (++o == kTcdNOP) o = 0;
        if (++g == kTcdNW) {
          g = 0;
          ++kk;
        }
        if (++a == NACC) {
          a = 0;
          ++ka;
        }
      }
    }
  } else if (warp == 3) {
    if (TCD_TRACE_ON && (p.dbg & 1024)) {
      // timing experiment: no scale / zero stager (the stage barrier expects the weight TMA only)
    } else {
    // ---- scale / zero stager: tile t's row slices s[g, nt*128 : +128] and z[g, ...] (256 B each)
    // go into the side area of its stage (after the R weight tiles).  Lane l copies columns
    // 4l .. 4l+3 with 8-byte cp.async (global -> shared, no registers), and after the stage's
    // last tile each lane arrives on the stage's full barrier when its copies have landed
    // (cp.async.mbarrier.arrive.noinc), so the stager runs as far ahead as the ring allows.
    const int tpg = p.G / kBK;
    int ntf = u0 / KT, ktf = u0 - (u0 / KT) * KT;
    int growf = ktf / tpg, gremf = ktf - growf * tpg;
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0, j = 0; t < T; ++t) {
      if (j == 0 && t >= NS * kR) {
        if (TCD_TRACE_ON && (p.dbg & 512)) mbar_wait(&empty_tma[s], ph ^ 1);  // 512: spinning waits
        else mbar_wait_sleepy(&empty_tma[s], ph ^ 1);
      }
      const uint32_t side = st_u + s * SB + kR * WB + 256 * j + 8 * lane;
      const int64_t off = (int64_t)growf * p.N + (int64_t)ntf * kBN + 4 * lane;
      if (!(TCD_TRACE_ON && (p.dbg & 256))) {  // 256: timing experiment, no scale / zero copies
        cp_async_8(side, p.scales + off);
        if (has_zeros) cp_async_8(side + kR * 256, p.zeros + off);
      }
      if (++ktf == KT) {
        ktf = 0;
        ++ntf;
        growf = 0;
        gremf = 0;
      } else if (++gremf == tpg) {
        gremf = 0;
        ++growf;
      }
      if (++j == kR || t == T - 1) {
        cp_async_mbar_arrive_noinc(&full_tma[s]);
        j = 0;
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    }
  } else {
    // ------------------------------ dequant groups ------------------------------
    const int dw = warp - 4;
    const int g = dw >> 2;
    const int q = warp & 3;
    const int n = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int wsl = g;          // W^T slot of the current tile (t % NW) and its lap (t / NW)
    uint32_t lapw = 0;
    const float c1mul = kInt ? 1.f : (float)(1 << (15 - F::bias));
    float tot[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) tot[m] = 0.f;

    auto fixup = [&](int tp, float c1) {
      if (TCD_TRACE_ON && (p.dbg & 16)) return;  // timing experiment: no fixups (results invalid)
      const int a = tp % NACC;
      mbar_wait(&full_acc[a], (uint32_t)(tp / NACC) & 1);
      tc_fence_after();
      const uint32_t ta = Cfg::kRot ? tmem + lane_off + kTcdAccCol + ((tp >> 4) & 1) * kTcdNB + (tp & 15)
                                    : tmem + lane_off + kTcdAccCol + a * kTcdNB;
      if constexpr (MT == 1) {
        const uint32_t d = tcd_ldtm_x1(ta);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        tot[0] = fmaf(c1, __uint_as_float(d), tot[0]);
      } else {
        uint32_t d[16];
        tmem_ld_32x32b_x16(ta, d);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
#pragma unroll
        for (int m = 0; m < MT; ++m) tot[m] = fmaf(c1, __uint_as_float(d[m]), tot[m]);
      }
    };

    int t = g;
    int qst = g / kR;  // stage of tile t, its ring slot and phase (tracked incrementally)
    int s = qst % NS;
    uint32_t ph = (uint32_t)(qst / NS) & 1;
    uint32_t kk = 0;   // this group's tile counter
    // the fixup of a tile is applied two group-iterations late, so the in-order MMA issuer has
    // reached it by then: tp2 (older) and tp1 are pending, with their scale * c1mul
    int tp1 = -1, tp2 = -1;
    float c1p1 = 0.f, c1p2 = 0.f;
    int t0 = 0;
    while (t0 < T) {
      const int ufirst = u0 + t0;
      const int nt = ufirst / KT;
      const int t1 = min(T, t0 + (KT - (ufirst - nt * KT)));
      for (; t < t1; t += NG, ++kk) {
        tcd_istamp(p, dw, lane, kk, 0);
        mbar_wait(&full_tma[s], ph);
        if (TCD_TRACE_ON && (p.dbg & 64)) {  // timing experiment: stream only (results invalid)
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_tma[s]);
          const int qn = (t + NG) / kR;
          s += qn - qst;
          qst = qn;
          while (s >= NS) {
            s -= NS;
            ph ^= 1;
          }
          continue;
        }
        tcd_istamp(p, dw, lane, kk, 1);
        if (kk == 0 && dw == 0 && lane == 0) tcd_stamp(p, 4);
        const int jt = t - qst * kR;  // tile within the stage
        const uint32_t st = st_u + s * SB;
        uint32_t words[4 * F::bits];
        tcd_load_words<F::bits>(st + jt * WB, n, words);
        const float sc = Act<BF>::to_float(lds16(st + kR * WB + 256 * jt + 2 * n));
        // ints: -z as fp16x2 (zero point of the tile's group; offset-binary ints: 2^(b-1))
        uint32_t zneg = 0;
        if constexpr (kInt) {
          if constexpr (F::kind == kUint) {
            if (has_zeros) {
              const uint32_t zb = Act<BF>::neg_zero_h(lds16(st + kR * WB + kR * 256 + 256 * jt + 2 * n));
              zneg = zb | (zb << 16);
            }
          } else {
            constexpr uint32_t zb = 0x8000u | ((uint32_t)(F::bits - 1 + 15) << 10);  // -2^(b-1)
            zneg = zb | (zb << 16);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_tma[s]);
        tcd_istamp(p, dw, lane, kk, 2);
        const uint32_t tslot = tmem + lane_off + wsl * 64;
        // per-P constants -(2^(10-P) + z) (exact: integers below 2048)
        uint32_t cp[10];
        static_for<0, 10>([&](auto PP) {
          constexpr int P = decltype(PP)::value;
          if constexpr (kInt && plan_uses_p<F>(P)) {
            constexpr uint32_t k = 0x8000u | ((uint32_t)(25 - P) << 10);  // fp16 -2^(10-P)
            cp[P] = h2_as_u32(__hadd2(u32_as_h2(zneg), u32_as_h2(k | (k << 16))));
          }
        });
        // chunk c = pairs 16c .. 16c+15 = the TMEM columns of MMAs 2c, 2c+1
        auto unpack = [&](auto CC, uint32_t (&r)[16]) {
          constexpr int c = decltype(CC)::value;
          constexpr int h = c >> 1;  // block
          uint32_t bw[2 * F::bits];
#pragma unroll
          for (int j = 0; j < 2 * F::bits; ++j) bw[j] = words[tile_word(h, j)];
          static_for<0, 16>([&](auto II) {
            constexpr int i = (c & 1) * 16 + decltype(II)::value;  // pair within the block
            if constexpr (kInt) {
              constexpr int P = kPlan<F::kind, F::bits, F::exp>.pr[i].P;
              const uint32_t x = extract_pair<F, i>(bw, p.magic);
              r[decltype(II)::value] = Act<BF>::from_h2(
                  h2_as_u32(__hfma2(u32_as_h2(x), u32_as_h2(h2_pow2_neg<P>()), u32_as_h2(cp[P]))));
            } else {
              r[decltype(II)::value] = Act<BF>::from_h2(extract_pair<F, i>(bw, 0u));
            }
          });
        };
        // the first half of the unpack runs BEFORE the W^T-slot wait (into registers: the asm
        // register fences keep the compiler from sinking it below the wait), so a group's
        // long ALU phase never waits for the in-order MMA of tile t - NW
        uint32_t r0[16], r1[16];
        unpack(std::integral_constant<int, 0>{}, r0);
        unpack(std::integral_constant<int, 1>{}, r1);
#pragma unroll
        for (int i = 0; i < 16; ++i) asm volatile("" : "+r"(r0[i]), "+r"(r1[i]));
        if (t >= kTcdNW) mbar_wait(&full_acc[(t - kTcdNW) % NACC], (uint32_t)((t - kTcdNW) / NACC) & 1);
        tcd_istamp(p, dw, lane, kk, 3);
        if (!(TCD_TRACE_ON && (p.dbg & 4))) {
          tcd_sttm_x16(tslot, r0);
          tcd_sttm_x16(tslot + 16, r1);
          static_for<2, 4>([&](auto CC) {
            uint32_t r[16];
            unpack(CC, r);
            tcd_sttm_x16(tslot + decltype(CC)::value * 16, r);
          });
        }
        tcd_istamp(p, dw, lane, kk, 4);
        tmem_st_wait();
        tcd_istamp(p, dw, lane, kk, 5);
        mbar_wait(&full_op[t % kTcdNOP], (uint32_t)(t / kTcdNOP) & 1);  // the tile's activation operand landed
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_w[wsl]);
        wsl += NG;
        while (wsl >= kTcdNW) {
          wsl -= kTcdNW;
          ++lapw;
        }
        if constexpr (Cfg::Lag == 2) {
          if (tp2 >= 0) fixup(tp2, c1p2);
          tp2 = tp1;
          c1p2 = c1p1;
        } else {
          if (tp1 >= 0) fixup(tp1, c1p1);
        }
        tcd_istamp(p, dw, lane, kk, 6);
        tp1 = t;
        c1p1 = sc * c1mul;
        {
          const int qn = (t + NG) / kR;
          s += qn - qst;
          qst = qn;
          while (s >= NS) {
            s -= NS;
            ph ^= 1;
          }
        }
      }
      if (dw == 0 && lane == 0) tcd_stamp(p, 5);
      if (tp2 >= 0) fixup(tp2, c1p2);
      if (tp1 >= 0) fixup(tp1, c1p1);
      tp1 = tp2 = -1;
      if (dw == 0 && lane == 0) tcd_stamp(p, 6);
      // ---- n-tile nt done by this CTA: sum the groups' totals, write Y or a stream-K partial ----
#pragma unroll
      for (int m = 0; m < MT; ++m)
        if (m < p.M) red[(g * p.M + m) * kBN + n] = tot[m];
      named_bar_sync(1, NG * 128);
      const int ua = nt * KT, ub = ua + KT;
      const bool complete = (u0 <= ua) && (u1 >= ub);
      const int col = nt * kBN + n;
      const int slot2 = (nt == u0 / KT) ? 0 : 1;
      float* part = p.partial + ((int64_t)(cta * 2 + slot2) * kTcdNB) * kBN;
      for (int m = g; m < p.M; m += NG) {
        float v = 0.f;
#pragma unroll
        for (int gg = 0; gg < NG; ++gg) v += red[(gg * p.M + m) * kBN + n];
        if (complete) {
          const unsigned short h = Act<BF>::from_float(v);
          reinterpret_cast<unsigned short*>(p.Y)[(int64_t)m * p.ldy + col] = h;
          peer_store(p.po, (int64_t)m * p.ldy + col, h);
        } else {
          __stcg(part + (int64_t)m * kBN + n, v);
        }
      }
      if (!complete) {
        // publish: the CTA barrier orders every thread's partial store before thread 128's
        // gpu-scope acq_rel increment (release for ours, acquire of the other CTAs' partials when
        // we are the last to arrive); no per-thread fences
        named_bar_sync(1, NG * 128);
        if (threadIdx.x == 128) {
          const int lo = (int)((((int64_t)ua + 1) * grid - 1) / p.units);
          const int hi = (int)((((int64_t)ub) * grid - 1) / p.units);
          int prev;
          asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(&p.sem[nt]) : "memory");
          flag[0] = (prev == hi - lo) ? 1 : 0;
          flag[1] = lo;
          flag[2] = hi;
          flag[3] = ((int)((int64_t)lo * p.units / grid) / KT == nt) ? 0 : 1;
        }
        named_bar_sync(1, NG * 128);
        if (flag[0]) {
          const int lo = flag[1], hi = flag[2];
          for (int m = g; m < p.M; m += NG) {
            const float sum = streamk_sum(p.partial, lo, hi, flag[3], (int64_t)kTcdNB * kBN, (int64_t)m * kBN + n);
            const unsigned short h = Act<BF>::from_float(sum);
            reinterpret_cast<unsigned short*>(p.Y)[(int64_t)m * p.ldy + col] = h;
            peer_store(p.po, (int64_t)m * p.ldy + col, h);
          }
          if (threadIdx.x == 128) p.sem[nt] = 0;
        }
      }
      named_bar_sync(1, NG * 128);
      if (dw == 0 && lane == 0) tcd_stamp(p, 9);
#pragma unroll
      for (int m = 0; m < MT; ++m) tot[m] = 0.f;
      t0 = t1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) peer_signal(p.po, gridDim.x);  // row f3: after every Y store of the CTA
  if (threadIdx.x == 0) tcd_stamp(p, 7);
}

template <class F, int MT, bool BF>
tl_status launch_tcd_mt(const TcdParams& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st) {
  if (prepare_kernel(reinterpret_cast<const void*>(tcd_kernel<F, MT, BF>), 227 * 1024, TcdCfg<MT>::Threads) == 0)
    return fail(TL_ECUDA, "tcd_kernel: %s", tl_last_error());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TcdCfg<MT>::Threads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (p.dbg & 128) ? 0 : 1;  // TL_TCD_DBG=128: plain stream order (A/B of the PDL overlap)
  cudaError_t e = cudaLaunchKernelEx(&cfg, tcd_kernel<F, MT, BF>, *tmap, p);
  if (e != cudaSuccess) return fail(TL_ECUDA, "tcd_kernel launch: %s", cudaGetErrorString(e));
  return check_launch("tcd_kernel");
}

template <class F>
tl_status launch_tcd(const TcdParams& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st) {
  if (p.bf) return p.rot ? launch_tcd_mt<F, 1, true>(p, tmap, grid, smem_bytes, st)
                       : launch_tcd_mt<F, kTcdNB, true>(p, tmap, grid, smem_bytes, st);
  return p.rot ? launch_tcd_mt<F, 1, false>(p, tmap, grid, smem_bytes, st)
               : launch_tcd_mt<F, kTcdNB, false>(p, tmap, grid, smem_bytes, st);
}

}  // namespace tl
