// tc2.cuh -- batched tensor-core path (any M, any group): SURVEY §8(a) rows a3-a11, K-B3.
//
// Paper: "Tensor Cores for 16 or more tokens" with software pipelining and stream-K
// (PAPER.md:546); the weight pipeline of fig:weight-pipeline(c).  B200 form:
//
//   D[n 128, m NB] (fp32, TMEM) += W^T[n 128, k 16] (fp16, TMEM) x A^T[k 16, m NB] (fp16, smem)
//
// (swap-AB: the weight tile fills the 128 MMA rows, the batch is MMA-N, NB <= 128 per launch).
//   warp 0      TMA producer: per k-tile one cp.async.bulk of the packed 128x128 weight tile
//               and two 2-D tensor boxes of the activations (128B swizzle, rows >= M
//               zero-filled) -> NS-stage ring.
//   warp 1      TMEM owner + MMA issuer (one thread): 8 x tcgen05.mma.cta_group::1.kind::f16 per
//               k-tile with the A operand (the dequantized W^T) read from TENSOR MEMORY ("TS"),
//               accumulating the whole K range of an n-tile in one TMEM accumulator.
//   warps 2..13 three dequant groups of 4 warps (warp%4 = TMEM lane quarter); group g handles
//               tiles t = g, g+3, ... into its two TMEM W^T slots (double buffer): LDS of the
//               column's words, LOP3 (layout v2, common.cuh) + HFMA2 (magic number) -> exact
//               (u - z) / value(code) fp16 pairs, HMUL2 by the group scale (reading R9),
//               tcgen05.st.  The same
//               warps run the epilogue (tcgen05.ld -> fp16 -> Y, or a stream-K partial with a
//               deterministic fixup) at the end of every 128-column n-tile.
// Scales / zeros are read by the dequant threads straight from global memory, PF tiles ahead.
#pragma once

#include <cuda.h>

#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

struct Tc2Params {
  int M, N, K, G;
  int NB;          // MMA N = batch tile (multiple of 16, <= 128)
  int units;
  int ns;          // TMA ring stages
  uint32_t stage_bytes, a_off_in_stage;
  const uint8_t* wt;
  const __half* scales;
  const __half* zeros;
  __half* Y;
  int64_t ldy;
  float* partial;  // [grid][2][NB][128]
  int* sem;
  uint32_t magic;  // 0x64006400
};

constexpr int kTc2Groups = 3;
constexpr int kTc2Threads = 64 + kTc2Groups * 128;
constexpr int kTc2WSlots = 2 * kTc2Groups;          // W^T tiles in TMEM (64 columns each)
constexpr uint32_t kTc2AccCol = 64 * kTc2WSlots;    // accumulator columns [384, 384 + NB)

__device__ __forceinline__ void tc2_tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tc2_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ uint64_t tc2_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// is P the field position of some pair of the format's plan (ints)?
template <class F>
__host__ __device__ constexpr bool tc2_plan_uses_p(int P) {
  for (int i = 0; i < 32; ++i)
    if (kPlan<F::kind, F::bits, F::exp>.pr[i].P == P) return true;
  return false;
}

// Dequantize row n of one tile (64 pairs, layout v2) into a TMEM W^T slot; scales / zeros of the
// tile's (up to four) 32-k sub-pieces come in sc[4] / zc[4] (fp16 bits).
//   ints:   LOP3(s) -> 1024 + u*2^P (magic form); HFMA2(x, 2^-P, -(2^(10-P) + z)) = u - z exactly;
//           HMUL2 by s (one fp16 rounding, reading R9)
//   floats: LOP3(s) -> value(code) * 2^(bias-15) exactly; HMUL2 by 2^(15-bias) (exact), HMUL2 by s
template <class F>
__device__ __forceinline__ void tc2_dequant_tile(uint32_t wtile, int n, uint32_t tslot, uint32_t magic,
                                                 const uint16_t (&sc)[4], const uint16_t (&zc)[4]) {
  constexpr int B = F::bits;
  uint32_t words[4 * B];
#pragma unroll
  for (int v = 0; v < B; ++v) {
    const uint4 x = lds128(wtile + (v * 128 + n) * 16);
    words[4 * v + 0] = x.x;
    words[4 * v + 1] = x.y;
    words[4 * v + 2] = x.z;
    words[4 * v + 3] = x.w;
  }
  static_for<0, 4>([&](auto CC) {
    constexpr int c = decltype(CC)::value;  // 16 pairs = one 32-k sub-piece = 16 TMEM columns
    constexpr int h = c >> 1;
    uint32_t bw[2 * B];
#pragma unroll
    for (int j = 0; j < 2 * B; ++j) bw[j] = words[tile_word(h, j)];
    const __half2 s2 = u32_as_h2((uint32_t)sc[c] | ((uint32_t)sc[c] << 16));
    uint32_t cp[10];
    if constexpr (F::kind != kFloat) {
      uint32_t zneg;
      if constexpr (F::kind == kUint) {
        const uint32_t zb = (uint32_t)zc[c] ^ 0x8000u;
        zneg = zb | (zb << 16);
      } else {
        constexpr uint32_t zb = 0x8000u | ((uint32_t)(B - 1 + 15) << 10);  // -2^(b-1)
        zneg = zb | (zb << 16);
      }
      static_for<0, 10>([&](auto PP) {
        constexpr int P = decltype(PP)::value;
        if constexpr (tc2_plan_uses_p<F>(P)) {
          constexpr uint32_t k = 0x8000u | ((uint32_t)(25 - P) << 10);  // fp16 -2^(10-P)
          cp[P] = h2_as_u32(__hadd2(u32_as_h2(zneg), u32_as_h2(k | (k << 16))));
        }
      });
    }
    uint32_t r[16];
    static_for<0, 16>([&](auto II) {
      constexpr int ii = decltype(II)::value;
      constexpr int i = (c & 1) * 16 + ii;  // pair within the block
      if constexpr (F::kind != kFloat) {
        constexpr int P = kPlan<F::kind, F::bits, F::exp>.pr[i].P;
        const uint32_t x = extract_pair<F, i>(bw, magic);
        const __half2 v = __hfma2(u32_as_h2(x), u32_as_h2(h2_pow2_neg<P>()), u32_as_h2(cp[P]));
        r[ii] = h2_as_u32(__hmul2(v, s2));
      } else {
        constexpr uint32_t e = (uint32_t)(30 - F::bias) << 10;  // fp16 bits of 2^(15-bias)
        const uint32_t x = extract_pair<F, i>(bw, 0u);
        r[ii] = h2_as_u32(__hmul2(__hmul2(u32_as_h2(x), u32_as_h2(e | (e << 16))), s2));
      }
    });
    tc2_tmem_st16(tslot + c * 16, r);
  });
}

template <class F>
__global__ void __launch_bounds__(kTc2Threads, 1) tc2_kernel(const __grid_constant__ CUtensorMap tmapA, Tc2Params p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr uint32_t WB = tile_bytes(F::bits);
  const int NS = p.ns;
  const int NB = p.NB;
  const uint32_t stage_bytes = p.stage_bytes;
  uint8_t* st = smem;  // NS x [activation boxes (1024-aligned) | packed weight tile]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * stage_bytes);
  uint64_t* full_tma = bars;
  uint64_t* empty_tma = bars + NS;
  uint64_t* full_w = bars + 2 * NS;             // [6]
  uint64_t* empty_w = full_w + kTc2WSlots;      // [6]
  uint64_t* acc_full = empty_w + kTc2WSlots;    // [1]
  uint64_t* acc_empty = acc_full + 1;           // [1]
  uint32_t* tslot_ptr = reinterpret_cast<uint32_t*>(acc_empty + 1);
  int* flag = reinterpret_cast<int*>(tslot_ptr + 4);

  const int KT = p.K / kBK;
  const int grid = gridDim.x;
  const int cta = blockIdx.x;
  const int u0 = (int)((int64_t)cta * p.units / grid);
  const int u1 = (int)((int64_t)(cta + 1) * p.units / grid);
  const int T = u1 - u0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool has_zeros = p.zeros != nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_tma[s], 1);
      mbar_init(&empty_tma[s], 4 + 1);  // the dequant group (4 warps) + the MMA commit
    }
    for (int i = 0; i < kTc2WSlots; ++i) {
      mbar_init(&full_w[i], 4);
      mbar_init(&empty_w[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, kTc2Groups * 4);
    fence_mbar_init();
    prefetch_tmap(&tmapA);
  }
  if (warp == 1) {
    tmem_alloc(tslot_ptr, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot_ptr;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_a = policy_evict_last();
      const uint32_t bytes = WB + (uint32_t)NB * 256;
      int s = 0, ph = 0, kt = u0 % KT;
      for (int t = 0; t < T; ++t) {
        if (t >= NS) mbar_wait_sleepy(&empty_tma[s], ph ^ 1);
        uint8_t* sp = st + s * stage_bytes;
        mbar_arrive_expect_tx(&full_tma[s], bytes);
        tma_load_2d(sp, &tmapA, kt * kBK, 0, &full_tma[s], pol_a);
        tma_load_2d(sp + NB * 128, &tmapA, kt * kBK + 64, 0, &full_tma[s], pol_a);
        tma_bulk_g2s(sp + p.a_off_in_stage, p.wt + (int64_t)(u0 + t) * WB, WB, &full_tma[s], pol_w);
        if (++kt == KT) kt = 0;
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (one thread) ------------------------------
    if (elect_one()) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t bblk = (uint32_t)NB * 8;  // NB*128 B in 16-B descriptor units
      int s = 0, ph = 0, kt = u0 % KT, seg = 0;
      bool first = true;
      for (int t = 0; t < T; ++t) {
        const int gk = t / kTc2Groups, gg = t - gk * kTc2Groups;
        const int ws = 2 * gg + (gk & 1);
        if (first && seg >= 1) mbar_wait(acc_empty, (seg - 1) & 1);  // epilogue drained the accumulator
        mbar_wait(&full_w[ws], (gk >> 1) & 1);
        mbar_wait(&full_tma[s], ph);
        tc_fence_after();
        const uint64_t bd0 = tc2_sw128_desc(smem_u32(st + s * stage_bytes));
        const uint32_t aw = tmem + ws * 64;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          tc2_mma_ts(tmem + kTc2AccCol, aw + j * 8, bd0 + (uint64_t)((j >> 2) * bblk + (j & 3) * 2), idesc,
                     (first && j == 0) ? 0u : 1u);
        tc_commit(&empty_w[ws]);
        tc_commit(&empty_tma[s]);
        first = false;
        if (kt == KT - 1 || t == T - 1) {
          tc_commit(acc_full);
          first = true;
          ++seg;
        }
        if (++kt == KT) kt = 0;
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ------------------------------ dequant groups + epilogue ------------------------------
    const int dw = warp - 2;            // 0..11
    const int g = dw >> 2;              // dequant group
    const int q = warp & 3;             // TMEM lane quarter
    const int n = q * 32 + lane;        // row of W^T = output column within the n-tile
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t st_u = smem_u32(st);
    const unsigned short* sg = reinterpret_cast<const unsigned short*>(p.scales);
    const unsigned short* zg = reinterpret_cast<const unsigned short*>(p.zeros);
    // scale / zero prefetch (PF group-iterations ahead), group rows tracked from (nt, kt)
    constexpr int PF = 2;
    const int lgG = p.G == 32 ? 5 : (p.G == 64 ? 6 : 0);  // G < 128: row = k >> lgG
    const int tpg = p.G >= kBK ? p.G / kBK : 1;            // G >= 128: k-tiles per group
    auto fetch = [&](int tt, uint16_t (&sc)[4], uint16_t (&zc)[4]) {
      const int u = u0 + tt, nt_ = u / KT, kt_ = u - nt_ * KT;
      const int trow = lgG ? 0 : (tpg == 1 ? kt_ : kt_ / tpg);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int row = lgG ? ((kt_ * kBK + c * 32) >> lgG) : trow;
        const int64_t off = (int64_t)row * p.N + nt_ * kBN + n;
        sc[c] = __ldg(sg + off);
        zc[c] = (F::kind == kUint && has_zeros) ? __ldg(zg + off) : (unsigned short)0;
      }
    };
    uint16_t scq[PF][4], zcq[PF][4];
#pragma unroll
    for (int pf = 0; pf < PF; ++pf)
      if (g + pf * kTc2Groups < T) fetch(g + pf * kTc2Groups, scq[pf], zcq[pf]);

    int t = g, kk = 0, seg = 0;
    int t0 = 0;
    while (t0 < T) {
      const int ufirst = u0 + t0;
      const int nt = ufirst / KT;
      const int t1 = min(T, t0 + (KT - (ufirst - nt * KT)));
      for (; t < t1; t += kTc2Groups, ++kk) {
        const int ws = 2 * g + (kk & 1);
        uint16_t sc[4], zc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          sc[c] = scq[0][c];
          zc[c] = zcq[0][c];
        }
#pragma unroll
        for (int pf = 0; pf + 1 < PF; ++pf)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            scq[pf][c] = scq[pf + 1][c];
            zcq[pf][c] = zcq[pf + 1][c];
          }
        if (t + PF * kTc2Groups < T) fetch(t + PF * kTc2Groups, scq[PF - 1], zcq[PF - 1]);
        const int s = t % NS;
        mbar_wait(&full_tma[s], (t / NS) & 1);
        if (kk >= 2) mbar_wait(&empty_w[ws], ((kk >> 1) - 1) & 1);
        tc2_dequant_tile<F>(st_u + s * stage_bytes + p.a_off_in_stage, n, tmem + lane_off + ws * 64, p.magic, sc, zc);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&full_w[ws]);
          mbar_arrive(&empty_tma[s]);
        }
      }
      // ---- epilogue of n-tile nt: the accumulator holds this CTA's K range of it ----
      mbar_wait(acc_full, seg & 1);
      tc_fence_after();
      const int ua = nt * KT, ub = ua + KT;
      const bool complete = (u0 <= ua) && (u1 >= ub);
      const int col = nt * kBN + n;
      const int slot2 = (nt == u0 / KT) ? 0 : 1;
      float* part = p.partial + ((int64_t)(cta * 2 + slot2) * NB) * kBN;
      for (int cb = g * 16; cb < NB; cb += kTc2Groups * 16) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tmem + lane_off + kTc2AccCol + cb, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = cb + j;
          if (m < p.M) {
            const float v = __uint_as_float(r[j]);
            if (complete) p.Y[(int64_t)m * p.ldy + col] = __float2half_rn(v);
            else __stcg(part + (int64_t)m * kBN + n, v);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      if (!complete) {
        __threadfence();
        named_bar_sync(1, kTc2Groups * 128);
        if (threadIdx.x == 64) {
          const int lo = (int)((((int64_t)ua + 1) * grid - 1) / p.units);
          const int hi = (int)((((int64_t)ub) * grid - 1) / p.units);
          const int prev = atomicAdd(&p.sem[nt], 1);
          flag[0] = (prev == hi - lo) ? 1 : 0;
          flag[1] = lo;
          flag[2] = hi;
          flag[3] = ((int)((int64_t)lo * p.units / grid) / KT == nt) ? 0 : 1;
        }
        named_bar_sync(1, kTc2Groups * 128);
        if (flag[0]) {
          __threadfence();
          const int lo = flag[1], hi = flag[2];
          for (int m = g; m < p.M; m += kTc2Groups) {
            const float sum = streamk_sum(p.partial, lo, hi, flag[3], (int64_t)NB * kBN, (int64_t)m * kBN + n);
            p.Y[(int64_t)m * p.ldy + col] = __float2half_rn(sum);
          }
          if (threadIdx.x == 64) p.sem[nt] = 0;
        }
        named_bar_sync(1, kTc2Groups * 128);
      }
      ++seg;
      t0 = t1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <class F>
tl_status launch_tc2(const Tc2Params& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st) {
  if (prepare_kernel(reinterpret_cast<const void*>(tc2_kernel<F>), 227 * 1024, kTc2Threads) == 0)
    return fail(TL_ECUDA, "tc2_kernel: %s", tl_last_error());
  tc2_kernel<F><<<grid, kTc2Threads, smem_bytes, st>>>(*tmap, p);
  return check_launch("tc2_kernel");
}

}  // namespace tl
