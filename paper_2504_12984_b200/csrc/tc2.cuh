// tc2.cuh -- batched tensor-core path (M > 16, any group): SURVEY §8(a) rows a3-a11, K-B3.
//
// Paper: "Tensor Cores for 16 or more tokens" with software pipelining and stream-K
// (PAPER.md:546); the weight pipeline of fig:weight-pipeline(c).  B200 form:
//
//   D_j[n 128, m NB] (fp32, TMEM) += W_j^T[n 128, k 16] (fp16, TMEM) x A^T[k 16, m NB] (fp16, smem)
//
// swap-AB: the weight tile fills the 128 MMA rows, the batch is MMA-N (NB <= 128 per launch).
// A UNIT is one k-tile of an n-PAIR: the activation tile A[:, kt*128 : +128] (NB x 256 B) is
// staged once and feeds the MMAs of two 128-column weight tiles (n-tiles 2p and 2p+1), halving
// the L2 -> SM activation traffic (at NB = 128 and full tensor rate, one activation tile per
// weight tile would need more L2 bandwidth than the chip has).
//   warp 0      TMA producer: per unit two 64-k x NB-row boxes of A (128B swizzle, rows >= M
//               zero-filled) + one cp.async.bulk per weight tile (2048*b B) -> NS-stage ring.
//   warp 1      TMEM owner + MMA issuer (one thread): 16 x tcgen05.mma.cta_group::1.kind::f16 per
//               unit, the A operand (the dequantized W^T) read from TENSOR MEMORY ("TS"), the two
//               accumulators D_0, D_1 hold the CTA's K range of the n-pair.
//   warps 2..9  two dequant groups of 4 warps (warp%4 = TMEM lane quarter); group g handles the
//               units t = g, g+2, ... into its W^T slot pair: LDS of the column's words,
//               LOP3 (layout v2, common.cuh) + HFMA2 (magic number) -> exact (u - z) /
//               value(code) fp16 pairs, HMUL2 by the group scale (reading R9), tcgen05.st.
//               At the end of an n-pair both groups run the epilogue (group j: accumulator D_j).
// TMEM columns: [0,128) W^T slots of group 0 (tile 0 | tile 1), [128,256) group 1,
// [256,384) D_0, [384,512) D_1.
#pragma once

#include <cuda.h>

#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

struct Tc2Params {
  int M, N, K, G;
  int NB;          // MMA N = batch tile (multiple of 16, <= 128)
  int NT;          // n-tiles (N / 128)
  int units;       // n-pairs * KT
  int ns;          // TMA ring stages
  uint32_t stage_bytes, w_off_in_stage;  // [A boxes NB*256 | W tile 0 | W tile 1]
  const uint8_t* wt;
  const __half* scales;
  const __half* zeros;
  __half* Y;
  int64_t ldy;
  float* partial;  // [grid][2 slots][2 tiles][NB][128]
  int* sem;        // [n-pairs]
  uint32_t magic;  // 0x64006400 (a kernel argument: the LOP3 takes one immediate, see tcd)
  int bf;          // 1: bf16 activations / scales / zeros / Y
  int dist;        // 1: distributed stream-K reduction (every contributor reduces 1/S of the tile; needs
                   //    all CTAs resident: grid <= SMs)
  PeerOut po;      // row f3: gathered output fused into the epilogue (peer.cuh); po.n == 0: local only
  int dbg;         // TL_TC2_DBG timing experiments (results invalid): 1 skip partial stores, 2 skip reduction
};

constexpr int kTc2Groups = 2;
constexpr int kTc2Threads = 64 + kTc2Groups * 128;
constexpr uint32_t kTc2AccCol = 256;  // D_0 at 256, D_1 at 384

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

// Dequantize column n of one weight tile (64 pairs, layout v2) into the 64 TMEM columns at
// tslot.  sc[c] / zc[c]: fp16 bits of the scale / zero of 32-k sub-piece c (all four equal when
// the group size is a multiple of 128).
//   ints:   LOP3(s) -> 1024 + u*2^P (magic form); HFMA2(x, 2^-P, -(2^(10-P) + z)) = u - z exactly;
//           HMUL2 by s (one fp16 rounding, reading R9)
//   floats: LOP3(s) -> value(code) * 2^(bias-15) exactly; HMUL2 by 2^(15-bias) (exact), HMUL2 by s
template <class F, bool kSubG, bool BF>
__device__ __forceinline__ void tc2_dequant_tile(uint32_t wtile, int n, uint32_t tslot, uint32_t magic,
                                                 const uint32_t (&sc)[4], const uint32_t (&zc)[4]) {
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
  uint32_t cp[kSubG ? 4 : 1][10];
  static_for<0, (kSubG ? 4 : 1)>([&](auto CC) {
    constexpr int c = decltype(CC)::value;
    if constexpr (F::kind != kFloat) {
      uint32_t zneg;
      if constexpr (F::kind == kUint) {
        const uint32_t zb = Act<BF>::neg_zero_h(zc[c]);
        zneg = zb | (zb << 16);
      } else {
        constexpr uint32_t zb = 0x8000u | ((uint32_t)(B - 1 + 15) << 10);  // -2^(b-1)
        zneg = zb | (zb << 16);
      }
      static_for<0, 10>([&](auto PP) {
        constexpr int P = decltype(PP)::value;
        if constexpr (tc2_plan_uses_p<F>(P)) {
          constexpr uint32_t k = 0x8000u | ((uint32_t)(25 - P) << 10);  // fp16 -2^(10-P)
          cp[c][P] = h2_as_u32(__hadd2(u32_as_h2(zneg), u32_as_h2(k | (k << 16))));
        }
      });
    }
  });
  static_for<0, 4>([&](auto CC) {
    constexpr int c = decltype(CC)::value;  // 16 pairs = one 32-k sub-piece = 16 TMEM columns
    constexpr int cs = kSubG ? c : 0;
    constexpr int h = c >> 1;
    uint32_t bw[2 * B];
#pragma unroll
    for (int j = 0; j < 2 * B; ++j) bw[j] = words[tile_word(h, j)];
    const __half2 s2 = u32_as_h2(sc[cs] | (sc[cs] << 16));  // fp16 activations
    const float sf = Act<BF>::to_float(sc[cs]);              // bf16 activations
    uint32_t r[16];
    static_for<0, 16>([&](auto II) {
      constexpr int ii = decltype(II)::value;
      constexpr int i = (c & 1) * 16 + ii;  // pair within the block
      __half2 v;                             // exact: u - z, or value(code) (floats)
      if constexpr (F::kind != kFloat) {
        constexpr int P = kPlan<F::kind, F::bits, F::exp>.pr[i].P;
        const uint32_t x = extract_pair<F, i>(bw, magic);
        v = __hfma2(u32_as_h2(x), u32_as_h2(h2_pow2_neg<P>()), u32_as_h2(cp[cs][P]));
      } else {
        constexpr uint32_t e = (uint32_t)(30 - F::bias) << 10;  // fp16 bits of 2^(15-bias)
        const uint32_t x = extract_pair<F, i>(bw, 0u);
        v = __hmul2(u32_as_h2(x), u32_as_h2(e | (e << 16)));
      }
      if constexpr (!BF) {
        r[ii] = h2_as_u32(__hmul2(v, s2));  // one fp16 rounding (reading R9)
      } else {
        const float2 f = __half22float2(v);   // exact; then one bf16 rounding of value * s
        const __nv_bfloat162 b = __floats2bfloat162_rn(f.x * sf, f.y * sf);
        r[ii] = *reinterpret_cast<const uint32_t*>(&b);
      }
    });
    tc2_tmem_st16(tslot + c * 16, r);
  });
}

template <class F, bool kSubG, bool BF>
__global__ void __launch_bounds__(kTc2Threads, 1) tc2_kernel(const __grid_constant__ CUtensorMap tmapA, Tc2Params p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr uint32_t WB = tile_bytes(F::bits);
  const int NS = p.ns;
  const int NB = p.NB;
  const uint32_t SB = p.stage_bytes;
  uint8_t* st = smem;  // NS x [activation boxes (1024-aligned) | weight tile 0 | weight tile 1]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * SB);
  uint64_t* full_tma = bars;
  uint64_t* empty_tma = bars + NS;                // the group (4 warps) + the MMA commit
  uint64_t* full_w = bars + 2 * NS;               // [2] group g's W^T slot pair written
  uint64_t* empty_w = full_w + kTc2Groups;        // [2] MMA done with it
  uint64_t* acc_full = empty_w + kTc2Groups;      // [1] the n-pair's last MMA completed
  uint64_t* acc_empty = acc_full + 1;             // [1] the epilogue drained both accumulators
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
      mbar_init(&empty_tma[s], 4 + 1);
    }
    for (int i = 0; i < kTc2Groups; ++i) {
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
      const uint32_t abytes = (uint32_t)NB * 256;
      int s = 0, ph = 0;
      int np = u0 / KT, kt = u0 - (u0 / KT) * KT;
      for (int t = 0; t < T; ++t) {
        const bool two = 2 * np + 1 < p.NT;
        if (t >= NS) mbar_wait_sleepy(&empty_tma[s], ph ^ 1);
        uint8_t* sp = st + s * SB;
        mbar_arrive_expect_tx(&full_tma[s], abytes + (two ? 2 : 1) * WB);
        tma_load_2d(sp, &tmapA, kt * kBK, 0, &full_tma[s], pol_a);
        tma_load_2d(sp + NB * 128, &tmapA, kt * kBK + 64, 0, &full_tma[s], pol_a);
        const uint8_t* w0 = p.wt + ((int64_t)(2 * np) * KT + kt) * WB;
        tma_bulk_g2s(sp + p.w_off_in_stage, w0, WB, &full_tma[s], pol_w);
        if (two) tma_bulk_g2s(sp + p.w_off_in_stage + WB, w0 + (int64_t)KT * WB, WB, &full_tma[s], pol_w);
        if (++kt == KT) {
          kt = 0;
          ++np;
        }
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (one thread) ------------------------------
    if (elect_one()) {
      const uint32_t idesc =
          (1u << 4) | Act<BF>::idesc_ab | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t bblk = (uint32_t)NB * 8;  // NB*128 B in 16-B descriptor units
      int s = 0, ph = 0, np = u0 / KT, kt = u0 - (u0 / KT) * KT, seg = 0;
      bool first = true;
      for (int t = 0; t < T; ++t) {
        const int g = t & 1;
        const bool two = 2 * np + 1 < p.NT;
        if (first && seg >= 1) mbar_wait(acc_empty, (seg - 1) & 1);  // epilogue drained the accumulators
        mbar_wait(&full_w[g], (t >> 1) & 1);
        tc_fence_after();
        const uint64_t bd0 = tc2_sw128_desc(smem_u32(st + s * SB));
        const uint32_t aw = tmem + g * 128;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j == 0 || two) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              tc2_mma_ts(tmem + kTc2AccCol + j * 128, aw + j * 64 + ks * 8,
                         bd0 + (uint64_t)((ks >> 2) * bblk + (ks & 3) * 2), idesc, (first && ks == 0) ? 0u : 1u);
          }
        }
        tc_commit(&empty_w[g]);
        tc_commit(&empty_tma[s]);
        first = false;
        if (kt == KT - 1 || t == T - 1) {
          tc_commit(acc_full);
          first = true;
          ++seg;
        }
        if (++kt == KT) {
          kt = 0;
          ++np;
        }
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ------------------------------ dequant groups + epilogue ------------------------------
    const int dw = warp - 2;            // 0..7
    const int g = dw >> 2;              // dequant group
    const int q = warp & 3;             // TMEM lane quarter
    const int n = q * 32 + lane;        // row of W^T = output column within the n-tile
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t st_u = smem_u32(st);
    const unsigned short* sg = reinterpret_cast<const unsigned short*>(p.scales);
    const unsigned short* zg = reinterpret_cast<const unsigned short*>(p.zeros);
    // scale / zero of this thread's column for both tiles of unit t, PF group-iterations ahead
    constexpr int PF = 2;
    constexpr int NSC = kSubG ? 4 : 1;
    const int lgG = p.G == 32 ? 5 : (p.G == 64 ? 6 : 0);  // G < 128: row = k >> lgG
    const int tpg = p.G >= kBK ? p.G / kBK : 1;            // G >= 128: k-tiles per group
    auto fetch = [&](int tt, uint32_t (&sc)[2][4], uint32_t (&zc)[2][4]) {
      const int u = u0 + tt, np_ = u / KT, kt_ = u - np_ * KT;
      const int trow = kSubG ? 0 : (tpg == 1 ? kt_ : kt_ / tpg);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = (2 * np_ + j) * kBN + n;
        const bool ok = (2 * np_ + j) < p.NT;
#pragma unroll
        for (int c = 0; c < NSC; ++c) {
          const int row = kSubG ? ((kt_ * kBK + c * 32) >> lgG) : trow;
          const int64_t off = (int64_t)row * p.N + col;
          sc[j][c] = ok ? (uint32_t)__ldg(sg + off) : 0u;
          zc[j][c] = (ok && F::kind == kUint && has_zeros) ? (uint32_t)__ldg(zg + off) : 0u;
        }
      }
    };
    uint32_t scq[PF][2][4], zcq[PF][2][4];
#pragma unroll
    for (int pf = 0; pf < PF; ++pf)
      if (g + pf * kTc2Groups < T) fetch(g + pf * kTc2Groups, scq[pf], zcq[pf]);

    int t = g, kk = 0, seg = 0;
    int t0 = 0;
    while (t0 < T) {
      const int ufirst = u0 + t0;
      const int np = ufirst / KT;
      const int t1 = min(T, t0 + (KT - (ufirst - np * KT)));
      const bool two = 2 * np + 1 < p.NT;
      for (; t < t1; t += kTc2Groups, ++kk) {
        uint32_t sc[2][4], zc[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            sc[j][c] = scq[0][j][c];
            zc[j][c] = zcq[0][j][c];
          }
#pragma unroll
        for (int pf = 0; pf + 1 < PF; ++pf)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              scq[pf][j][c] = scq[pf + 1][j][c];
              zcq[pf][j][c] = zcq[pf + 1][j][c];
            }
        if (t + PF * kTc2Groups < T) fetch(t + PF * kTc2Groups, scq[PF - 1], zcq[PF - 1]);
        const int s = t % NS;
        mbar_wait(&full_tma[s], (t / NS) & 1);
        if (kk >= 1) mbar_wait(&empty_w[g], (kk - 1) & 1);  // MMA of this group's previous unit done
        const uint32_t wst = st_u + s * SB + p.w_off_in_stage;
        tc2_dequant_tile<F, kSubG, BF>(wst, n, tmem + lane_off + g * 128, p.magic, sc[0], zc[0]);
        if (two) tc2_dequant_tile<F, kSubG, BF>(wst + WB, n, tmem + lane_off + g * 128 + 64, p.magic, sc[1], zc[1]);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&full_w[g]);
          mbar_arrive(&empty_tma[s]);
        }
      }
      // ---- epilogue of n-pair np: group j owns accumulator D_j (n-tile 2np + j) ----
      mbar_wait(acc_full, seg & 1);
      tc_fence_after();
      const int nt = 2 * np + g;
      const int ua = np * KT, ub = ua + KT;
      const bool complete = (u0 <= ua) && (u1 >= ub);
      const int col = nt * kBN + n;
      const bool mine = g == 0 || two;
      const int slot2 = (np == u0 / KT) ? 0 : 1;
      float* part = p.partial + (((int64_t)(cta * 2 + slot2) * 2 + g) * NB) * kBN;
      if (mine) {
        for (int cb = 0; cb < NB; cb += 16) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem + lane_off + kTc2AccCol + g * 128 + cb, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int m = cb + j;
            if (m < p.M) {
              const float v = __uint_as_float(r[j]);
              if (complete) {
                const unsigned short h = Act<BF>::from_float(v);
                reinterpret_cast<unsigned short*>(p.Y)[(int64_t)m * p.ldy + col] = h;
                peer_store(p.po, (int64_t)m * p.ldy + col, h);
              } else if (!(p.dbg & 1)) {
                __stcg(part + (int64_t)m * kBN + n, v);
              }
            }
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
          if (p.dist) {
            // distributed: publish, then wait for every contributor's partial (all CTAs of the grid
            // are resident, so the wait cannot block a contributor from running)
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&p.sem[np]) : "memory");
            for (;;) {
              int v;
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(&p.sem[np]) : "memory");
              if (v >= hi - lo + 1) break;
              __nanosleep(32);
            }
            flag[0] = 1;
          } else {
            const int prev = atomicAdd(&p.sem[np], 1);
            flag[0] = (prev == hi - lo) ? 1 : 0;
          }
          flag[1] = lo;
          flag[2] = hi;
          flag[3] = ((int)((int64_t)lo * p.units / grid) / KT == np) ? 0 : 1;
        }
        named_bar_sync(1, kTc2Groups * 128);
        if (flag[0] && !(p.dbg & 2)) {
          // last contributor: Y = the contributors' partials summed in fixed CTA order (reading
          // R12).  All 256 threads over the flattened partial tile as float4 (16 B loads, 512 B
          // per warp row), 4 elements x up to 4 contributors of loads in flight per thread before
          // any store (the reduction is latency-bound otherwise).
          __threadfence();
          const int lo = flag[1], hi = flag[2];
          const int64_t sstride = (int64_t)2 * NB * kBN;
          const int tid = threadIdx.x - 64;
          const int nvt = p.M * (kBN / 4);  // float4 per tile
          // distributed: contributor ci of S reduces elements [ci*nvt/S, (ci+1)*nvt/S) of each tile
          const int S = hi - lo + 1, ci = p.dist ? cta - lo : 0, SS = p.dist ? S : 1;
          const int ebeg = (int)((int64_t)ci * nvt / SS), nv = (int)((int64_t)(ci + 1) * nvt / SS);
          // loads in flight per thread per round: kC contributors x kJ float4 (TC2_RED_J / TC2_RED_C)
#ifndef TC2_RED_J
#define TC2_RED_J 4
#endif
#ifndef TC2_RED_C
#define TC2_RED_C 4
#endif
          constexpr int kJ = TC2_RED_J, kC = TC2_RED_C;
          for (int tj = 0; tj < (two ? 2 : 1); ++tj) {
            const float* pb = p.partial + (int64_t)tj * NB * kBN;
            for (int e0 = ebeg + tid; e0 < nv; e0 += kJ * kTc2Groups * 128) {
              float4 acc[kJ];
#pragma unroll
              for (int j = 0; j < kJ; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
              for (int qb = lo; qb <= hi; qb += kC) {
                float4 v[kC][kJ];
#pragma unroll
                for (int c = 0; c < kC; ++c) {
                  const int qc = qb + c;
                  const float4* src =
                      reinterpret_cast<const float4*>(pb + (int64_t)(qc * 2 + (qc == lo ? flag[3] : 0)) * sstride);
#pragma unroll
                  for (int j = 0; j < kJ; ++j) {
                    const int e = e0 + j * kTc2Groups * 128;
                    v[c][j] = (qc <= hi && e < nv) ? __ldcg(src + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                  }
                }
#pragma unroll
                for (int c = 0; c < kC; ++c)
#pragma unroll
                  for (int j = 0; j < kJ; ++j)
                    if (qb + c <= hi) {
                      acc[j].x += v[c][j].x;
                      acc[j].y += v[c][j].y;
                      acc[j].z += v[c][j].z;
                      acc[j].w += v[c][j].w;
                    }
              }
#pragma unroll
              for (int j = 0; j < kJ; ++j) {
                const int e = e0 + j * kTc2Groups * 128;
                if (e < nv) {
                  const int m = e >> 5, c4 = e & 31;  // kBN / 4 == 32 float4 per row
                  const uint2 o = make_uint2(
                      (uint32_t)Act<BF>::from_float(acc[j].x) | ((uint32_t)Act<BF>::from_float(acc[j].y) << 16),
                      (uint32_t)Act<BF>::from_float(acc[j].z) | ((uint32_t)Act<BF>::from_float(acc[j].w) << 16));
                  const int64_t off = (int64_t)m * p.ldy + (2 * np + tj) * kBN + 4 * c4;
                  *reinterpret_cast<uint2*>(p.Y + off) = o;
                  peer_store4(p.po, off, o);
                }
              }
            }
          }
        }
        if (p.dist) {
          // second arrival after the slice: the last of the 2S resets the semaphore
          named_bar_sync(1, kTc2Groups * 128);
          if (threadIdx.x == 64) {
            const int S2 = 2 * (flag[2] - flag[1] + 1);
            if (atomicAdd(&p.sem[np], 1) == S2 - 1) p.sem[np] = 0;
          }
        } else if (flag[0] && threadIdx.x == 64) {
          p.sem[np] = 0;
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
  if (threadIdx.x == 0) peer_signal(p.po, gridDim.x);  // row f3: after every Y store of the CTA
}

template <class F>
tl_status launch_tc2(const Tc2Params& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st) {
  auto go = [&](auto kern) -> tl_status {
    if (prepare_kernel(reinterpret_cast<const void*>(kern), 227 * 1024, kTc2Threads) == 0)
      return fail(TL_ECUDA, "tc2_kernel: %s", tl_last_error());
    if (!p.dist) {
      kern<<<grid, kTc2Threads, smem_bytes, st>>>(*tmap, p);
      return TL_OK;
    }
    // the distributed reduction waits for sibling CTAs: a cooperative launch guarantees that every
    // CTA of the grid is resident at once (no deadlock even with other kernels on other streams)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTc2Threads);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, *tmap, p);
    if (e != cudaSuccess) return fail(TL_ECUDA, "tc2_kernel cooperative launch: %s", cudaGetErrorString(e));
    return TL_OK;
  };
  tl_status r;
  if (p.G < kBK) r = p.bf ? go(tc2_kernel<F, true, true>) : go(tc2_kernel<F, true, false>);
  else r = p.bf ? go(tc2_kernel<F, false, true>) : go(tc2_kernel<F, false, false>);
  if (r != TL_OK) return r;
  return check_launch("tc2_kernel");
}

}  // namespace tl
