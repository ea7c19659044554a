// tcs.cuh -- decode-batch tensor-core path (M <= 16, G >= 128): SURVEY §8(a) rows a3-a11.
//
// Same MMA as tc.cuh (swap-AB, tcgen05.mma.cta_group::1.kind::f16, M_mma = 128 weight
// columns, N_mma = 16 batch rows) but built so the per-weight work is ONE LOP3 per pair:
//
//  * the dequantized W^T tile is written to TENSOR MEMORY with tcgen05.st and fed to the MMA as
//    its A operand ("TS" form): no shared-memory staging, no swizzle arithmetic;
//  * an integer code u is not converted at all: the pair's bits placed at bit P of each
//    16-bit half ARE the fp16 subnormal u * 2^(P-24) (exact -- fp16 subnormals are multiplied
//    exactly by the tensor core, checked by tools/tc_probe.cu), and the activation operand is
//    pre-scaled by 2^-P per k, so the MMA accumulates 2^-24 * sum_k A[m,k] u[k,n] in fp32;
//  * the zero point is removed with one exact HSUB2 per pair ((u - z) * 2^(P-24) is still an
//    exact fp16), and the group scale is applied once per (128-k tile, batch row) in fp32 from
//    TMEM: Y += s * 2^24 * D  (int codes are stored offset-binary, so ints use z = 2^(b-1));
//    float codes are placed on the fp16 exponent/mantissa fields (value * 2^(bias-15), exact)
//    and Y += s * 2^(15-bias) * D.  Every product is exact; sums are fp32.
//
// Roles (576 threads): warp 0 TMA producer (weight tile, raw activation rows, scale/zero rows);
// warp 1 TMEM owner + MMA issuer; warps 2..17 = 4 dequant groups of 4 warps (warp%4 = TMEM
// lane quarter).  Group g handles tiles t = g, g+4, ... of the CTA's stream-K range: it unpacks
// its tile into TMEM slot g, converts the activation slice into the 128B-swizzled MMA operand,
// hands both to the MMA warp, and then -- one group-iteration late, so it never waits for its own
// MMA -- applies the fixup of its previous tile from accumulator slot (t-4)&7 into per-thread fp32
// totals.  At the end of every 128-column n-tile the four groups' totals are summed through
// shared memory and written (or stored as stream-K partials).
#pragma once

#include <cuda.h>

#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

struct TcsParams {
  int M, N, K, G;
  int units;
  int ns, lg_ns;                      // TMA ring stages (power of two)
  uint32_t stage_bytes;               // packed tile | scale row | zero row | M activation rows
  uint32_t ap_off, st_off, red_off, bar_off;
  const uint8_t* wt;
  const __half* A;
  int64_t lda;
  const __half* scales;
  const __half* zeros;
  __half* Y;
  int64_t ldy;
  float* partial;  // [grid][2][16][128]
  int* sem;
  long long* trace;  // optional [5][256] clock64 stamps of CTA 0 (debug)
};

constexpr int kTcsGroups = 3;        // dequant groups; each owns 2 TMEM W^T slots
constexpr int kTcsThreads = 64 + kTcsGroups * 128;
constexpr int kTcsNB = 16;
constexpr uint32_t kTcsApBytes = kTcsNB * 256;  // activation operand tile (16 rows x 128 k fp16)
constexpr int kTcsWSlots = 2 * kTcsGroups;        // W^T tiles in TMEM (64 columns each)
// TMEM columns: W^T slots [0,384) (6 x 64), accumulators [384,512) (8 x 16)
constexpr uint32_t kTcsAccCol = 64 * kTcsWSlots;

__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem], kind::f16
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ uint64_t sw128_desc_s(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int B>
__device__ __forceinline__ void tcs_load_words(uint32_t wtile, int n, uint32_t* words) {
#pragma unroll
  for (int s = 0; s < num_segs(B); ++s) {
    const int w = seg_width(B, s), base = seg_base(B, s);
#pragma unroll
    for (int v = 0; v < w; ++v) {
      const uint4 x = lds128(wtile + 2048 * base + (v * 128 + n) * 16);
      words[4 * base + 4 * v + 0] = x.x;
      words[4 * base + 4 * v + 1] = x.y;
      words[4 * base + 4 * v + 2] = x.z;
      words[4 * base + 4 * v + 3] = x.w;
    }
  }
}

// One 128x128 tile: row n's 64 pairs -> TMEM slot (4 x tcgen05.st of 16 columns).
// ints: the raw pair is (u * 2^(P-24)) in fp16 (subnormal or small normal, exact); one HSUB2
// with the row's constant z * 2^(P-24) leaves (u - z) * 2^(P-24), still exact, so the zero point
// needs no correction term later.  floats: the raw pair is value * 2^(bias-15), exact.
template <class F>
__device__ __forceinline__ void tcs_dequant_tile(const uint32_t* words, uint32_t tslot, const uint32_t (&cz)[11]) {
  static_for<0, 4>([&](auto CC) {
    constexpr int c = decltype(CC)::value;
    uint32_t r[16];
    static_for<0, 16>([&](auto II) {
      constexpr int ii = decltype(II)::value;
      constexpr int i = c * 16 + ii;
      const uint32_t x = raw_pair_bits<F, i>(words);
      if constexpr (F::kind != kFloat) r[ii] = h2_as_u32(__hsub2(u32_as_h2(x), u32_as_h2(cz[SubP<F::bits, i>::value])));
      else r[ii] = x;
    });
    tmem_st_32x32b_x16(tslot + c * 16, r);
  });
}

// z * 2^(P-24) as fp16x2 for every P a pair of a b-bit code can sit at
template <class F>
__device__ __forceinline__ void tcs_zero_consts(float z, uint32_t (&cz)[11]) {
#pragma unroll
  for (int P = 0; P <= 10; ++P) {
    if (pair_p_used<F::bits>(P)) {
      const __half h = __float2half_rn(z * __int_as_float((127 + P - 24) << 23));
      cz[P] = h2_as_u32(__halves2half2(h, h));
    }
  }
}

__device__ __forceinline__ void tcs_stamp(const TcsParams& p, int kind, int t) {
  if (p.trace != nullptr && blockIdx.x == 0 && t < 256) p.trace[kind * 256 + t] = clock64();  // kinds 0..7
}

template <class F, int MT>
__global__ void __launch_bounds__(kTcsThreads, 1) tcs_kernel(TcsParams p) {
  // MT: compile-time bound on M (1 or 16) -- sizes the per-thread totals and activation buffers
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr bool kD2 = F::kind != kFloat;  // zero point / offset-binary correction needed
  constexpr uint32_t WB = tile_bytes(F::bits);
  const int NS = p.ns;
  const uint32_t stage_bytes = p.stage_bytes;
  uint8_t* ap = smem + p.ap_off;        // 4 x activation operand tiles (swizzled, prescaled)
  uint8_t* st = smem + p.st_off;        // NS x packed weight tiles
  float* red = reinterpret_cast<float*>(smem + p.red_off);  // [4][M][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* full_tma = bars;
  uint64_t* empty_tma = bars + NS;
  uint64_t* full_w = bars + 2 * NS;     // [6]  W^T slot written by its group
  uint64_t* empty_w = full_w + kTcsWSlots;  // [6]  MMA done with W^T slot
  uint64_t* full_acc = empty_w + kTcsWSlots;  // [8]  accumulator slot t&7 ready
  uint64_t* empty_acc = full_acc + 8;   // [8]  accumulator slot read back
  uint32_t* tslot_ptr = reinterpret_cast<uint32_t*>(empty_acc + 8);
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
      mbar_init(&empty_tma[s], 4);
    }
    for (int i = 0; i < kTcsWSlots; ++i) {
      mbar_init(&full_w[i], 4);
      mbar_init(&empty_w[i], 1);
    }
    for (int i = 0; i < 8; ++i) {
      mbar_init(&full_acc[i], 1);
      mbar_init(&empty_acc[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tslot_ptr, 512);
    tmem_relinquish();
  }
  // zero the activation operand tiles (rows >= M stay zero)
  for (uint32_t i = threadIdx.x; i < kTcsWSlots * kTcsApBytes / 16; i += kTcsThreads)
    sts128(smem_u32(ap) + i * 16, 0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot_ptr;

  if (warp == 0) {
    // ------------------------------ TMA producer: packed weight tiles only ------------------------------
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      for (int t = 0; t < T; ++t) {
        const int s = t & (NS - 1);
        if (t >= NS) mbar_wait_sleepy(&empty_tma[s], ((t >> p.lg_ns) - 1) & 1);
        tcs_stamp(p, 0, t);
        mbar_arrive_expect_tx(&full_tma[s], WB);
        tma_bulk_g2s(st + s * stage_bytes, p.wt + (int64_t)(u0 + t) * WB, WB, &full_tma[s], pol_w);
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (one thread for the whole loop) ------------------------------
    if (elect_one()) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(kTcsNB >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t bd_base = sw128_desc_s(smem_u32(ap));
      for (int t = 0; t < T; ++t) {
        // tile t belongs to group t%3; its k-th tile (k = t/3) uses W^T slot 2g + (k&1)
        const int gk = t / kTcsGroups, gg = t - gk * kTcsGroups;
        const int ws = 2 * gg + (gk & 1), as = t & 7;
        mbar_wait(&full_w[ws], (gk >> 1) & 1);
        tcs_stamp(p, 7, t);
        if (t >= 8) mbar_wait(&empty_acc[as], ((t >> 3) - 1) & 1);
        tc_fence_after();
        tcs_stamp(p, 1, t);
        // B descriptor: +32 B per k-step inside a 64-k block, +2 KB per block (16-B units)
        const uint64_t bd0 = bd_base + (uint64_t)(ws * (kTcsApBytes >> 4));
        const uint32_t d = tmem + kTcsAccCol + as * kTcsNB;
        const uint32_t aw = tmem + ws * 64;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          tc_mma_f16_ts(d, aw + j * 8, bd0 + (uint64_t)((j >> 2) * 128 + (j & 3) * 2), idesc, j > 0 ? 1u : 0u);
        tcs_stamp(p, 5, t);
        tc_commit(&empty_w[ws]);
        tc_commit(&full_acc[as]);
        tcs_stamp(p, 6, t);
      }
    }
  } else {
    // ------------------------------ dequant groups ------------------------------
    const int dw = warp - 2;            // 0..11
    const int g = dw >> 2;              // dequant group
    const int q = warp & 3;             // TMEM lane quarter
    const int n = q * 32 + lane;        // row of W^T = output column within the n-tile
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t st_u = smem_u32(st);
    // activation conversion: lane L of warp q handles the 4 k of chunk c = 8q + (L&7)
    // (pairs 2c, 2c+1) of rows m = (L>>3) + 4j, so every warp shares the work at any M
    const int ac = q * 8 + (lane & 7);
    const int ar0 = lane >> 3;
    float pre0 = 1.f, pre1 = 1.f;  // 2^-P for the lane's two pairs (ints); 1 for floats
    if constexpr (kD2) {
      int P0 = 0, P1 = 0;
      static_for<0, 64>([&](auto II) {
        constexpr int i = decltype(II)::value;
        if (i == 2 * ac) P0 = SubP<F::bits, i>::value;
        if (i == 2 * ac + 1) P1 = SubP<F::bits, i>::value;
      });
      pre0 = __int_as_float((127 - P0) << 23);
      pre1 = __int_as_float((127 - P1) << 23);
    }
    const __half2 pre0h = __float2half2_rn(pre0), pre1h = __float2half2_rn(pre1);
    const uint32_t a_kb = (uint32_t)(ac >> 4) * (kTcsNB * 128);   // 64-k block
    const uint32_t a_c = (uint32_t)((ac & 15) >> 1);              // 16-byte chunk in the row
    const uint32_t a_h = (uint32_t)(ac & 1) * 8;                  // half of the chunk
    const float c1mul = kD2 ? 16777216.f : (float)(1 << (15 - F::bias));
    constexpr int RJ = (MT + 3) / 4;  // activation rows per warp
    float tot[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) tot[m] = 0.f;

    auto load_a = [&](int kt_, uint2 (&ar)[RJ]) {
#pragma unroll
      for (int j = 0; j < RJ; ++j) {
        const int m = ar0 + 4 * j;
        if (m < p.M)
          ar[j] = __ldg(reinterpret_cast<const uint2*>(p.A + (int64_t)m * p.lda + (int64_t)kt_ * kBK + ac * 4));
      }
    };
    // raw fp16 bits; converted only in the (lagged) fixup so the load latency is never waited on
    auto load_sz = [&](int nt_, int kt_, uint16_t& sc_, uint16_t& z_) {
      const int gg = (int)((int64_t)kt_ * kBK / p.G);
      const int64_t off = (int64_t)gg * p.N + nt_ * kBN + n;
      sc_ = __ldg(reinterpret_cast<const unsigned short*>(p.scales) + off);
      z_ = 0;
      if constexpr (F::kind == kUint)
        if (has_zeros) z_ = __ldg(reinterpret_cast<const unsigned short*>(p.zeros) + off);
    };
    // the fixup of tile tp (accumulator slot tp&7), applied one group-iteration late so the
    // dequant never waits for its own MMA
    // the fixup of tile tp (accumulator slot tp&7): Y += s * c1 * D, applied one group-iteration
    // late so the dequant never waits for its own MMA
    auto fixup = [&](int tp, uint16_t scb) {
      const float sc_ = __half2float(__ushort_as_half(scb));
      const int as = tp & 7;
      mbar_wait(&full_acc[as], (tp >> 3) & 1);
      tc_fence_after();
      uint32_t d[16];
      tmem_ld_32x32b_x16(tmem + lane_off + kTcsAccCol + as * kTcsNB, d);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_acc[as]);
      if (lane == 0 && q == 2) tcs_stamp(p, 4, tp);
      const float c1 = sc_ * c1mul;
#pragma unroll
      for (int m = 0; m < MT; ++m)
        if (m < p.M) tot[m] = fmaf(c1, __uint_as_float(d[m]), tot[m]);
      if (lane == 0 && q == 2) tcs_stamp(p, 8, tp);
    };

    // side inputs (activation slice from L2, scale / zero from HBM) are prefetched two group
    // iterations ahead into a 2-slot register ring: HBM latency under the weight stream is ~2 us
    uint2 araw_q[2][RJ];
    uint16_t sc_q[2] = {0, 0}, z_q[2] = {0, 0};
    int t = g;
    int kk = 0;                  // this group's tile counter (t = g + 3*kk)
    int nt_f = (u0 + t) / KT, kt_f = (u0 + t) - ((u0 + t) / KT) * KT;  // tile being prefetched
    auto advance_f = [&]() {
      kt_f += kTcsGroups;
      while (kt_f >= KT) { kt_f -= KT; ++nt_f; }
    };
#pragma unroll
    for (int pf = 0; pf < 2; ++pf) {
      if (t + pf * kTcsGroups < T) {
        load_a(kt_f, araw_q[pf]);
        load_sz(nt_f, kt_f, sc_q[pf], z_q[pf]);
      }
      advance_f();
    }
    int tp = -1;                 // this group's tile whose fixup is pending
    uint16_t sc_p = 0;           // its scale (fp16 bits)
    int t0 = 0;
    while (t0 < T) {
      const int ufirst = u0 + t0;
      const int nt = ufirst / KT;
      const int t1 = min(T, t0 + (KT - (ufirst - nt * KT)));
      for (; t < t1; t += kTcsGroups, ++kk) {
        if (lane == 0 && q == 2) tcs_stamp(p, 9, t);
        const int ws = 2 * g + (kk & 1);
        const uint32_t tslot = tmem + lane_off + ws * 64;
        const uint32_t ap_u = smem_u32(ap + ws * kTcsApBytes);
        const int pq = kk & 1;
        uint2 araw[RJ];
#pragma unroll
        for (int j = 0; j < RJ; ++j) araw[j] = pq ? araw_q[1][j] : araw_q[0][j];
        const uint16_t sc_c = pq ? sc_q[1] : sc_q[0], z_c = pq ? z_q[1] : z_q[0];
        if (t + 2 * kTcsGroups < T) {
          if (pq) {
            load_a(kt_f, araw_q[1]);
            load_sz(nt_f, kt_f, sc_q[1], z_q[1]);
          } else {
            load_a(kt_f, araw_q[0]);
            load_sz(nt_f, kt_f, sc_q[0], z_q[0]);
          }
        }
        advance_f();
        const int s = t & (NS - 1);
        if (lane == 0 && q == 2) tcs_stamp(p, 10, t);
        mbar_wait(&full_tma[s], (t >> p.lg_ns) & 1);
        if (lane == 0 && q == 2) tcs_stamp(p, 11, t);
        if (kk >= 2) mbar_wait(&empty_w[ws], ((kk >> 1) - 1) & 1);
        if (lane == 0 && q == 2) tcs_stamp(p, 2, t);
        uint32_t words[4 * F::bits];
        tcs_load_words<F::bits>(st_u + s * stage_bytes, n, words);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_tma[s]);   // the stage goes back to the TMA ring now
        uint32_t cz[11];
        if constexpr (F::kind == kUint) tcs_zero_consts<F>(__half2float(__ushort_as_half(z_c)), cz);
        if constexpr (F::kind == kInt) tcs_zero_consts<F>((float)(1 << (F::bits - 1)), cz);
        tcs_dequant_tile<F>(words, tslot, cz);
        // activation operand, prescaled by 2^-P per k (ints); this warp converts its k-quarter
#pragma unroll
        for (int j = 0; j < RJ; ++j) {
          const int m = ar0 + 4 * j;
          if (m < p.M) {
            __half2 a0 = u32_as_h2(araw[j].x), a1 = u32_as_h2(araw[j].y);
            if constexpr (kD2) {
              a0 = __hmul2(a0, pre0h);
              a1 = __hmul2(a1, pre1h);
            }
            const uint32_t dst = ap_u + a_kb + m * 128 + (((a_c ^ (uint32_t)(m & 7))) << 4) + a_h;
            asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(dst), "r"(h2_as_u32(a0)), "r"(h2_as_u32(a1))
                         : "memory");
          }
        }
        tmem_st_wait();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_w[ws]);
        if (lane == 0 && q == 2) tcs_stamp(p, 3, t);
        if (tp >= 0) fixup(tp, sc_p);
        tp = t;
        sc_p = sc_c;
      }
      // drain this group's pending fixup before the n-tile is summed
      if (tp >= 0) {
        fixup(tp, sc_p);
        tp = -1;
      }
      // ---- n-tile nt done by this CTA: sum the 4 groups' totals, write Y or a partial ----
#pragma unroll
      for (int m = 0; m < MT; ++m)
        if (m < p.M) red[(g * p.M + m) * kBN + n] = tot[m];
      named_bar_sync(1, kTcsGroups * 128);
      const int ua = nt * KT, ub = ua + KT;
      const bool complete = (u0 <= ua) && (u1 >= ub);
      const int col = nt * kBN + n;
      const int slot2 = (nt == u0 / KT) ? 0 : 1;
      float* part = p.partial + ((int64_t)(cta * 2 + slot2) * kTcsNB) * kBN;
      for (int m = g; m < p.M; m += kTcsGroups) {
        const float v = red[(0 * p.M + m) * kBN + n] + red[(1 * p.M + m) * kBN + n] +
                        red[(2 * p.M + m) * kBN + n];
        if (complete) p.Y[(int64_t)m * p.ldy + col] = __float2half_rn(v);
        else __stcg(part + (int64_t)m * kBN + n, v);
      }
      if (!complete) {
        __threadfence();
        named_bar_sync(1, kTcsGroups * 128);
        if (threadIdx.x == 64) {
          const int lo = (int)((((int64_t)ua + 1) * grid - 1) / p.units);
          const int hi = (int)((((int64_t)ub) * grid - 1) / p.units);
          const int prev = atomicAdd(&p.sem[nt], 1);
          flag[0] = (prev == hi - lo) ? 1 : 0;
          flag[1] = lo;
          flag[2] = hi;
        }
        named_bar_sync(1, kTcsGroups * 128);
        if (flag[0]) {
          __threadfence();
          const int lo = flag[1], hi = flag[2];
          for (int m = g; m < p.M; m += kTcsGroups) {
            float sum = 0.f;
            for (int qq = lo; qq <= hi; ++qq) {
              const int q_first = (int)((int64_t)qq * p.units / grid) / KT;
              const int qslot = (nt == q_first) ? 0 : 1;
              sum += __ldcg(p.partial + ((int64_t)(qq * 2 + qslot) * kTcsNB + m) * kBN + n);
            }
            p.Y[(int64_t)m * p.ldy + col] = __float2half_rn(sum);
          }
          if (threadIdx.x == 64) p.sem[nt] = 0;
        }
      }
      named_bar_sync(1, kTcsGroups * 128);
#pragma unroll
      for (int m = 0; m < MT; ++m) tot[m] = 0.f;
      t0 = t1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <class F, int MT>
tl_status launch_tcs_mt(const TcsParams& p, int grid, uint32_t smem_bytes, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(tcs_kernel<F, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
        cudaSuccess)
      return fail(TL_ECUDA, "cudaFuncSetAttribute(tcs smem)");
    configured = true;
  }
  tcs_kernel<F, MT><<<grid, kTcsThreads, smem_bytes, st>>>(p);
  return check_launch("tcs_kernel");
}

template <class F>
tl_status launch_tcs(const TcsParams& p, int grid, uint32_t smem_bytes, cudaStream_t st) {
  return p.M <= 1 ? launch_tcs_mt<F, 1>(p, grid, smem_bytes, st) : launch_tcs_mt<F, kTcsNB>(p, grid, smem_bytes, st);
}

}  // namespace tl
