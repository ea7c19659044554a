// gemv.cuh -- decode-shape path on CUDA cores: SURVEY §8(a) rows a3-a11, K-B2.
//
// Paper: "CUDA Cores for 1-15 tokens"; the weight pipeline of
// fig:weight-pipeline(c): (1) pipelined asynchronous copy
// global -> shared, (2) shared -> registers, (3) reinterpret, (4) vectorised cast;
// plus software pipelining and k-dimension parallelisation (stream-K).
// B200 form:
//   * the producer warp streams whole 128x128 weight tiles (2048*b contiguous bytes, one
//     cp.async.bulk each) and the k-tile's activation rows into an NS-stage shared-memory
//     ring (mbarriers); a few stages behind, the same warp pre-scales the activations by
//     2^-P per k and writes the sum of A over every 32-k sub-piece into the stage;
//   * 256 consumer threads: thread (c, kh) owns column c of the tile and the k-half kh; it
//     reads its column's k-half block words with 8-byte LDS; one LOP3 per pair of codes (layout
//     v2, common.cuh) places them in the two fp16 lanes as u * 2^(P-24) (exact fp16 subnormals --
//     no conversion instruction at all), and FHFMA (fma.rn.f32.f16: fp16 x fp16 + fp32) accumulates
//     u * A * 2^-24 exactly in fp32 (reading R10).  The zero point and the
//     group scale are applied once per 32-k sub-piece: Y += s * (2^24 * acc - z * sum(A));
//     float codes are placed on the fp16 exponent/mantissa fields (value * 2^(bias-15)) and
//     Y += s * 2^(15-bias) * acc;
//   * scales and zero points are read by the consumers straight from global memory, two tiles
//     ahead, so the TMA ring carries only two bulk copies per tile;
//   * stream-K: the linear unit space u = nt*KT + kt (n-tile major = the byte order of the
//     transformed weight) is cut into `grid` equal contiguous ranges, so every CTA streams one
//     contiguous byte range; n-tiles shared between CTAs are reduced deterministically (fixed
//     CTA order) by whichever CTA arrives last (reading R12).
#pragma once
#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

constexpr int kGemvConsumers = 256;
constexpr int kGemvThreads = kGemvConsumers + 64;  // + TMA issuer warp + preparation warp

template <class F, int MT>
struct GemvLayout {
  static constexpr int w_bytes = tile_bytes(F::bits);
  static constexpr int a_bytes = MT * kBK * 2;      // activations A'[MT][128] fp16 (pre-scaled in place)
  static constexpr int s_bytes = MT * 4 * 4;        // sum_k A over each 32-k sub-piece, fp32 [MT][4]
  static constexpr int stage_bytes = (w_bytes + a_bytes + s_bytes + 127) / 128 * 128;
  static constexpr int stages_raw = (96 * 1024) / stage_bytes;
  static constexpr int stages = stages_raw < 4 ? 4 : (stages_raw > 16 ? 16 : stages_raw);
  static constexpr int red_bytes = MT * kBN * 4;
  static constexpr int smem = stages * stage_bytes + red_bytes + 3 * stages * 8 + 16;
};

// acc += w.lo * a.lo + w.hi * a.hi  (two FHFMA reading the 16-bit halves in place)
__device__ __forceinline__ float fhfma2(uint32_t w, uint32_t a, float c) {
  asm("{\n\t.reg .b16 wl, wh, al, ah;\n\t"
      "mov.b32 {wl, wh}, %1;\n\t"
      "mov.b32 {al, ah}, %2;\n\t"
      "fma.rn.f32.f16 %0, wl, al, %0;\n\t"
      "fma.rn.f32.f16 %0, wh, ah, %0;\n\t}"
      : "+f"(c)
      : "r"(w), "r"(a));
  return c;
}

// One k-half of one tile for column c.  sc/zc: fp16 bits of the scale / zero of the half's
// two 32-k sub-pieces.
template <class F, int MT, int KH>
__device__ __forceinline__ void gemv_tile_half(const uint8_t* stage, int c, const uint16_t (&sc)[2],
                                               const uint16_t (&zc)[2], float (&tot)[MT]) {
  using L = GemvLayout<F, MT>;
  constexpr int B = F::bits;
  uint32_t bw[2 * B];
  load_block_words<B, KH>(stage, c, bw);  // layout v2: k-half KH = block KH
  const __half* As = reinterpret_cast<const __half*>(stage + L::w_bytes);
  const float* Ss = reinterpret_cast<const float*>(stage + L::w_bytes + L::a_bytes);
  float acc[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m] = 0.f;
  static_for<0, 32>([&](auto II) {
    constexpr int ii = decltype(II)::value;
    constexpr int i = KH * 32 + ii;
    // raw fields (no magic): ints u * 2^(P-24) (exact fp16 subnormal), floats value * 2^(bias-15)
    const uint32_t wp = extract_pair<F, ii>(bw, 0u);
#pragma unroll
    for (int m = 0; m < MT; ++m)
      acc[m] = fhfma2(wp, *reinterpret_cast<const uint32_t*>(As + m * kBK + 2 * i), acc[m]);
    if constexpr (ii % 16 == 15) {
      constexpr int h = ii / 16;               // sub-piece within the half
      constexpr int sp = KH * 2 + h;           // sub-piece within the tile
      const float s = __half2float(__ushort_as_half(sc[h]));
      if constexpr (F::kind != kFloat) {
        float z = 0.f;
        if constexpr (F::kind == kUint) z = __half2float(__ushort_as_half(zc[h]));
        if constexpr (F::kind == kInt) z = (float)(1 << (B - 1));
        const float c1 = s * 16777216.f, c2 = -s * z;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          tot[m] = fmaf(c2, Ss[m * 4 + sp], fmaf(c1, acc[m], tot[m]));
          acc[m] = 0.f;
        }
      } else {
        const float c1 = s * (float)(1 << (15 - F::bias));
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          tot[m] = fmaf(c1, acc[m], tot[m]);
          acc[m] = 0.f;
        }
      }
    }
  });
}

template <class F, int MT>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(GemvParams p) {
  using L = GemvLayout<F, MT>;
  constexpr int NS = L::stages;
  constexpr bool kPre = F::kind != kFloat;  // integer codes: pre-scale A by 2^-P, need sum(A)
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  float* red = reinterpret_cast<float*>(smem + NS * L::stage_bytes);
  uint64_t* full_tma = reinterpret_cast<uint64_t*>(smem + NS * L::stage_bytes + L::red_bytes);
  uint64_t* full = full_tma + NS;   // stage prepared (activations pre-scaled, sums written)
  uint64_t* empty = full + NS;
  int* flag = reinterpret_cast<int*>(empty + NS);

  const int KT = p.K / kBK;
  const int grid = gridDim.x;
  const int cta = blockIdx.x;
  const int u0 = (int)((int64_t)cta * p.units / grid);
  const int u1 = (int)((int64_t)(cta + 1) * p.units / grid);
  const int T = u1 - u0;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_tma[s], 1);
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemvConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kGemvConsumers / 32) {
    // ---------------- TMA issuer warp: weight tile + activation rows per stage ----------------
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_a = policy_evict_last();
      const uint32_t bytes = L::w_bytes + p.M * kBK * 2;
      int s = 0, ph = 0, kt = u0 % KT;
      for (int t = 0; t < T; ++t) {
        if (t >= NS) mbar_wait_sleepy(&empty[s], ph ^ 1);
        uint8_t* st = stages + s * L::stage_bytes;
        mbar_arrive_expect_tx(&full_tma[s], bytes);
        tma_bulk_g2s(st, p.wt + (int64_t)(u0 + t) * L::w_bytes, L::w_bytes, &full_tma[s], pol_w);
        for (int m = 0; m < p.M; ++m)
          tma_bulk_g2s(st + L::w_bytes + m * kBK * 2, p.A + m * p.lda + (int64_t)kt * kBK, kBK * 2, &full_tma[s],
                       pol_a);
        if (++kt == KT) kt = 0;
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  if (warp == kGemvConsumers / 32 + 1) {
    // ---------------- preparation warp: pre-scale the activations, sub-piece sums ----------------
    // lane L owns k = 4L..4L+3 = pairs 2L, 2L+1
    __half2 pre0 = __float2half2_rn(1.f), pre1 = __float2half2_rn(1.f);
    if constexpr (kPre) {
      int P0 = 0, P1 = 0;
      static_for<0, 64>([&](auto II) {
        constexpr int i = decltype(II)::value;
        constexpr int Pi = kPlan<F::kind, F::bits, F::exp>.pr[i & 31].P;
        if (i == 2 * lane) P0 = Pi;
        if (i == 2 * lane + 1) P1 = Pi;
      });
      pre0 = __float2half2_rn(__int_as_float((127 - P0) << 23));
      pre1 = __float2half2_rn(__int_as_float((127 - P1) << 23));
    }
    int s = 0, ph = 0;
    for (int t = 0; t < T; ++t) {
      mbar_wait(&full_tma[s], ph);
      if constexpr (kPre) {
        uint8_t* st = stages + s * L::stage_bytes;
        for (int m = 0; m < p.M; ++m) {
          uint2* ap = reinterpret_cast<uint2*>(st + L::w_bytes + m * kBK * 2) + lane;
          const uint2 a = *ap;
          const float2 f0 = __half22float2(u32_as_h2(a.x)), f1 = __half22float2(u32_as_h2(a.y));
          float sum = (f0.x + f0.y) + (f1.x + f1.y);
          sum += __shfl_xor_sync(0xffffffffu, sum, 4);
          sum += __shfl_xor_sync(0xffffffffu, sum, 2);
          sum += __shfl_xor_sync(0xffffffffu, sum, 1);
          if ((lane & 7) == 0)
            reinterpret_cast<float*>(st + L::w_bytes + L::a_bytes)[m * 4 + (lane >> 3)] = sum;
          *ap = make_uint2(h2_as_u32(__hmul2(u32_as_h2(a.x), pre0)), h2_as_u32(__hmul2(u32_as_h2(a.y), pre1)));
        }
        fence_proxy_async_smem();  // order these generic writes before the stage's next TMA refill
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int c = tid & (kBN - 1);
  const int kh = tid >> 7;
  float tot[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) tot[m] = 0.f;
  const bool has_zeros = p.zeros != nullptr;
  const unsigned short* sg = reinterpret_cast<const unsigned short*>(p.scales);
  const unsigned short* zg = reinterpret_cast<const unsigned short*>(p.zeros);
  // scale / zero rows of this thread's two sub-pieces of tile (nt, kt)
  // Scale / zero prefetch, PF tiles ahead (HBM latency under the weight stream is ~2 us): a
  // shift register of fp16 bits.  The group row of the prefetched tile is tracked incrementally.
  constexpr int PF = 4;
  const int lgG = p.G == 32 ? 5 : (p.G == 64 ? 6 : 0);   // G < 128: row = (k >> lgG)
  const int tpg = p.G >= kBK ? p.G / kBK : 1;             // G >= 128: k-tiles per group
  int nt_f = u0 / KT, kt_f = u0 % KT;
  int grow = lgG ? 0 : kt_f / tpg, grem = lgG ? 0 : kt_f % tpg;
  auto fetch = [&](uint16_t (&sc)[2], uint16_t (&zc)[2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = lgG ? ((kt_f * kBK + kh * 64 + h * 32) >> lgG) : grow;
      const int64_t off = (int64_t)row * p.N + nt_f * kBN + c;
      sc[h] = __ldg(sg + off);
      zc[h] = (F::kind == kUint && has_zeros) ? __ldg(zg + off) : (unsigned short)0;
    }
    if (++kt_f == KT) {
      kt_f = 0;
      ++nt_f;
      grow = 0;
      grem = 0;
    } else if (++grem == tpg) {
      grem = 0;
      ++grow;
    }
  };
  uint16_t scq[PF][2], zcq[PF][2];
#pragma unroll
  for (int pf = 0; pf < PF; ++pf)
    if (pf < T) fetch(scq[pf], zcq[pf]);

  int s = 0, ph = 0, nt = u0 / KT, kt = u0 % KT;
  for (int u = u0; u < u1; ++u) {
    const int t = u - u0;
    uint16_t sc[2] = {scq[0][0], scq[0][1]}, zc[2] = {zcq[0][0], zcq[0][1]};
#pragma unroll
    for (int pf = 0; pf + 1 < PF; ++pf) {
      scq[pf][0] = scq[pf + 1][0];
      scq[pf][1] = scq[pf + 1][1];
      zcq[pf][0] = zcq[pf + 1][0];
      zcq[pf][1] = zcq[pf + 1][1];
    }
    if (t + PF < T) fetch(scq[PF - 1], zcq[PF - 1]);
    mbar_wait(&full[s], ph);
    const uint8_t* st = stages + s * L::stage_bytes;
    if (kh == 0) gemv_tile_half<F, MT, 0>(st, c, sc, zc, tot);
    else gemv_tile_half<F, MT, 1>(st, c, sc, zc, tot);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == NS) { s = 0; ph ^= 1; }
    const int cur_nt = nt, cur_kt = kt;
    if (++kt == KT) { kt = 0; ++nt; }

    const bool last_of_tile = (cur_kt == KT - 1) || (u == u1 - 1);
    if (!last_of_tile) continue;
    // ---- flush n-tile cur_nt: reduce the two k-halves, then write Y or a partial ----
    if (kh == 1) {
#pragma unroll
      for (int m = 0; m < MT; ++m) red[m * kBN + c] = tot[m];
    }
    named_bar_sync(1, kGemvConsumers);
    if (kh == 0) {
#pragma unroll
      for (int m = 0; m < MT; ++m) tot[m] += red[m * kBN + c];
      const int n = cur_nt * kBN + c;
      const int ua = cur_nt * KT, ub = ua + KT;  // units of this n-tile
      const bool complete = (u0 <= ua) && (u1 >= ub);
      if (complete) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
          if (m < p.M) p.Y[(int64_t)m * p.ldy + n] = __float2half_rn(tot[m]);
      } else {
        const int nt_first = u0 / KT;
        const int slot = (cur_nt == nt_first) ? 0 : 1;
        float* part = p.partial + ((int64_t)(cta * 2 + slot) * p.M) * kBN;
#pragma unroll
        for (int m = 0; m < MT; ++m)
          if (m < p.M) __stcg(part + m * kBN + c, tot[m]);
        __threadfence();
        named_bar_sync(2, kBN);
        if (c == 0) {
          // the CTAs whose ranges intersect [ua, ub) are owner(ua) .. owner(ub - 1)
          const int lo = (int)((((int64_t)ua + 1) * grid - 1) / p.units);
          const int hi = (int)((((int64_t)ub) * grid - 1) / p.units);
          const int prev = atomicAdd(&p.sem[cur_nt], 1);
          flag[0] = (prev == hi - lo) ? 1 : 0;
          flag[1] = lo;
          flag[2] = hi;
          flag[3] = ((int)((int64_t)lo * p.units / grid) / KT == cur_nt) ? 0 : 1;
        }
        named_bar_sync(2, kBN);
        if (flag[0]) {
          __threadfence();
          const int lo = flag[1], hi = flag[2];
          for (int m = 0; m < p.M; ++m) {
            const float sum = streamk_sum(p.partial, lo, hi, flag[3], (int64_t)p.M * kBN, (int64_t)m * kBN + c);
            p.Y[(int64_t)m * p.ldy + n] = __float2half_rn(sum);
          }
          if (c == 0) p.sem[cur_nt] = 0;  // leave the semaphore clean for the next call
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) tot[m] = 0.f;
    named_bar_sync(1, kGemvConsumers);  // `red` / `flag` reuse
  }
}

// ---------------------------------------------------------------------------------------
template <class F, int MT>
static tl_status launch_gemv_mt(const GemvParams& p0, int grid_req, cudaStream_t st) {
  using L = GemvLayout<F, MT>;
  const int max_ctas = prepare_kernel(reinterpret_cast<const void*>(gemv_kernel<F, MT>), L::smem, kGemvThreads);
  if (max_ctas == 0) return fail(TL_ECUDA, "gemv_kernel: %s", tl_last_error());
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  GemvParams p = p0;
  int grid = grid_req > 0 ? grid_req : sms * max_ctas;
  if (grid > kGemvMaxCtas) grid = kGemvMaxCtas;  // the workspace holds partial slots for this many CTAs
  if (grid > p.units) grid = p.units;
  gemv_kernel<F, MT><<<grid, kGemvThreads, L::smem, st>>>(p);
  return check_launch("gemv_kernel");
}

template <class F>
tl_status launch_gemv(const GemvParams& p, int grid_req, cudaStream_t st) {
  if (p.M <= 1) return launch_gemv_mt<F, 1>(p, grid_req, st);
  if (p.M <= 2) return launch_gemv_mt<F, 2>(p, grid_req, st);
  if (p.M <= 4) return launch_gemv_mt<F, 4>(p, grid_req, st);
  if (p.M <= 8) return launch_gemv_mt<F, 8>(p, grid_req, st);
  return launch_gemv_mt<F, 16>(p, grid_req, st);
}

}  // namespace tl
