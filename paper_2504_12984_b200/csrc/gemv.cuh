// gemv.cu -- decode-shape path (M <= 16) on CUDA cores: SURVEY §8(a) rows a3-a11, K-B2.
//
// Paper: "CUDA Cores for 1-15 tokens"; the weight pipeline of
// fig:weight-pipeline(c): (1) pipelined asynchronous copy
// global -> shared, (2) shared -> registers, (3) reinterpret, (4) vectorised cast;
// plus software pipelining and k-dimension parallelisation (stream-K)
// (PAPER.md:546).  B200 form:
//   * a producer warp streams whole 128x128 weight tiles (2048*b contiguous bytes,
//     one cp.async.bulk each) plus the activation / scale / zero slices of that
//     k-tile into an NS-stage shared-memory ring guarded by mbarriers;
//   * 256 consumer threads: thread (c, kh) owns column c of the tile and the k-half
//     kh; it reads its column's segment words with 16-byte LDS, turns every pair of
//     codes into an exact fp16x2 (u - z) with one LOP3 + one HFMA2 (common.cuh
//     pair_value), and accumulates w*A with FHFMA (fp16 x fp16 + fp32 -> fp32, the
//     PTX fma.rn.f32.f16), i.e. fp32 accumulation (reading R10);
//     the group scale is applied in fp32 once per (group, k-half) sub-piece;
//   * stream-K: the linear unit space u = nt*KT + kt (n-tile major = the byte order
//     of the transformed weight) is cut into `grid` equal contiguous ranges, so
//     every CTA streams one contiguous byte range and the load is balanced to one
//     tile; n-tiles shared between CTAs are reduced deterministically (fixed CTA
//     order) by whichever CTA arrives last (reading R12).
#pragma once
#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

constexpr int kGemvConsumers = 256;
constexpr int kGemvThreads = kGemvConsumers + 32;

template <class F, int MT>
struct GemvLayout {
  static constexpr int w_bytes = tile_bytes(F::bits);
  static constexpr int a_bytes = MT * kBK * 2;  // fp16 [MT][128]
  static constexpr int sz_bytes = 4 * kBN * 2;  // up to 4 group rows of 128 fp16
  static constexpr int stage_bytes = w_bytes + a_bytes + 2 * sz_bytes;
  static constexpr int stages = (stage_bytes * 8 <= 96 * 1024) ? 8 : ((stage_bytes * 4 <= 96 * 1024) ? 4 : 3);
  static constexpr int red_bytes = MT * kBN * 4;
  static constexpr int smem = stages * stage_bytes + red_bytes + 2 * stages * 8 + 16;
};

__device__ __forceinline__ float fhfma(uint16_t a, uint16_t b, float c) {
  asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(c) : "h"(a), "h"(b));
  return c;
}

template <class F, int MT, int KH>
__device__ __forceinline__ void gemv_tile_half(const uint8_t* stage, int c, uint32_t magic, int G, bool has_zeros,
                                               float (&tot)[MT]) {
  using L = GemvLayout<F, MT>;
  constexpr int B = F::bits;
  // this thread's words: segment s, words j in [2w*KH, 2w*KH + 2w)
  uint32_t words[4 * B];
#pragma unroll
  for (int s = 0; s < F::nseg; ++s) {
    constexpr int dummy = 0;
    (void)dummy;
    const int w = seg_width(B, s), base = seg_base(B, s);
    const uint8_t* sp = stage + 2048 * base;
    if (w == 1) {
      const uint2 x = *reinterpret_cast<const uint2*>(sp + c * 16 + KH * 8);
      words[4 * base + 2 * KH + 0] = x.x;
      words[4 * base + 2 * KH + 1] = x.y;
    } else {
#pragma unroll
      for (int v = 0; v < w / 2; ++v) {
        const int vv = KH * (w / 2) + v;
        const uint4 x = *reinterpret_cast<const uint4*>(sp + (vv * 128 + c) * 16);
        words[4 * base + 4 * vv + 0] = x.x;
        words[4 * base + 4 * vv + 1] = x.y;
        words[4 * base + 4 * vv + 2] = x.z;
        words[4 * base + 4 * vv + 3] = x.w;
      }
    }
  }
  const __half* As = reinterpret_cast<const __half*>(stage + L::w_bytes);
  const __half* Ss = reinterpret_cast<const __half*>(stage + L::w_bytes + L::a_bytes);
  const __half* Zs = reinterpret_cast<const __half*>(stage + L::w_bytes + L::a_bytes + L::sz_bytes);
  // sub-pieces of 32 k (16 pairs): every group boundary (G = 32, 64, 128*j) is one
  const int lg = G == 32 ? 5 : 6;          // log2 G for G < 128
  float acc[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m] = 0.f;
  PairConsts pc;
  pc.magic = magic;
  float s = 0.f;
  static_for<0, 32>([&](auto II) {
    constexpr int i = KH * 32 + decltype(II)::value;
    if constexpr (i % 16 == 0) {
      const int r = (G >= kBK) ? 0 : ((2 * i) >> lg);  // group row of this sub-piece in the stage slice
      s = __half2float(Ss[r * kBN + c]);
      float z = 0.f;
      if constexpr (F::kind == kUint) z = has_zeros ? __half2float(Zs[r * kBN + c]) : 0.f;
      if constexpr (F::kind == kInt) z = (float)(1 << (B - 1));
      make_pair_consts<F>(pc, z);
    }
    const uint32_t wp = h2_as_u32(pair_value<F, i>(words, pc));
    const uint16_t wlo = (uint16_t)(wp & 0xFFFF), whi = (uint16_t)(wp >> 16);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const uint32_t a2 = *reinterpret_cast<const uint32_t*>(As + m * kBK + 2 * i);
      acc[m] = fhfma(wlo, (uint16_t)(a2 & 0xFFFF), acc[m]);
      acc[m] = fhfma(whi, (uint16_t)(a2 >> 16), acc[m]);
    }
    if constexpr (i % 16 == 15) {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        tot[m] = fmaf(s, acc[m], tot[m]);
        acc[m] = 0.f;
      }
    }
  });
}

template <class F, int MT>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(GemvParams p) {
  using L = GemvLayout<F, MT>;
  constexpr int NS = L::stages;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  float* red = reinterpret_cast<float*>(smem + NS * L::stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * L::stage_bytes + L::red_bytes);
  uint64_t* empty = full + NS;
  int* flag = reinterpret_cast<int*>(empty + NS);

  const int KT = p.K / kBK;
  const int grid = gridDim.x;
  const int cta = blockIdx.x;
  const int u0 = (int)((int64_t)cta * p.units / grid);
  const int u1 = (int)((int64_t)(cta + 1) * p.units / grid);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemvConsumers / 32);
    }
    fence_mbar_init();
  }
  // zero the activation rows >= M of every stage once (TMA never writes them)
  for (int s = 0; s < NS; ++s) {
    __half* As = reinterpret_cast<__half*>(stages + s * L::stage_bytes + L::w_bytes);
    for (int e = tid; e < (MT - p.M) * kBK; e += kGemvThreads) As[p.M * kBK + e] = __float2half_rn(0.f);
  }
  fence_proxy_async_smem();
  __syncthreads();

  const int spt = p.G >= kBK ? 1 : kBK / p.G;  // group rows per tile
  const bool has_zeros = p.zeros != nullptr;

  if (warp == kGemvConsumers / 32) {
    // ---------------- producer warp ----------------
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_a = policy_evict_last();
      const uint32_t bytes = L::w_bytes + p.M * kBK * 2 + spt * kBN * 2 * (has_zeros ? 2 : 1);
      int s = 0, ph = 0, nt = u0 / KT, kt = u0 % KT;
      for (int u = u0; u < u1; ++u) {
        if (u - u0 >= NS) mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = stages + s * L::stage_bytes;
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_bulk_g2s(st, p.wt + (int64_t)u * L::w_bytes, L::w_bytes, &full[s], pol_w);
        for (int m = 0; m < p.M; ++m)
          tma_bulk_g2s(st + L::w_bytes + m * kBK * 2, p.A + m * p.lda + (int64_t)kt * kBK, kBK * 2, &full[s], pol_a);
        const int g0 = (int)((int64_t)kt * kBK / p.G);
        for (int r = 0; r < spt; ++r) {
          tma_bulk_g2s(st + L::w_bytes + L::a_bytes + r * kBN * 2, p.scales + (int64_t)(g0 + r) * p.N + nt * kBN,
                       kBN * 2, &full[s], pol_w);
          if (has_zeros)
            tma_bulk_g2s(st + L::w_bytes + L::a_bytes + L::sz_bytes + r * kBN * 2,
                         p.zeros + (int64_t)(g0 + r) * p.N + nt * kBN, kBN * 2, &full[s], pol_w);
        }
        if (++kt == KT) { kt = 0; ++nt; }
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int c = tid & (kBN - 1);
  const int kh = tid >> 7;
  float tot[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) tot[m] = 0.f;

  int s = 0, ph = 0, nt = u0 / KT, kt = u0 % KT;
  for (int u = u0; u < u1; ++u) {
    mbar_wait(&full[s], ph);
    const uint8_t* st = stages + s * L::stage_bytes;
    if (kh == 0) gemv_tile_half<F, MT, 0>(st, c, p.magic, p.G, has_zeros, tot);
    else gemv_tile_half<F, MT, 1>(st, c, p.magic, p.G, has_zeros, tot);
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
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
        }
        named_bar_sync(2, kBN);
        if (flag[0]) {
          __threadfence();
          const int lo = flag[1], hi = flag[2];
          for (int m = 0; m < p.M; ++m) {
            float sum = 0.f;
            for (int q = lo; q <= hi; ++q) {
              const int q_first = (int)((int64_t)q * p.units / grid) / KT;
              const int qslot = (cur_nt == q_first) ? 0 : 1;
              sum += __ldcg(p.partial + ((int64_t)(q * 2 + qslot) * p.M + m) * kBN + c);
            }
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
  static int max_ctas = 0;  // per instantiation: resident CTAs per SM
  if (max_ctas == 0) {
    if (cudaFuncSetAttribute(gemv_kernel<F, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::smem) != cudaSuccess)
      return fail(TL_ECUDA, "cudaFuncSetAttribute(gemv smem=%d)", L::smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_kernel<F, MT>, kGemvThreads, L::smem);
    max_ctas = occ > 0 ? occ : 1;
  }
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  GemvParams p = p0;
  int grid = grid_req > 0 ? grid_req : sms * max_ctas;
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
