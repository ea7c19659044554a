// gv1.cuh -- decode GEMV on CUDA cores for M = 1 (group a multiple of 128): SURVEY §8(a) rows
// a3-a11, the "CUDA Cores for 1-15 tokens" regime of PAPER.md:546 (K-B2).
//
// Why a CUDA-core kernel at M = 1 on B200: one tcgen05.mma.kind::f16 (M = 128, K = 16) occupies the
// tensor pipe for ~74 cycles whatever its N (16 ... 128; measured, tools/mma_probe.cu), so the
// tensor-core decode kernel (tcd) needs 8 x 74 = 592 cycles per 128 x 128 weight tile and cannot
// stream tiles of b <= 6 bits faster than that (u1 ... u4 gate_up all take ~58 us).  Here each
// weight costs one FHFMA (fma.rn.f32.f16: fp16 x fp16 + fp32, exact product, fp32 accumulation --
// PAPER.md:191, reading R10) on the FMA pipe: 128 per tile per column, ~256 cycles per tile.
//
//  * the packed tile arrives with R tiles per cp.async.bulk stage, their scale / zero rows with
//    one 3-D tensor box per n-tile segment (as tcd); A[0, :] is resident in shared memory;
//  * thread = output column n of a tile; 4 groups of 4 warps take tiles t = g, g+4, ...;
//  * unpack (layout v2, common.cuh) WITHOUT the magic number: an int code u lands at bits
//    [P, P+b) of each 16-bit half, which IS the fp16 subnormal u * 2^(P-24) (exact); floats land on
//    the sign / exponent / mantissa fields (value * 2^(bias-15), exact).  FHFMA multiplies these
//    exactly, so per pair: the extraction LOP3(s) + 2 FHFMA into the accumulator of its P class;
//  * per tile: Y += s * (sum_P 2^(24-P) acc_P - z * sum_{k in tile} A[k])  (ints; the activation sums
//    per k-tile come from a prologue over the resident A row), floats: Y += s * 2^(15-bias) * acc;
//  * stream-K over (n-tile, k-tile) units with the deterministic fixed-order reduction (R12).
#pragma once

#include <cuda.h>

#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

struct Gv1Params {
  int N, K, G;
  int units;
  int ns;
  uint32_t stage_bytes;  // [R weight tiles | R scale row slices | R zero row slices]
  uint32_t stash_off;    // A[0, :] (K*2 bytes)
  uint32_t sums_off;     // sum of A over each 128-k tile (KT floats, ints only)
  uint32_t red_off;      // [4 groups][128] fp32 cross-group reduction
  uint32_t bar_off;
  const uint8_t* wt;
  const __half* A;
  const __half* scales;
  const __half* zeros;
  __half* Y;
  float* partial;  // [grid][2][128]
  int* sem;
  int static_w;
  int dbg;  // TL_GV1_DBG timing experiments (results invalid): 2 no compute
};

constexpr int kGv1Groups = 4;
constexpr int kGv1Threads = 128 + kGv1Groups * 128;

// acc += w.lo * a.lo + w.hi * a.hi  (two FHFMA on the register halves)
__device__ __forceinline__ float gv1_fhfma2(uint32_t w, uint32_t a, float c) {
  asm("{\n\t.reg .b16 wl, wh, al, ah;\n\t"
      "mov.b32 {wl, wh}, %1;\n\t"
      "mov.b32 {al, ah}, %2;\n\t"
      "fma.rn.f32.f16 %0, wl, al, %0;\n\t"
      "fma.rn.f32.f16 %0, wh, ah, %0;\n\t}"
      : "+f"(c)
      : "r"(w), "r"(a));
  return c;
}

template <class F>
__host__ __device__ constexpr int gv1_num_p() {  // accumulator classes: field positions P (ints) / 1 (floats)
  if (F::kind == kFloat) return 1;
  int n = 0;
  for (int P = 0; P < 10; ++P)
    for (int i = 0; i < 32; ++i)
      if (kPlan<F::kind, F::bits, F::exp>.pr[i].P == P) {
        ++n;
        break;
      }
  return n;
}
template <class F>
__host__ __device__ constexpr int gv1_p_index(int P) {  // accumulator index of class P
  if (F::kind == kFloat) return 0;
  int n = 0;
  for (int Q = 0; Q < P; ++Q)
    for (int i = 0; i < 32; ++i)
      if (kPlan<F::kind, F::bits, F::exp>.pr[i].P == Q) {
        ++n;
        break;
      }
  return n;
}
template <class F>
__host__ __device__ constexpr int gv1_p_of_index(int j) {
  for (int P = 0; P < 10; ++P) {
    bool used = false;
    for (int i = 0; i < 32; ++i) used = used || kPlan<F::kind, F::bits, F::exp>.pr[i].P == P;
    if (used && gv1_p_index<F>(P) == j) return P;
  }
  return 0;
}

__host__ __device__ constexpr int gv1_tiles_per_stage(int b) { return (6 + b - 1) / b; }

template <class F>
__global__ void __launch_bounds__(kGv1Threads, 1) gv1_kernel(const __grid_constant__ CUtensorMap tmapS,
                                                              const __grid_constant__ CUtensorMap tmapZ, Gv1Params p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  constexpr bool kInt = F::kind != kFloat;
  constexpr uint32_t WB = tile_bytes(F::bits);
  constexpr int kR = gv1_tiles_per_stage(F::bits);
  constexpr int NG = kGv1Groups;
  constexpr int NP = gv1_num_p<F>();
  const int NS = p.ns;
  const uint32_t SB = p.stage_bytes;
  const uint32_t st_u = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* full_tma = bars;         // [NS] weights landed (TMA) + scale / zero rows landed (cp.async)
  uint64_t* empty_tma = bars + NS;   // [NS] every tile of the stage read by its group
  uint64_t* stash_bar = bars + 2 * NS;
  int* flag = reinterpret_cast<int*>(stash_bar + 1);
  float* red = reinterpret_cast<float*>(smem + p.red_off);
  float* sums = reinterpret_cast<float*>(smem + p.sums_off);

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
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_tma[s], 1);
      mbar_init(&empty_tma[s], 4 * kR);
    }
    mbar_init(stash_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  // programmatic dependent launch: see tcd.cuh / TL_FLAG_STATIC_WEIGHTS
  if (warp == 0) {
    if (!p.static_w) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }

  if (warp == 0) {
    // ---- weight stream: stage q = tiles [q*R, q*R + R), one contiguous bulk copy ----
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      const uint8_t* src = p.wt + (int64_t)u0 * WB;
      const int tpg = p.G / kBK;
      const uint32_t box = (uint32_t)kR * 256u;
      int nt = u0 / KT, kt = u0 - (u0 / KT) * KT;
      int s = 0;
      uint32_t ph = 0;
      prefetch_tmap(&tmapS);
      if (has_zeros) prefetch_tmap(&tmapZ);
      for (int t0 = 0, q = 0; t0 < T; t0 += kR, ++q) {
        const int n_t = min(kR, T - t0);
        if (q >= NS) mbar_wait_sleepy(&empty_tma[s], ph ^ 1);
        const int n0 = min(n_t, KT - kt);
        const int nseg = n0 < n_t ? 2 : 1;
        const uint32_t bar = smem_u32(&full_tma[s]);
        const uint32_t st = st_u + s * SB;
        mbar_arrive_expect_tx_u32(bar, (uint32_t)n_t * WB + (uint32_t)nseg * box * (has_zeros ? 2u : 1u));
        tma_bulk_g2s_cta(st, src, (uint32_t)n_t * WB, bar, pol);
        const uint32_t side = st + kR * WB;
        tma_load_3d(side, &tmapS, 0, kt / tpg, nt, bar, pol);
        if (has_zeros) tma_load_3d(side + 2 * box, &tmapZ, 0, kt / tpg, nt, bar, pol);
        if (nseg == 2) {
          tma_load_3d(side + box, &tmapS, 0, 0, nt + 1, bar, pol);
          if (has_zeros) tma_load_3d(side + 3 * box, &tmapZ, 0, 0, nt + 1, bar, pol);
        }
        kt += n_t;
        while (kt >= KT) {
          kt -= KT;
          ++nt;
        }
        src += (int64_t)n_t * WB;
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---- A[0, :] into the stash (after griddepcontrol.wait: A is the previous grid's output) ----
    if (elect_one()) {
      mbar_arrive_expect_tx(stash_bar, (uint32_t)p.K * 2u);
      tma_bulk_g2s(smem + p.stash_off, p.A, (uint32_t)p.K * 2u, stash_bar, policy_evict_last());
    }
  } else if (warp >= 4) {
    // ------------------------------ dequant + FHFMA groups ------------------------------
    mbar_wait(stash_bar, 0);
    if constexpr (kInt) {
      // activation sum of every 128-k tile (zero-point term), summed once per CTA
      const __half* a = reinterpret_cast<const __half*>(smem + p.stash_off);
      const int tid = threadIdx.x - 128;  // 0..511
      for (int kt = tid; kt < KT; kt += NG * 128) {
        const uint4* v = reinterpret_cast<const uint4*>(a + kt * kBK);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint4 x = v[j];
          const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __half22float2(u32_as_h2(w4[e]));
            acc[e] += f.x + f.y;
          }
        }
        sums[kt] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      }
      named_bar_sync(2, NG * 128);
    }
    const int dw = warp - 4;
    const int g = dw >> 2;
    const int n = (warp & 3) * 32 + lane;
    const uint32_t stash_u = st_u + p.stash_off;
    const float c1mul = kInt ? 16777216.f : (float)(1 << (15 - F::bias));
    float tot = 0.f;
    int t = g;
    int qst = g / kR;
    int s = qst % NS;
    uint32_t ph = (uint32_t)(qst / NS) & 1;
    int t0 = 0;
    while (t0 < T) {
      const int ufirst = u0 + t0;
      const int nt = ufirst / KT;
      const int t1 = min(T, t0 + (KT - (ufirst - nt * KT)));
      for (; t < t1; t += NG) {
        const int kt = u0 + t - nt * KT;
        mbar_wait(&full_tma[s], ph);
        const int jt = t - qst * kR;
        const uint32_t st = st_u + s * SB;
        uint32_t words[4 * F::bits];
#pragma unroll
        for (int v = 0; v < F::bits; ++v) {
          const uint4 x = lds128(st + jt * WB + (v * 128 + n) * 16);
          words[4 * v + 0] = x.x;
          words[4 * v + 1] = x.y;
          words[4 * v + 2] = x.z;
          words[4 * v + 3] = x.w;
        }
        const int uq = u0 + qst * kR, ntq = uq / KT;
        const uint32_t srow = st + kR * WB + side_row_off(kR, p.G / kBK, nt, kt, ntq, uq - ntq * KT) + 2 * n;
        const float sc = __half2float(__ushort_as_half(lds16(srow)));
        float z = 0.f;
        if constexpr (F::kind == kUint) z = has_zeros ? __half2float(__ushort_as_half(lds16(srow + 2 * kR * 256))) : 0.f;
        if constexpr (F::kind == kInt) z = (float)(1 << (F::bits - 1));
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_tma[s]);
        float acc[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[j] = 0.f;
        const uint32_t arow = stash_u + kt * 256;
        if (!(p.dbg & 2)) static_for<0, 2>([&](auto HH) {
          constexpr int h = decltype(HH)::value;
          uint32_t bw[2 * F::bits];
#pragma unroll
          for (int j = 0; j < 2 * F::bits; ++j) bw[j] = words[tile_word(h, j)];
          static_for<0, 8>([&](auto QQ) {
            constexpr int q4 = decltype(QQ)::value;  // 4 pairs = 8 k = one 16-byte activation load
            const uint4 av = lds128(arow + (h * 32 + q4 * 4) * 4);  // broadcast: every lane, same k
            const uint32_t a4[4] = {av.x, av.y, av.z, av.w};
            static_for<0, 4>([&](auto II) {
              constexpr int i = q4 * 4 + decltype(II)::value;  // pair within the block
              constexpr int pi = kInt ? gv1_p_index<F>(kPlan<F::kind, F::bits, F::exp>.pr[i].P) : 0;
              const uint32_t x = extract_pair<F, i>(bw, 0u);
              acc[pi] = gv1_fhfma2(x, a4[decltype(II)::value], acc[pi]);
            });
          });
        });
        float d = 0.f;
        static_for<0, NP>([&](auto JJ) {
          constexpr int j = decltype(JJ)::value;
          constexpr int P = kInt ? gv1_p_of_index<F>(j) : 0;
          d = fmaf(1.f / (float)(1 << P), acc[j], d);
        });
        // ints: acc_P holds sum A * u * 2^(P-24), so d = sum_P 2^-P acc_P = 2^-24 sum_k A u
        if constexpr (kInt) tot = fmaf(sc * c1mul, d, fmaf(-sc * z, sums[kt], tot));
        else tot = fmaf(sc * c1mul, d, tot);
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
      // ---- n-tile nt done by this CTA: sum the groups, write Y or a stream-K partial ----
      red[g * kBN + n] = tot;
      named_bar_sync(1, NG * 128);
      const int ua = nt * KT, ub = ua + KT;
      const bool complete = (u0 <= ua) && (u1 >= ub);
      const int col = nt * kBN + n;
      const int slot2 = (nt == u0 / KT) ? 0 : 1;
      if (g == 0) {
        float v = 0.f;
#pragma unroll
        for (int gg = 0; gg < NG; ++gg) v += red[gg * kBN + n];
        if (complete) p.Y[col] = __float2half_rn(v);
        else __stcg(p.partial + (int64_t)(cta * 2 + slot2) * kBN + n, v);
      }
      if (!complete) {
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
        if (flag[0] && g == 0) {
          const float sum = streamk_sum(p.partial, flag[1], flag[2], flag[3], (int64_t)kBN, (int64_t)n);
          p.Y[col] = __float2half_rn(sum);
          if (threadIdx.x == 128) p.sem[nt] = 0;
        }
      }
      named_bar_sync(1, NG * 128);
      tot = 0.f;
      t0 = t1;
    }
  }
}

template <class F>
tl_status launch_gv1(const Gv1Params& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st) {
  if (prepare_kernel(reinterpret_cast<const void*>(gv1_kernel<F>), 227 * 1024, kGv1Threads) == 0)
    return fail(TL_ECUDA, "gv1_kernel: %s", tl_last_error());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGv1Threads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gv1_kernel<F>, tmap[0], tmap[1], p);
  if (e != cudaSuccess) return fail(TL_ECUDA, "gv1_kernel launch: %s", cudaGetErrorString(e));
  return check_launch("gv1_kernel");
}

}  // namespace tl
