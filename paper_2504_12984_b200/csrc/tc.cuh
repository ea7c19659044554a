// tc.cuh -- batched path on the 5th-generation tensor cores (tcgen05): SURVEY §8(a)
// rows a3-a11, K-B3.
//
// Paper: "Tensor Cores for 16 or more tokens" with software pipelining and stream-K
// (PAPER.md:546); the weight pipeline of fig:weight-pipeline(c):
// async copy to shared memory, load to registers, reinterpret, vectorised cast, then the
// tensor-core MMA on the cast tile.  B200 form (swap-AB):
//
//   D[n 128, m NB] (fp32, TMEM) += W^T[n 128, k 16] (fp16, smem) x A^T[k 16, m NB] (fp16, smem)
//
// so the weight tile fills the 128 rows of tcgen05.mma.cta_group::1.kind::f16 and the
// batch is the MMA N dimension (16..256), i.e. small batches waste no tensor rows.
//   warp 0      TMA producer: per k-tile one cp.async.bulk of the packed 128x128 weight
//               tile (2048*b B), the 128B-swizzled activation boxes (cp.async.bulk.tensor,
//               zero-filled beyond M) and the scale / zero slices -> NS-stage ring.
//   warp 1      TMEM allocator + MMA issuer (one elected thread): 8 MMAs (K=16) per
//               k-tile, tcgen05.commit frees the smem stages and signals the epilogue.
//   warps 2..9  dequant (row n = lane + 32*(warp%4), k-half = (warp-2)/4): 16-byte LDS of
//               the segment words, LOP3 + HFMA2 unpack to exact fp16 pairs (pair_value),
//               HMUL2 by the group scale (reading R9), 16-byte STS into the 128B-swizzled
//               K-major operand tile; the same warps are the epilogue (tcgen05.ld ->
//               fp16 RN -> Y, or stream-K partials with a deterministic fixup).
// Accumulators are double-buffered in TMEM so the epilogue of one n-tile overlaps the
// MMAs of the next.
#pragma once

#include <cuda.h>

#include "paths.cuh"
#include "ptx.cuh"

namespace tl {

struct TcParams {
  int M, N, K, G;
  int NB;          // MMA N = batch tile (multiple of 16, <= 256)
  int units;       // (N/128) * (K/128)
  int ns;          // TMA ring stages
  int nd;          // dequantized-tile ring stages (2..4)
  uint32_t a_off, w_off, sz_off, bar_off;  // smem carve-up (bytes from the 1024-aligned base)
  const uint8_t* wt;
  const __half* scales;
  const __half* zeros;
  __half* Y;
  int64_t ldy;
  float* partial;  // [grid][2][NB][128]
  int* sem;        // [N/128]
  uint32_t magic;  // 0x64006400
  uint32_t tmem_cols;
};

constexpr int kTcDeqWarps = 16;                 // 4 per SM sub-partition
constexpr int kTcThreads = 64 + 32 * kTcDeqWarps;  // + TMA warp + MMA warp
constexpr uint32_t kDeqBytes = 128 * 128 * 2;   // one fp16 W^T tile, two 64-k swizzle blocks

// SWIZZLE_128B K-major UMMA shared-memory descriptor (SBO = 1024 B between 8-row atoms).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint32_t tc_idesc(int nb) {
  // kind::f16: D fp32 (bits 4-5 = 1), A = B = fp16, both K-major, N>>3 at 17, M>>4 at 24
  return (1u << 4) | ((uint32_t)(nb >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// Segment words of column c, k-quarter KQ (pairs [16*KQ, 16*KQ+16)) of a transformed tile
// in shared memory (32-bit shared address), at the positions assemble_pair<> reads.
template <int B, int KQ>
__device__ __forceinline__ void load_quarter_words(uint32_t tile, int c, uint32_t* words) {
#pragma unroll
  for (int s = 0; s < num_segs(B); ++s) {
    const int w = seg_width(B, s), base = seg_base(B, s);
    const uint32_t sp = tile + 2048 * base;
    const int j0 = w * KQ;                      // first word of this quarter
    const uint32_t a = sp + ((j0 >> 2) * 128 + c) * 16 + (j0 & 3) * 4;
    if (w == 1) {
      words[4 * base + j0] = lds32(a);
    } else if (w == 2) {
      const uint2 x = lds64(a);
      words[4 * base + j0] = x.x;
      words[4 * base + j0 + 1] = x.y;
    } else {
#pragma unroll
      for (int v = 0; v < w / 4; ++v) {
        const uint4 x = lds128(a + v * 128 * 16);
        words[4 * base + j0 + 4 * v + 0] = x.x;
        words[4 * base + j0 + 4 * v + 1] = x.y;
        words[4 * base + j0 + 4 * v + 2] = x.z;
        words[4 * base + j0 + 4 * v + 3] = x.w;
      }
    }
  }
}

// Dequantize pairs [16*KQ, 16*KQ+16) of row n into the 128B-swizzled K-major W^T tile:
// 4 chunks of 8 k, logical chunk (KQ&1)*4 + j of 64-k block KQ>>1.  row_sw is the shared
// address of (block KQ>>1, row n) XOR the row's swizzle (n&7)<<4.
template <class F, int KQ>
__device__ __forceinline__ void tc_dequant_quarter(uint32_t wtile, uint32_t ss, uint32_t zs, int n, bool has_zeros,
                                                   uint32_t magic, uint32_t row_sw) {
  constexpr int B = F::bits;
  uint32_t words[4 * B];
  load_quarter_words<B, KQ>(wtile, n, words);
  PairConsts pc;
  pc.magic = magic;
  const uint16_t sh = lds16(ss);
  const __half2 s2 = u32_as_h2((uint32_t)sh | ((uint32_t)sh << 16));
  float z = 0.f;
  if constexpr (F::kind == kUint) z = has_zeros ? __half2float(__ushort_as_half(lds16(zs))) : 0.f;
  if constexpr (F::kind == kInt) z = (float)(1 << (B - 1));
  make_pair_consts<F>(pc, z);
  uint32_t chunk[4];
  static_for<0, 16>([&](auto II) {
    constexpr int ii = decltype(II)::value;
    constexpr int i = KQ * 16 + ii;
    chunk[ii & 3] = h2_as_u32(__hmul2(pair_value<F, i>(words, pc), s2));
    if constexpr ((ii & 3) == 3) {
      constexpr uint32_t cl = (uint32_t)(((KQ & 1) * 4 + (ii >> 2)) << 4);  // logical chunk byte offset
      sts128(row_sw ^ cl, chunk[0], chunk[1], chunk[2], chunk[3]);
    }
  });
}

template <class F>
__global__ void __launch_bounds__(kTcThreads, 1) tc_kernel(const __grid_constant__ CUtensorMap tmapA, TcParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned, still shared
  const int NS = p.ns;
  const int NB = p.NB;
  constexpr uint32_t WB = tile_bytes(F::bits);
  const uint32_t a_stage = (uint32_t)NB * 256;  // two 64-k boxes of NB rows x 128 B
  uint8_t* deq = smem;                           // ND x 32 KB
  uint8_t* a_s = smem + p.a_off;
  uint8_t* w_s = smem + p.w_off;
  uint8_t* sz_s = smem + p.sz_off;               // per stage: scales [4][128] + zeros [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* full_tma = bars;
  uint64_t* empty_tma = bars + NS;
  const int ND = p.nd;
  uint64_t* full_deq = bars + 2 * NS;
  uint64_t* empty_deq = full_deq + 4;
  uint64_t* tmem_full = empty_deq + 4;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  int* flag = reinterpret_cast<int*>(tmem_base_slot + 4);

  const int KT = p.K / kBK;
  const int grid = gridDim.x;
  const int cta = blockIdx.x;
  const int u0 = (int)((int64_t)cta * p.units / grid);
  const int u1 = (int)((int64_t)(cta + 1) * p.units / grid);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int spt = p.G >= kBK ? 1 : kBK / p.G;
  const bool has_zeros = p.zeros != nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_tma[s], 1);
      mbar_init(&empty_tma[s], kTcDeqWarps + 1);
    }
    for (int d = 0; d < ND; ++d) {
      mbar_init(&full_deq[d], kTcDeqWarps);
      mbar_init(&empty_deq[d], 1);
    }
    for (int d = 0; d < 2; ++d) {
      mbar_init(&tmem_full[d], 1);
      mbar_init(&tmem_empty[d], kTcDeqWarps);
    }
    fence_mbar_init();
    prefetch_tmap(&tmapA);
  }
  if (warp == 1) {
    tmem_alloc(tmem_base_slot, p.tmem_cols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_slot;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_a = policy_evict_last();
      const uint32_t bytes = WB + a_stage + spt * kBN * 2 * (has_zeros ? 2 : 1);
      int s = 0, ph = 0, nt = u0 / KT, kt = u0 % KT;
      for (int u = u0; u < u1; ++u) {
        if (u - u0 >= NS) mbar_wait(&empty_tma[s], ph ^ 1);
        mbar_arrive_expect_tx(&full_tma[s], bytes);
        tma_bulk_g2s(w_s + s * WB, p.wt + (int64_t)u * WB, WB, &full_tma[s], pol_w);
        uint8_t* as = a_s + s * a_stage;
        tma_load_2d(as, &tmapA, kt * kBK, 0, &full_tma[s], pol_a);
        tma_load_2d(as + NB * 128, &tmapA, kt * kBK + 64, 0, &full_tma[s], pol_a);
        const int g0 = (int)((int64_t)kt * kBK / p.G);
        uint8_t* sz = sz_s + s * 2048;
        for (int r = 0; r < spt; ++r) {
          tma_bulk_g2s(sz + r * 256, p.scales + (int64_t)(g0 + r) * p.N + nt * kBN, 256, &full_tma[s], pol_w);
          if (has_zeros)
            tma_bulk_g2s(sz + 1024 + r * 256, p.zeros + (int64_t)(g0 + r) * p.N + nt * kBN, 256, &full_tma[s],
                         pol_w);
        }
        if (++kt == KT) { kt = 0; ++nt; }
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    const uint32_t idesc = tc_idesc(NB);
    int s = 0, ph = 0, d = 0, dph = 0, kt = u0 % KT, seg = 0;
    bool first = true;
    for (int u = u0; u < u1; ++u) {
      const int a = seg & 1;
      if (first) {
        if (seg >= 2) mbar_wait(&tmem_empty[a], ((seg >> 1) - 1) & 1);
        tc_fence_after();
      }
      mbar_wait(&full_deq[d], dph);
      mbar_wait(&full_tma[s], ph);
      tc_fence_after();
      if (elect_one()) {
        // descriptors advance 32 B per k-step inside a 64-k block (+2 in 16-B units); the W^T
        // tile's second block is 16 KB on (+1024), the activation tile's NB*128 B on
        const uint64_t ad0 = sw128_desc(smem_u32(deq + d * kDeqBytes));
        const uint64_t bd0 = sw128_desc(smem_u32(a_s + s * a_stage));
        const uint32_t dt = tmem + (uint32_t)(a * NB);
        const uint32_t bblk = (uint32_t)NB * 8;  // NB*128 B in 16-B units
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint64_t ad = ad0 + (uint64_t)((j >> 2) * 1024 + (j & 3) * 2);
          const uint64_t bd = bd0 + (uint64_t)((j >> 2) * bblk + (j & 3) * 2);
          tc_mma_f16_ss(dt, ad, bd, idesc, (first && j == 0) ? 0u : 1u);
        }
        tc_commit(&empty_deq[d]);
        tc_commit(&empty_tma[s]);
        if (kt == KT - 1 || u == u1 - 1) tc_commit(&tmem_full[a]);
      }
      __syncwarp();
      first = false;
      if (kt == KT - 1 || u == u1 - 1) {
        first = true;
        ++seg;
      }
      if (++kt == KT) kt = 0;
      if (++s == NS) { s = 0; ph ^= 1; }
      if (++d == ND) { d = 0; dph ^= 1; }
    }
  } else {
    // ------------------------------ dequant + epilogue ------------------------------
    const int dw = warp - 2;             // 0..15
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int kq = dw >> 2;              // k-quarter of the tile this warp dequantizes
    const int n = q * 32 + lane;         // row of W^T (column of the weight / Y)
    const uint32_t deq_u = smem_u32(deq);
    const uint32_t w_u = smem_u32(w_s);
    const uint32_t sz_u = smem_u32(sz_s);
    // this thread's swizzled row address in dequant buffer 0 (block kq>>1, row n)
    const uint32_t row_sw0 = (deq_u + (kq >> 1) * 16384 + n * 128) ^ ((uint32_t)(n & 7) << 4);
    const int lg = p.G == 32 ? 5 : 6;
    const int srow = (p.G >= kBK) ? 0 : ((32 * kq) >> lg);  // group row of this k-quarter in the slice
    int s = 0, ph = 0, d = 0, dph = 0, nt = u0 / KT, kt = u0 % KT, seg = 0;
    for (int u = u0; u < u1; ++u) {
      mbar_wait(&full_tma[s], ph);
      if (u - u0 >= ND) mbar_wait(&empty_deq[d], dph ^ 1);
      const uint32_t wtile = w_u + s * WB;
      const uint32_t ss = sz_u + s * 2048 + (srow * kBN + n) * 2;
      const uint32_t row_sw = row_sw0 + d * kDeqBytes;
      switch (kq) {
        case 0: tc_dequant_quarter<F, 0>(wtile, ss, ss + 1024, n, has_zeros, p.magic, row_sw); break;
        case 1: tc_dequant_quarter<F, 1>(wtile, ss, ss + 1024, n, has_zeros, p.magic, row_sw); break;
        case 2: tc_dequant_quarter<F, 2>(wtile, ss, ss + 1024, n, has_zeros, p.magic, row_sw); break;
        default: tc_dequant_quarter<F, 3>(wtile, ss, ss + 1024, n, has_zeros, p.magic, row_sw); break;
      }
      fence_proxy_async_smem();  // make the STS visible to the tensor core (async proxy)
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&full_deq[d]);
        mbar_arrive(&empty_tma[s]);
      }
      const bool seg_end = (kt == KT - 1) || (u == u1 - 1);
      const int cur_nt = nt;
      if (++kt == KT) { kt = 0; ++nt; }
      if (++s == NS) { s = 0; ph ^= 1; }
      if (++d == ND) { d = 0; dph ^= 1; }
      if (!seg_end) continue;

      // ---- epilogue of n-tile cur_nt (accumulator a) ----
      const int a = seg & 1;
      mbar_wait(&tmem_full[a], (seg >> 1) & 1);
      tc_fence_after();
      const int ua = cur_nt * KT, ub = ua + KT;
      const bool complete = (u0 <= ua) && (u1 >= ub);
      const int col0 = cur_nt * kBN + n;
      const int nt_first = u0 / KT;
      const int slot = (cur_nt == nt_first) ? 0 : 1;
      float* part = p.partial + ((int64_t)(cta * 2 + slot) * NB) * kBN;
      for (int cb = kq * 16; cb < NB; cb += 64) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * NB + cb), r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = cb + j;
          if (m < p.M) {
            const float v = __uint_as_float(r[j]);
            if (complete) p.Y[(int64_t)m * p.ldy + col0] = __float2half_rn(v);
            else __stcg(part + (int64_t)m * kBN + n, v);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[a]);
      if (!complete) {
        __threadfence();
        named_bar_sync(1, kTcDeqWarps * 32);
        if (threadIdx.x == 64) {
          const int lo = (int)((((int64_t)ua + 1) * grid - 1) / p.units);
          const int hi = (int)((((int64_t)ub) * grid - 1) / p.units);
          const int prev = atomicAdd(&p.sem[cur_nt], 1);
          flag[0] = (prev == hi - lo) ? 1 : 0;
          flag[1] = lo;
          flag[2] = hi;
        }
        named_bar_sync(1, kTcDeqWarps * 32);
        if (flag[0]) {
          __threadfence();
          const int lo = flag[1], hi = flag[2];
          for (int m = kq; m < p.M; m += 4) {
            float sum = 0.f;
            for (int qq = lo; qq <= hi; ++qq) {
              const int q_first = (int)((int64_t)qq * p.units / grid) / KT;
              const int qslot = (cur_nt == q_first) ? 0 : 1;
              sum += __ldcg(p.partial + ((int64_t)(qq * 2 + qslot) * NB + m) * kBN + n);
            }
            p.Y[(int64_t)m * p.ldy + col0] = __float2half_rn(sum);
          }
          if (threadIdx.x == 64) p.sem[cur_nt] = 0;
        }
        named_bar_sync(1, kTcDeqWarps * 32);
      }
      ++seg;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, p.tmem_cols);
}

// ---------------------------------------------------------------------------------------
template <class F>
tl_status launch_tc(const TcParams& p, const CUtensorMap* tmap, int grid, uint32_t smem_bytes, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(tc_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return fail(TL_ECUDA, "cudaFuncSetAttribute(tc smem)");
    configured = true;
  }
  tc_kernel<F><<<grid, kTcThreads, smem_bytes, st>>>(*tmap, p);
  return check_launch("tc_kernel");
}

}  // namespace tl
