// common.cuh -- shared definitions of the B200-native A16Wx library.
//
// Part of the product path (libtilus_b200.so).  Shares nothing with oracle/.
//
// Transformed weight layout, version 2  (DESIGN.md §5 "Transformed layout")
// ----------------------------------------------------------------------
// The paper re-lays the weight out "from i6[K, N] to u8[K / BK, N / BN, BK * BN * 6 / 8]" so that
// each thread's bytes are contiguous and load with wide vector instructions (PAPER.md:187,
// PAPER.md:409-416, the gcd rule of PAPER.md:416), and casts "within registers" with PRMT / LOP3
// (PAPER.md:419).  Here BK = BN = 128, and:
//
//  * tiles are stored n-tile major: tile (kt, nt) starts at byte (nt * K/128 + kt) * 2048*b, so
//    the K-stream of one 128-column block is one contiguous region (one cp.async.bulk per tile);
//  * column n of a tile owns 4b 32-bit words (128 codes x b bits), stored as b 16-byte vectors;
//    vector v of column n sits at byte (v*128 + n)*16 (a warp's 32 lanes read 512 contiguous
//    bytes -- the paper's local(n2).spatial(T).local(16));
//  * the words serve 64 PAIRS of codes (k = 2i, 2i+1 in the low / high 16-bit half of the output
//    word that feeds one fp16x2 operand).  The two halves of a word are two independent 16-bit
//    streams (even k, odd k) that always receive the same shift and mask, so each pair is
//    extracted by a few LOP3s on whole words;
//  * pairs 0..31 (k < 64) live in BLOCK 0 = words {4v, 4v+1}, pairs 32..63 in block 1 = words
//    {4v+2, 4v+3} (a k-half is b 8-byte loads);
//  * inside a block (2b words), make_plan() assigns every code a field that is extracted by as few
//    operations as possible (the B200 unpack is integer-ALU bound):
//      ints: the b-bit code lands at bits [P, P+b) of each half, P + b <= 10, so
//            (x & mask) | 0x6400 is the fp16 1024 + u*2^P and ONE HFMA2 (x*2^-P - (2^(10-P) + z))
//            gives u - z exactly.  Per word: codes at shift 0 while they end below bit 10, the
//            next ones after one shared right shift, the leftover bits of all words pooled into
//            "spare" codes assembled from several (word, shift) terms;
//      floats: sign | exponent | mantissa land on the fp16 sign bit 15 and the exponent/mantissa
//            fields [10-M, 10+E): value(code) * 2^(bias-15), exact.  Greedy over shifts
//            0, <<1..<<15, >>1..>>15, then spare codes;
//  * int formats are stored offset-binary (code XOR 2^(b-1)): every integer format is "unsigned
//    with a zero point" (the constant 2^(b-1)).
// Size = K*N*b/8 bytes exactly (no padding, as PAPER.md:187).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace tl {

// compile-time loop
template <int I, int N, class Fn>
__host__ __device__ __forceinline__ void static_for(Fn&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

constexpr int kBK = 128;
constexpr int kBN = 128;
constexpr uint32_t kFormatVersion = 2;

enum Kind : int { kUint = 0, kInt = 1, kFloat = 2 };

__host__ __device__ constexpr int tile_bytes(int b) { return 2048 * b; }

// ---- layout v2 plan ------------------------------------------------------------------------
// A TERM contributes (word >> shift) & (mask | mask << 16) (shift < 0: << -shift) to a pair; a
// pair is the OR of its terms (and of the fp16 magic 0x6400 for ints).
struct Term {
  int8_t word;    // block-local word 0..2b-1
  int8_t shift;   // > 0: right shift, < 0: left shift
  uint16_t mask;  // destination bits within each 16-bit half
};
struct PairPlan {
  int8_t nt;  // number of terms (1..8)
  int8_t P;   // ints: the field starts at bit P (P + b <= 10); floats: 0
  Term t[8];
};
struct BlockPlan {
  PairPlan pr[32];
};

// destination bit of code bit cb
__host__ __device__ constexpr int fin_pos(int kind, int b, int E, int P, int cb) {
  return kind == 2 ? (cb < b - 1 ? 10 - (b - 1 - E) + cb : 15) : P + cb;
}

__host__ __device__ constexpr BlockPlan make_plan(int kind, int b, int E) {
  BlockPlan pl{};
  int np = 0;
  int8_t spw[256] = {}, spq[256] = {};
  int ns = 0;
  const int nw = 2 * b;
  for (int j = 0; j < nw; ++j) {
    uint32_t used = 0;
    if (kind != 2) {
      int s = 0, d = 0;
      while (s + b <= 16 && np < 32) {
        int P = 0, sh = 0;
        if (d == 0 && s + b <= 10) {
          P = s;
        } else {
          if (d == 0) d = s;
          P = s - d;
          if (P + b > 10) {
            d = s;
            P = 0;
          }
          sh = d;
        }
        used |= ((1u << b) - 1u) << s;
        pl.pr[np].nt = 1;
        pl.pr[np].P = (int8_t)P;
        pl.pr[np].t[0] = Term{(int8_t)j, (int8_t)sh, (uint16_t)(((1u << b) - 1u) << P)};
        ++np;
        s += b;
      }
    } else {
      bool placed = true;
      while (placed && np < 32) {
        placed = false;
        for (int k = 0; k < 31 && !placed; ++k) {
          const int sh = k == 0 ? 0 : (k <= 15 ? -k : k - 15);
          uint32_t src = 0;
          uint32_t m = 0;
          bool ok = true;
          for (int cb = 0; cb < b; ++cb) {
            const int f = fin_pos(kind, b, E, 0, cb);
            const int q = f + sh;
            if (q < 0 || q > 15 || (((used | src) >> q) & 1u)) {
              ok = false;
              break;
            }
            src |= 1u << q;
            m |= 1u << f;
          }
          if (ok) {
            used |= src;
            pl.pr[np].nt = 1;
            pl.pr[np].P = 0;
            pl.pr[np].t[0] = Term{(int8_t)j, (int8_t)sh, (uint16_t)m};
            ++np;
            placed = true;
          }
        }
      }
    }
    for (int q = 0; q < 16; ++q)
      if (!((used >> q) & 1u)) {
        spw[ns] = (int8_t)j;
        spq[ns] = (int8_t)q;
        ++ns;
      }
  }
  // spare codes: the pooled leftover bits, b at a time, in word order; runs with a common
  // (word, shift) share one term
  int idx = 0;
  while (np < 32 && idx + b <= ns) {
    PairPlan& pp = pl.pr[np];
    pp.nt = 0;
    pp.P = 0;
    for (int cb = 0; cb < b; ++cb, ++idx) {
      const int f = fin_pos(kind, b, E, 0, cb);
      const int sh = spq[idx] - f;
      int t = 0;
      while (t < pp.nt && !(pp.t[t].word == spw[idx] && pp.t[t].shift == sh)) ++t;
      if (t == pp.nt) {
        pp.t[t] = Term{spw[idx], (int8_t)sh, 0};
        ++pp.nt;
      }
      pp.t[t].mask = (uint16_t)(pp.t[t].mask | (1u << f));
    }
    ++np;
  }
  return pl;
}

template <int KIND, int B, int E>
inline constexpr BlockPlan kPlan = make_plan(KIND, B, E);

// is P the field position of some pair of the format's plan (ints)?
template <class F>
__host__ __device__ constexpr bool plan_has_p(int P) {
  for (int i = 0; i < 32; ++i)
    if (kPlan<F::kind, F::bits, F::exp>.pr[i].P == P) return true;
  return false;
}

// tile word (0..4b-1, vector-major: word 4v + r is lane r of 16-byte vector v) of block-local
// word j of block h
__host__ __device__ constexpr int tile_word(int h, int j) { return (j >> 1) * 4 + 2 * h + (j & 1); }

// ---- format traits -------------------------------------------------------------
template <int KIND, int BITS, int EXP>
struct Fmt {
  static constexpr int kind = KIND;
  static constexpr int bits = BITS;
  static constexpr int exp = EXP;
  static constexpr int man = KIND == kFloat ? BITS - 1 - EXP : 0;
  static constexpr int bias = KIND == kFloat ? (1 << (EXP - 1)) - 1 : 0;
  // words of one 128-k column run, per segment: 4*w
};

// ---- activation type (tl_atype): A, scales, zero points and Y share it -----------------------
// fp16 (TL_ACT_F16) or bf16 (TL_ACT_BF16).  The dequantized weight is
// built exactly in fp16 (u - z, value(code)) and converted where the MMA or the GEMM needs bf16.
template <bool BF>
struct Act {
  // instruction-descriptor a_format / b_format bits of tcgen05.mma.kind::f16 (0 = F16, 1 = BF16)
  static constexpr uint32_t idesc_ab = BF ? ((1u << 7) | (1u << 10)) : 0u;
  __device__ static __forceinline__ float to_float(uint32_t bits16) {
    if constexpr (BF) return __uint_as_float(bits16 << 16);
    else return __half2float(__ushort_as_half((unsigned short)bits16));
  }
  __device__ static __forceinline__ unsigned short from_float(float v) {
    if constexpr (BF) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
    else return __half_as_ushort(__float2half_rn(v));
  }
  // an exact fp16x2 pair -> the same two values in this type (exact: |value| <= 2^16, <= 8 bits)
  __device__ static __forceinline__ uint32_t from_h2(uint32_t h) {
    if constexpr (BF) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h));
      const __nv_bfloat162 b = __floats2bfloat162_rn(f.x, f.y);
      return *reinterpret_cast<const uint32_t*>(&b);
    } else {
      return h;
    }
  }
  // fp16 bits of -z for a zero point given in this type (integer-valued, |z| <= 255: exact)
  __device__ static __forceinline__ uint32_t neg_zero_h(uint32_t bits16) {
    if constexpr (BF) return (uint32_t)__half_as_ushort(__float2half_rn(-to_float(bits16)));
    else return bits16 ^ 0x8000u;
  }
};

// ---- PTX helpers ------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u32_as_h2(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

// Shift helper usable with a compile-time signed shift (right if D > 0).
template <int D>
__device__ __forceinline__ uint32_t shr_signed(uint32_t x) {
  if constexpr (D > 0) return x >> D;
  else if constexpr (D < 0) return x << (-D);
  else return x;
}

// Pair I (0..31) of block H of a column: OR of its plan terms over the block-local words
// bw[j] = tile words[tile_word(H, j)], plus `base` (0x64006400 for the int magic form, 0 for raw
// fields).  With one term this is a single LOP3 (the shifts are shared by the pairs of a word).
template <class F, int I>
__device__ __forceinline__ uint32_t extract_pair(const uint32_t* bw, uint32_t base) {
  constexpr PairPlan pp = kPlan<F::kind, F::bits, F::exp>.pr[I];
  uint32_t x = base;
  static_for<0, pp.nt>([&](auto TT) {
    constexpr Term t = pp.t[decltype(TT)::value];
    constexpr uint32_t m = (uint32_t)t.mask | ((uint32_t)t.mask << 16);
    x |= shr_signed<t.shift>(bw[t.word]) & m;
  });
  return x;
}

// the fp16 constant 2^-P (both halves) for the int magic form
template <int P>
__device__ __forceinline__ uint32_t h2_pow2_neg() {
  constexpr uint32_t e = (uint32_t)(15 - P) << 10;
  return e | (e << 16);
}

// Block H's 2b words of column c from a transformed tile in shared memory (b 8-byte loads).
template <int B, int H>
__device__ __forceinline__ void load_block_words(const uint8_t* tile, int c, uint32_t* bw) {
#pragma unroll
  for (int v = 0; v < B; ++v) {
    const uint2 x = *reinterpret_cast<const uint2*>(tile + (v * 128 + c) * 16 + H * 8);
    bw[2 * v] = x.x;
    bw[2 * v + 1] = x.y;
  }
}

// ---- scale / zero rows of a weight stage (CUDA-core decode kernel gv1) ---------------------
// The [K/G, N] scale (and zero-point) array is viewed as a 3-D tensor {128 columns, K/G rows,
// N/128 n-tiles} (strides N*2 and 256 bytes); one box of {128, R, 1} brings the rows of up to R
// consecutive k-tiles of ONE n-tile.  A stage of R consecutive units spans at most two n-tiles
// (segment 0: the first tile's n-tile, segment 1: the next), so its side area holds two regions
// of R rows per array: [scales seg0 | scales seg1 | zeros seg0 | zeros seg1], 256 B per row.
__host__ __device__ constexpr uint32_t side_bytes(int R) { return (uint32_t)R * 4u * 256u; }

// byte offset, within the side area, of the scale row of a tile at k-tile kt of n-tile nt in a
// stage whose first unit is (nt0, kt0); add R*512 for its zero row
__device__ __forceinline__ uint32_t side_row_off(int R, int tpg, int nt, int kt, int nt0, int kt0) {
  const int seg = nt != nt0;
  const int first = seg ? 0 : kt0;
  return (uint32_t)(seg * R + kt / tpg - first / tpg) * 256u;
}

// Deterministic stream-K reduction (reading R12) of one output element of n-tile nt: the partial
// tiles of CTAs lo..hi summed in CTA order.  CTA q keeps two partial slots (0: its first n-tile,
// 1: its last); every q > lo starts inside nt (slot 0), only q == lo may have started earlier
// (lo_slot).  The loads are independent and issued eight at a time; the sum order is fixed.
__device__ __forceinline__ float streamk_sum(const float* partial, int lo, int hi, int lo_slot, int64_t slot_stride,
                                             int64_t off) {
  float sum = 0.f;
  for (int q0 = lo; q0 <= hi; q0 += 8) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = q0 + j;
      v[j] = q <= hi ? __ldcg(partial + (int64_t)(q * 2 + (q == lo ? lo_slot : 0)) * slot_stride + off) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (q0 + j <= hi) sum += v[j];
  }
  return sum;
}

}  // namespace tl
