// common.cuh -- shared definitions of the B200-native A16Wx library.
//
// Part of the product path (libtilus_b200.so).  Shares nothing with oracle/.
//
// Transformed weight layout, version 1
// ----------------------------------------------------------------------
// The paper re-lays the weight out "from i6[K, N] to u8[K / BK, N / BN,
// BK * BN * 6 / 8]" so that each thread's bytes are contiguous and load with
// wide vector instructions (the gcd rule of
// PAPER.md:416).  Here BK = BN = 128 and:
//
//  * tiles are stored n-tile major: tile (kt, nt) starts at byte
//    (nt * K/128 + kt) * 2048*b, so the K-stream of one 128-column block is one
//    contiguous region (TMA bulk copies / long coalesced streams);
//  * the b-bit code is split into power-of-two SEGMENTS (b = 8 | 4+2+1 | 4+2 |
//    4+1 | 4 | 2+1 | 2 | 1), so that no code straddles a 32-bit word; segment s
//    of width w holds code bits [base_s, base_s + w) and occupies 2048*w bytes of
//    the tile starting at byte 2048*base_s;
//  * inside a segment, column n's 128 k-values form w 16-byte vectors; vector v
//    of column n is at vector index v*128 + n (lanes = consecutive n = one
//    coalesced 512-byte warp access, the paper's local(n2).spatial(T).local(16));
//  * word j (0 <= j < 4w) of a column holds 16/w PAIRS: pair p (bit offset
//    o = p*w in each 16-bit half) holds k = j*(32/w) + 2p in the low half and
//    k + 1 in the high half.  A single LOP3 therefore turns a pair into two fp16
//    lanes ("PRMT / LOP3 ... within registers");
//  * int formats are stored offset-binary (code XOR 2^(b-1)), so the kernels
//    treat them as unsigned with the constant zero point 2^(b-1).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tl {

constexpr int kBK = 128;
constexpr int kBN = 128;
constexpr uint32_t kFormatVersion = 1;

enum Kind : int { kUint = 0, kInt = 1, kFloat = 2 };

// ---- segments ---------------------------------------------------------------
__host__ __device__ constexpr int num_segs(int b) {
  return b == 8 ? 1 : ((b >> 2) & 1) + ((b >> 1) & 1) + (b & 1);
}
__host__ __device__ constexpr int seg_width(int b, int s) {
  // widths in descending order: the set bits of b (8 alone)
  if (b == 8) return 8;
  int i = 0;
  for (int w = 4; w >= 1; w >>= 1) {
    if (b & w) {
      if (i == s) return w;
      ++i;
    }
  }
  return 0;
}
__host__ __device__ constexpr int seg_base(int b, int s) {
  int base = 0;
  for (int i = 0; i < s; ++i) base += seg_width(b, i);
  return base;
}
__host__ __device__ constexpr int tile_bytes(int b) { return 2048 * b; }

// Location of code bit `cb` of element (kl, nl) of a tile (kl, nl in [0,128)).
// Returns the byte offset within the tile and the bit within that byte.
__host__ __device__ inline void locate_bit(int b, int kl, int nl, int cb, int* byte_off, int* bit) {
  int s = 0;
  while (!(cb >= seg_base(b, s) && cb < seg_base(b, s) + seg_width(b, s))) ++s;
  const int w = seg_width(b, s);
  const int per_word = 32 / w;
  const int j = kl / per_word;
  const int rem = kl % per_word;
  const int p = rem >> 1, h = rem & 1;
  const int q = h * 16 + p * w + (cb - seg_base(b, s));
  const int v = j >> 2, r = j & 3;
  *byte_off = 2048 * seg_base(b, s) + (v * 128 + nl) * 16 + r * 4 + (q >> 3);
  *bit = q & 7;
}

// ---- format traits -------------------------------------------------------------
template <int KIND, int BITS, int EXP>
struct Fmt {
  static constexpr int kind = KIND;
  static constexpr int bits = BITS;
  static constexpr int exp = EXP;
  static constexpr int man = KIND == kFloat ? BITS - 1 - EXP : 0;
  static constexpr int nseg = num_segs(BITS);
  static constexpr int bias = KIND == kFloat ? (1 << (EXP - 1)) - 1 : 0;
  // words of one 128-k column run, per segment: 4*w
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

// Shift helper usable with a compile-time signed shift (right if d > 0).
template <int D>
__device__ __forceinline__ uint32_t shr_signed(uint32_t x) {
  if constexpr (D > 0) return x >> D;
  else if constexpr (D < 0) return x << (-D);
  else return x;
}

// ---- pair assembly (TC path and the dequant hook) --------------------------------------
// For pair i of a column run (k = 2i, 2i+1) build a 32-bit word holding, in each
// 16-bit half, the b-bit stored code placed at bit P of the half (all other bits 0),
// reading the segment words `sw` (sw[s][j], j < 4*w_s).
template <int B, int I, int S>
struct SegPos {
  static constexpr int w = seg_width(B, S);
  static constexpr int per_word = 32 / w;
  static constexpr int j = (2 * I) / per_word;
  static constexpr int o = (((2 * I) % per_word) >> 1) * w;
};

// Position chosen for the uint/int pair so that segment 0 needs no (or a shared) shift:
// the fp16 magic form needs P + b <= 10.
template <int B, int I>
struct PairP {
  static constexpr int o0 = SegPos<B, I, 0>::o;
  static constexpr int value = (o0 + B <= 10) ? o0 : ((o0 >= 8 && o0 - 8 + B <= 10) ? o0 - 8 : 0);
};

template <int B, int S, int I, int P>
__device__ __forceinline__ uint32_t seg_part(const uint32_t* words_s) {
  using SP = SegPos<B, I, S>;
  constexpr int t = P + seg_base(B, S);
  constexpr uint32_t m = ((1u << SP::w) - 1u) << t;
  constexpr uint32_t mask = m | (m << 16);
  return shr_signed<SP::o - t>(words_s[SP::j]) & mask;
}

// words: pointer to a flat array holding the segments back to back
// (segment s starts at word 4*seg_base(B, s)).
template <int B, int I, int P>
__device__ __forceinline__ uint32_t assemble_pair(const uint32_t* words) {
  uint32_t x = seg_part<B, 0, I, P>(words);
  if constexpr (num_segs(B) > 1) x |= seg_part<B, 1, I, P>(words + 4 * seg_base(B, 1));
  if constexpr (num_segs(B) > 2) x |= seg_part<B, 2, I, P>(words + 4 * seg_base(B, 2));
  return x;
}

// fp16x2 pair of EXACT unscaled values for pair I:
//   uint/int: (u - z) with u the stored code (z = zero point, 2^(b-1) for int)
//   float   : value(code)
// zc: per-group constants prepared by pair_consts().
struct PairConsts {
  // uint/int: hz[P] = -(2^(10-P) + z) as fp16x2 for every P in [0, 10]
  // float   : unused
  __half2 neg_off[11];
  // 0x64006400 (fp16 1024.0 in both halves), passed in from a kernel argument so the
  // compiler keeps it in a register and fuses AND-mask + OR-magic into ONE LOP3
  uint32_t magic;
};

// Is P used by any pair of a b-bit column run?  (Only those constants are built.)
template <int B>
__host__ __device__ constexpr bool pair_p_used(int P) {
  for (int i = 0; i < 64; ++i) {
    const int w = seg_width(B, 0), per_word = 32 / w;
    const int o0 = (((2 * i) % per_word) >> 1) * w;
    const int v = (o0 + B <= 10) ? o0 : ((o0 >= 8 && o0 - 8 + B <= 10) ? o0 - 8 : 0);
    if (v == P) return true;
  }
  return false;
}

template <class F>
__device__ __forceinline__ void make_pair_consts(PairConsts& c, float z) {
  if constexpr (F::kind != kFloat) {
#pragma unroll
    for (int P = 0; P <= 10; ++P) {
      if (pair_p_used<F::bits>(P)) {
        const __half h = __float2half_rn(-(float)(1 << (10 - P)) - z);
        c.neg_off[P] = __halves2half2(h, h);
      }
    }
  }
}

template <class F, int I>
__device__ __forceinline__ __half2 pair_value(const uint32_t* words, const PairConsts& c) {
  if constexpr (F::kind != kFloat) {
    constexpr int P = PairP<F::bits, I>::value;
    const uint32_t x = assemble_pair<F::bits, I, P>(words) | c.magic;  // 1024 + 2^P u
    constexpr uint32_t sc = (uint32_t)(15 - P) << 10;                   // fp16 bits of 2^-P
    return __hfma2(u32_as_h2(x), u32_as_h2(sc | (sc << 16)), c.neg_off[P]);  // u - z, exact
  } else {
    constexpr int P = 10 - F::man;  // magnitude lands on the fp16 exponent/mantissa fields
    uint32_t x = assemble_pair<F::bits, I, P>(words);
    constexpr uint32_t sb = 1u << (10 + F::exp);  // where the code's sign bit landed
    const uint32_t y = x & (sb | (sb << 16));
    x = x + y * ((1u << (5 - F::exp)) - 1u);       // move the sign bit to bit 15 of each half
    constexpr uint32_t e = (uint32_t)(30 - F::bias) << 10;              // fp16 bits of 2^(15-bias)
    return __hmul2(u32_as_h2(x), u32_as_h2(e | (e << 16)));               // value(code), exact
  }
}

// Load the segment words of column c, k-half KH (pairs [32*KH, 32*KH+32)) of one transformed
// tile held in shared memory, into words[] at the positions assemble_pair<> reads.
template <int B, int KH>
__device__ __forceinline__ void load_half_words(const uint8_t* tile, int c, uint32_t* words) {
#pragma unroll
  for (int s = 0; s < num_segs(B); ++s) {
    const int w = seg_width(B, s), base = seg_base(B, s);
    const uint8_t* sp = tile + 2048 * base;
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
}

// Raw pair bits for the tensor-core decode path and the CUDA-core GEMV (no magic number):
//   ints:   the b-bit code u placed at bit P of each 16-bit half IS the fp16 u * 2^(P-24)
//           (subnormal, or a small normal) -- exact; the activations are pre-scaled by 2^-P
//   floats: the code's E+M field on the fp16 exponent/mantissa fields and the sign moved to
//           bit 15: the fp16 value(code) * 2^(bias-15), exact
template <int B, int I>
struct SubP {
  static constexpr int value = PairP<B, I>::value;
};

template <class F, int I>
__device__ __forceinline__ uint32_t raw_pair_bits(const uint32_t* words) {
  if constexpr (F::kind != kFloat) {
    return assemble_pair<F::bits, I, SubP<F::bits, I>::value>(words);
  } else {
    constexpr int P = 10 - F::man;
    uint32_t x = assemble_pair<F::bits, I, P>(words);
    constexpr uint32_t sb = 1u << (10 + F::exp);
    const uint32_t y = x & (sb | (sb << 16));
    return x + y * ((1u << (5 - F::exp)) - 1u);
  }
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
