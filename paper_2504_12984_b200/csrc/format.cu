// format.cu -- the one-time weight preparation kernels (rows a1 of SURVEY §8):
//   tl_pack / tl_unpack           compact LSB-first bitstream
//   tl_transform_weights          the "Change Layout" step
//   tl_untransform_weights        its exact inverse (test hook)
//   tl_dequant                    exact fp32 dequant of the TRANSFORMED weight through
//                                 the same pair unpack the tensor-core path uses (test hook)
// These run once per weight (the paper: "a pre-processing step before launching the
// kernel"), so they are simple bit-gather kernels, not tuned.
#include <cstring>

#include "api_util.cuh"

namespace tl {

// ---------------------------------------------------------------------------------
// pack: thread per output byte; bit t of byte j is stream bit 8j+t = bit (8j+t)%b of
// element (8j+t)/b (reading R1: LSB-first; R2: row-major [K,N]).
__global__ void pack_kernel(const uint8_t* __restrict__ codes, uint8_t* __restrict__ out, int64_t count, int bits,
                            int64_t nbytes) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nbytes; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int64_t pos = j * 8 + t;
      const int64_t e = pos / bits;
      if (e < count) byte |= ((uint32_t)(codes[e] >> (pos % bits)) & 1u) << t;
    }
    out[j] = (uint8_t)byte;
  }
}

__global__ void unpack_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ codes, int64_t count, int bits) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (int t = 0; t < bits; ++t) {
      const int64_t pos = e * bits + t;
      c |= ((uint32_t)(in[pos >> 3] >> (pos & 7)) & 1u) << t;
    }
    codes[e] = (uint8_t)c;
  }
}

// ---------------------------------------------------------------------------------
// Layout v2 tables (common.cuh make_plan), built on the host from the same plan the kernels
// unpack with, passed by value:
//   inv[j*16 + q] = 8*i + cb : bit q of each half of block-local word j holds code bit cb of pair i
//   fwd[8*i + cb] = 16*j + q : the inverse
struct LayoutTables {
  uint8_t inv[256];
  uint8_t fwd[256];
};

static LayoutTables layout_tables(tl_wtype w) {
  LayoutTables t{};
  const int b = w.bits, E = w.kind == 2 ? w.exp_bits : 0, M = b - 1 - E;
  const BlockPlan pl = make_plan(w.kind, b, E);
  for (int i = 0; i < 32; ++i)
    for (int k = 0; k < pl.pr[i].nt; ++k) {
      const Term& tm = pl.pr[i].t[k];
      for (int fb = 0; fb < 16; ++fb)
        if ((tm.mask >> fb) & 1) {
          const int cb = w.kind == 2 ? (fb == 15 ? b - 1 : fb - (10 - M)) : fb - pl.pr[i].P;
          const int q = fb + tm.shift;
          t.inv[tm.word * 16 + q] = (uint8_t)(8 * i + cb);
          t.fwd[8 * i + cb] = (uint8_t)(16 * tm.word + q);
        }
    }
  return t;
}

// transform: thread per output 32-bit word.  Word r of 16-byte vector v of column nl of a tile
// is block h = r/2, block-local word j = 2v + (r&1); its bit 16*hh + q holds code bit cb of
// pair i (inv table), i.e. of element k = 2*(32h + i) + hh.
__global__ void transform_kernel(const uint8_t* __restrict__ bs, uint32_t* __restrict__ out, int64_t K, int64_t N,
                                 int bits, uint32_t flip_top, int64_t nwords, LayoutTables lt) {
  const int64_t KT = K / kBK;
  const int words_per_tile = 512 * bits;
  for (int64_t wi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; wi < nwords; wi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = wi / words_per_tile;
    const int wt = (int)(wi % words_per_tile);
    const int64_t nt = tile / KT, kt = tile % KT;
    const int vi = wt >> 2, r = wt & 3;
    const int v = vi >> 7, nl = vi & 127;
    const int h = r >> 1, j = 2 * v + (r & 1);
    uint32_t word = 0;
    for (int q = 0; q < 32; ++q) {
      const int hh = q >> 4;
      const int e = lt.inv[j * 16 + (q & 15)];
      const int i = e >> 3, cbit = e & 7;
      const int kl = 2 * (32 * h + i) + hh;
      const int64_t k = kt * kBK + kl, n = nt * kBN + nl;
      const int64_t pos = (k * N + n) * bits + cbit;
      uint32_t bit = (bs[pos >> 3] >> (pos & 7)) & 1u;
      if (cbit == bits - 1) bit ^= flip_top;  // int: offset binary
      word |= bit << q;
    }
    out[wi] = word;
  }
}

// untransform: thread per output byte of the bitstream.
__global__ void untransform_kernel(const uint8_t* __restrict__ wt, uint8_t* __restrict__ bs, int64_t K, int64_t N,
                                   int bits, uint32_t flip_top, int64_t nbytes, LayoutTables lt) {
  const int64_t KT = K / kBK;
  const int64_t total_bits = K * N * bits;
  for (int64_t jb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; jb < nbytes; jb += (int64_t)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
    for (int t = 0; t < 8; ++t) {
      const int64_t pos = jb * 8 + t;
      if (pos >= total_bits) break;
      const int64_t e = pos / bits;
      const int cbit = (int)(pos % bits);
      const int64_t k = e / N, n = e % N;
      const int64_t kt = k / kBK, nt = n / kBN;
      const int kl = (int)(k % kBK), nl = (int)(n % kBN);
      const int pair = kl >> 1, hh = kl & 1, h = pair >> 5, i = pair & 31;
      const int f = lt.fwd[8 * i + cbit];
      const int j = f >> 4, q = (f & 15) + 16 * hh;
      const int off = ((j >> 1) * 128 + nl) * 16 + 4 * (2 * h + (j & 1)) + (q >> 3);
      const int64_t tile = nt * KT + kt;
      uint32_t v = (wt[tile * (int64_t)tile_bytes(bits) + off] >> (q & 7)) & 1u;
      if (cbit == bits - 1) v ^= flip_top;
      byte |= v << t;
    }
    bs[jb] = (uint8_t)byte;
  }
}

template <class F>
void launch_dequant(const uint8_t* wt, const __half* scales, const __half* zeros, float* out, int64_t K, int64_t N,
                    int G, unsigned tiles, cudaStream_t st);

}  // namespace tl

using namespace tl;

static int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (int)g;
}

extern "C" {

size_t tl_packed_bytes(tl_wtype w, int64_t K, int64_t N) {
  if (K < 0 || N < 0 || w.bits < 1 || w.bits > 8) return 0;
  return (size_t)((K * N * (int64_t)w.bits + 7) / 8);
}

size_t tl_transformed_bytes(tl_wtype w, int64_t K, int64_t N) {
  if (!wtype_ok(w) || K <= 0 || N <= 0 || K % kBK || N % kBN) return 0;
  return (size_t)(K * N * (int64_t)w.bits / 8);
}

uint32_t tl_format_version(void) { return kFormatVersion; }

tl_status tl_pack(tl_wtype w, int64_t K, int64_t N, const uint8_t* codes, uint8_t* bitstream, void* stream) {
  if (w.bits < 1 || w.bits > 8) return fail(TL_EINVAL_DTYPE, "bits must be 1..8");
  if (K < 0 || N < 0) return fail(TL_EINVAL_SHAPE, "negative shape");
  if (K * N == 0) return TL_OK;
  if (!codes || !bitstream) return fail(TL_ENULL, "tl_pack: NULL pointer");
  const int64_t nb = (int64_t)tl_packed_bytes(w, K, N);
  pack_kernel<<<grid_for(nb, 256), 256, 0, as_stream(stream)>>>(codes, bitstream, K * N, w.bits, nb);
  return check_launch("pack_kernel");
}

tl_status tl_unpack(tl_wtype w, int64_t K, int64_t N, const uint8_t* bitstream, uint8_t* codes, void* stream) {
  if (w.bits < 1 || w.bits > 8) return fail(TL_EINVAL_DTYPE, "bits must be 1..8");
  if (K < 0 || N < 0) return fail(TL_EINVAL_SHAPE, "negative shape");
  if (K * N == 0) return TL_OK;
  if (!codes || !bitstream) return fail(TL_ENULL, "tl_unpack: NULL pointer");
  unpack_kernel<<<grid_for(K * N, 256), 256, 0, as_stream(stream)>>>(bitstream, codes, K * N, w.bits);
  return check_launch("unpack_kernel");
}

tl_status tl_transform_weights(tl_wtype w, int64_t K, int64_t N, const uint8_t* bitstream, void* w_t, void* stream) {
  tl_status st;
  if ((st = check_wtype(w)) != TL_OK) return st;
  if ((st = check_kn(K, N)) != TL_OK) return st;
  if (!bitstream || !w_t) return fail(TL_ENULL, "tl_transform_weights: NULL pointer");
  if (!aligned16(w_t)) return fail(TL_EALIGN, "w_t must be 16-byte aligned");
  const int64_t nwords = K * N * w.bits / 32;
  transform_kernel<<<grid_for(nwords, 256), 256, 0, as_stream(stream)>>>(
      bitstream, reinterpret_cast<uint32_t*>(w_t), K, N, w.bits, w.kind == 1 ? 1u : 0u, nwords, layout_tables(w));
  return check_launch("transform_kernel");
}

tl_status tl_untransform_weights(tl_wtype w, int64_t K, int64_t N, const void* w_t, uint8_t* bitstream,
                                 void* stream) {
  tl_status st;
  if ((st = check_wtype(w)) != TL_OK) return st;
  if ((st = check_kn(K, N)) != TL_OK) return st;
  if (!bitstream || !w_t) return fail(TL_ENULL, "tl_untransform_weights: NULL pointer");
  const int64_t nb = (int64_t)tl_packed_bytes(w, K, N);
  untransform_kernel<<<grid_for(nb, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint8_t*>(w_t), bitstream, K, N, w.bits, w.kind == 1 ? 1u : 0u, nb, layout_tables(w));
  return check_launch("untransform_kernel");
}

tl_status tl_dequant(tl_wtype w, int64_t K, int64_t N, int32_t group, const void* w_t, const void* scales,
                     const void* zeros, float* out, void* stream) {
  tl_status st;
  if ((st = check_wtype(w)) != TL_OK) return st;
  if ((st = check_kn(K, N)) != TL_OK) return st;
  if ((st = check_group(K, group)) != TL_OK) return st;
  if (!w_t || !scales || !out) return fail(TL_ENULL, "tl_dequant: NULL pointer");
  if (zeros && w.kind != 0) return fail(TL_EZEROS, "zero points are for uint formats only");
  const int64_t tiles = (K / kBK) * (N / kBN);
  if (tiles > (1ll << 31) - 1) return fail(TL_EINVAL_SHAPE, "too many tiles");
  dispatch_format(w.kind, w.bits, w.kind == 2 ? w.exp_bits : 0, [&](auto f) {
    using F = decltype(f);
    launch_dequant<F>(reinterpret_cast<const uint8_t*>(w_t), reinterpret_cast<const __half*>(scales),
                      reinterpret_cast<const __half*>(zeros), out, K, N, group, (unsigned)tiles, as_stream(stream));
  });
  return check_launch("dequant_kernel");
}

}  // extern "C"
