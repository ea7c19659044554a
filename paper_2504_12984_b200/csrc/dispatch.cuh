// dispatch.cuh -- runtime weight format -> compile-time Fmt<kind, bits, exp>.
//
// The 37 kernel formats (reading R4): uint1..8, int1..8 and the 21
// float splits with 1 <= E <= 4, M = b-1-E >= 0.  (kind, bits) and E are all
// template parameters so every shift / mask in the unpack is an immediate
// (SURVEY H7).
#pragma once

#include <type_traits>

#include "common.cuh"

#define TL_FOR_EACH_FORMAT(X)                                                              \
  X(0, 1, 0) X(0, 2, 0) X(0, 3, 0) X(0, 4, 0) X(0, 5, 0) X(0, 6, 0) X(0, 7, 0) X(0, 8, 0)    \
  X(1, 1, 0) X(1, 2, 0) X(1, 3, 0) X(1, 4, 0) X(1, 5, 0) X(1, 6, 0) X(1, 7, 0) X(1, 8, 0)    \
  X(2, 3, 1) X(2, 3, 2)                                                                    \
  X(2, 4, 1) X(2, 4, 2) X(2, 4, 3)                                                         \
  X(2, 5, 1) X(2, 5, 2) X(2, 5, 3) X(2, 5, 4)                                              \
  X(2, 6, 1) X(2, 6, 2) X(2, 6, 3) X(2, 6, 4)                                              \
  X(2, 7, 1) X(2, 7, 2) X(2, 7, 3) X(2, 7, 4)                                              \
  X(2, 8, 1) X(2, 8, 2) X(2, 8, 3) X(2, 8, 4)

namespace tl {

__host__ __device__ constexpr int fmt_key(int kind, int bits, int exp) { return kind * 100 + bits * 10 + exp; }

// Calls f(Fmt<...>{}) for the runtime format; returns false if it is not a kernel format.
template <class Fn>
inline bool dispatch_format(int kind, int bits, int exp, Fn&& f) {
  switch (fmt_key(kind, bits, exp)) {
#define TL_CASE(K, B, E)         \
  case fmt_key(K, B, E):         \
    f(Fmt<K, B, E>{});           \
    return true;
    TL_FOR_EACH_FORMAT(TL_CASE)
#undef TL_CASE
    default:
      return false;
  }
}

}  // namespace tl
