"""O5 -- group-wise dequantization.  TEST INFRASTRUCTURE ONLY.

The paper names the step ("casting and de-quantizing low-precision weights to
high-precision (e.g., float16)") but gives no formula.  SPEC: out[k] =
decode(w[k]) * scale[k / group_size].  The north star adds zero
points for unsigned formats.

Readings:
  R6  uint: w = (q - z[g,n]) * s[g,n]; int and float: w = value(q) * s[g,n].
  R7  scales and zeros are [K/G, N] row-major fp16; zeros are integer-valued.
  R8  g = k // G, G divides K.
  R13 sign of zero follows IEEE: value -0.0 times s gives -0.0*s; (q-z)=0 gives +0*s.

The result is returned in float64.  It is exact: |value| has <= 8 significant
bits (R4), s has 11, so every product is exact in fp64 and -- as the test
suite checks exhaustively -- also exactly representable in fp32.
"""

from __future__ import annotations

import numpy as np

from .formats import WType, code_values


def dequant(wt: WType, codes: np.ndarray, scales: np.ndarray, zeros: np.ndarray | None,
            group: int) -> np.ndarray:
    """codes [K,N] uint8, scales [K/G,N] fp16, zeros [K/G,N] fp16 or None -> w [K,N] float64."""
    codes = np.asarray(codes)
    K, N = codes.shape
    if K % group:
        raise ValueError("group size must divide K (R8)")
    if scales.shape != (K // group, N):
        raise ValueError("scales must be [K/G, N] (R7)")
    if zeros is not None and wt.kind != "u":
        raise ValueError("zero points are for unsigned formats only (R6)")
    vals = code_values(wt)[codes.astype(np.int64)]            # value(q), exact
    g = np.arange(K) // group                                   # group of each row k
    s = scales.astype(np.float64)[g, :]                         # s[g(k), n]
    if zeros is not None:
        z = zeros.astype(np.float64)[g, :]
        return (vals - z) * s
    return vals * s
