"""O9 -- encoder (value -> code), used only to build test data.  TEST INFRASTRUCTURE ONLY.

SPEC encode: inverse of decode for representable values;
unrepresentable values go to the nearest representable value,
round-to-nearest-even for floats, saturation for integers.

Written as a brute-force nearest search over the value table (O2), so it
cannot disagree with ``formats.code_value``.  Ties go to the even code (the
code whose least-significant bit is 0), which is round-half-to-even for every
integer format and for every float format with M >= 1.
"""

from __future__ import annotations

import numpy as np

from .formats import WType, code_values


def encode(wt: WType, v: np.ndarray) -> np.ndarray:
    """Nearest code for every value in ``v`` (float array) -> uint8 codes."""
    v = np.asarray(v, dtype=np.float64)
    table = code_values(wt)
    codes = np.arange(table.size)
    # prefer +0 over -0 for zero inputs and never pick a code of the wrong sign
    # when an equally near one of the right sign exists: sort key below.
    dist = np.abs(v.reshape(-1, 1) - table.reshape(1, -1))
    best = dist.min(axis=1, keepdims=True)
    cand = dist == best
    # among the candidates: prefer the same sign as v (matters only for +-0), then the even code
    same_sign = (np.signbit(table).reshape(1, -1) == np.signbit(v).reshape(-1, 1))
    key = cand * (4 + 2 * same_sign + (codes % 2 == 0).reshape(1, -1))
    return key.argmax(axis=1).astype(np.uint8).reshape(v.shape)
