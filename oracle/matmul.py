"""O6/O7 -- the matmul C = A x B and the tolerance comparator.  TEST INFRASTRUCTURE ONLY.

Paper: "Matrix multiplication is defined as C_{M,N} = A_{M,K} x B_{K,N}, where A
and B are float16 and int6"; "the accumulation tensor is cast from f32
to f16".  The method reaches (up to rounding order) the plain
definition, so the oracle is that definition in fp64: Y64[m,n] = sum_k
A[m,k] * w[k,n] with w = dequant(...) (O5).  Every product is exact in fp64
(11 + <=19 significant bits); only the sum rounds (|error| <= K * 2^-53 * sum|terms|).

O7 (north star tolerance): rel-Frobenius ||Y - Y64||_F / ||Y64||_F <= 1e-3 and,
element-wise, |Y - Y64| <= 1e-2 * ||A[m,:]||_2 * ||w[:,n]||_2; no NaN/Inf.
Reading R15: bf16 outputs get both bounds x8 (3 fewer mantissa bits).
"""

from __future__ import annotations

import numpy as np

from .dequant import dequant
from .formats import WType


def matmul_fp64(A: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Y64 = A @ w in float64 (A [M,K] fp16/any, w [K,N] float64 dequantized weights)."""
    return np.matmul(A.astype(np.float64), w.astype(np.float64))


def matmul_cols_fp64(wt: WType, A: np.ndarray, codes_cols: np.ndarray, scales_cols: np.ndarray,
                     zeros_cols: np.ndarray | None, group: int) -> np.ndarray:
    """Y64[:, cols] for a column sample: the same definition restricted to the given columns.

    ``codes_cols`` is [K, C] (the sampled columns of the code matrix), scales/zeros [K/G, C].
    Output column c depends only on column c of the weight (independent tiles).
    """
    w = dequant(wt, codes_cols, scales_cols, zeros_cols, group)
    return matmul_fp64(A, w)


def tolerance_check(Y: np.ndarray, Y64: np.ndarray, A: np.ndarray, w: np.ndarray,
                    out_dtype: str = "f16") -> dict:
    """O7.  Returns a dict with the measured errors and ``ok``.

    ``w`` is the (dequantized, float64) weight restricted to the columns of Y.
    """
    Yd = Y.astype(np.float64)
    factor = 8.0 if out_dtype == "bf16" else 1.0
    finite = bool(np.isfinite(Yd).all()) or not bool(np.isfinite(Y64).all())
    diff = Yd - Y64
    den = np.linalg.norm(Y64)
    rel_fro = float(np.linalg.norm(diff) / den) if den > 0 else float(np.linalg.norm(diff))
    row = np.linalg.norm(A.astype(np.float64), axis=1)[:, None]
    col = np.linalg.norm(w, axis=0)[None, :]
    bound = 1e-2 * factor * row * col
    excess = np.abs(diff) - bound
    max_ratio = float(np.max(np.abs(diff) / np.maximum(row * col, 1e-300))) if diff.size else 0.0
    ok = finite and rel_fro <= 1e-3 * factor and bool((excess <= 0).all())
    return {"ok": ok, "rel_fro": rel_fro, "max_abs_ratio": max_ratio, "finite": finite}
