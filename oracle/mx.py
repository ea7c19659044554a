"""Row f4 -- microscaling (MX) block scales.  TEST INFRASTRUCTURE ONLY.

The paper: "Microscaling data types [mx-format] can be thought as a more fine-grained
quantization thus we could also support it".  It gives no formula; reading R25
 takes the cited format's definition: a block of 32 consecutive weights along K
shares one E8M0 scale code e (8 exponent bits, no sign, no mantissa), whose value is
2^(e - 127); code 0xFF is NaN.  An element's value is value(code) * 2^(e - 127), with the
element formats fp4 e2m1, fp6 e2m3 / e3m2 and fp8 e4m3 (kernel formats, reading R3's value
table) and MXINT8 = int8 with an implicit 2^-6 (passed as ``exp_adjust = -6``).

The library converts E8M0 codes to its fp16 group scales once (tl_mx_scales_to_f16); the
fp16 value of the scale is exactly 2^x for x = e - 127 + adj in [-24, 15] and NaN otherwise.
"""

from __future__ import annotations

import numpy as np

from .formats import WType, code_values

MX_BLOCK = 32


def e8m0_value(e: np.ndarray, exp_adjust: int = 0) -> np.ndarray:
    """E8M0 code -> 2^(e - 127 + exp_adjust) in float64; 0xFF -> NaN (R25)."""
    e = np.asarray(e).astype(np.int64)
    v = np.ldexp(1.0, e - 127 + exp_adjust)
    return np.where(e == 0xFF, np.nan, v)


def e8m0_to_f16_scale(e: np.ndarray, exp_adjust: int = 0) -> np.ndarray:
    """The library's fp16 group scale for an E8M0 code: the exact value when it is an fp16
    number (2^-24 .. 2^15), else NaN (R25)."""
    v = e8m0_value(e, exp_adjust)
    x = np.asarray(e).astype(np.int64) - 127 + exp_adjust
    ok = np.isfinite(v) & (x >= -24) & (x <= 15)
    return np.where(ok, v, np.nan).astype(np.float16)


def e8m0_to_bf16_scale(e: np.ndarray, exp_adjust: int = 0) -> np.ndarray:
    """The library's bf16 group scale for an E8M0 code (bf16 activations): the exact value when it is
    a bf16 number (2^-133 .. 2^127), else NaN (R25).  Returned as float64 values."""
    v = e8m0_value(e, exp_adjust)
    x = np.asarray(e).astype(np.int64) - 127 + exp_adjust
    ok = np.isfinite(v) & (x >= -133) & (x <= 127)
    return np.where(ok, v, np.nan)


def mx_dequant(wt: WType, codes: np.ndarray, e8m0: np.ndarray, exp_adjust: int = 0) -> np.ndarray:
    """codes [K,N] uint8, e8m0 [K/32,N] uint8 -> w [K,N] float64 = value(code) * 2^(e-127+adj).

    Exact: value has <= 8 significant bits and the scale is a power of two.
    """
    codes = np.asarray(codes)
    K, N = codes.shape
    if K % MX_BLOCK or e8m0.shape != (K // MX_BLOCK, N):
        raise ValueError("MX scales must be [K/32, N]")
    vals = code_values(wt)[codes.astype(np.int64)]
    blk = np.arange(K) // MX_BLOCK
    return vals * e8m0_value(e8m0, exp_adjust)[blk, :]
