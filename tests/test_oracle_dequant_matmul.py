"""Pins for oracle O5 (dequant), O6 (fp64 matmul), O7 (tolerance), O9 (encode) -- CPU only.

Independent references: exact rational arithmetic (fractions.Fraction) brute
force on tiny shapes, fp32 exactness of every dequantized value, SPEC's worked
examples, and the special cases W=0, M=K=1, A=I.
"""

import json
import os
from fractions import Fraction

import numpy as np
import pytest

import workloads as wl
from oracle import (all_kernel_formats, code_values, dequant, encode, matmul_fp64, parse_wtype,
                    tolerance_check)

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLDEN["dequant"], ids=lambda e: e["cite"])
def test_golden_dequant(ex):
    wt = parse_wtype(ex["dtype"])
    w = dequant(wt, np.array(ex["codes"], dtype=np.uint8), np.array(ex["scales"], dtype=np.float16),
                None, ex["group"])
    assert w.tolist() == ex["values"]


def _fraction_dequant(wt, q, s, z):
    """Exact rational (value(q) - z) * s, written from the value definition with Fractions."""
    b = wt.bits
    if wt.kind == "u":
        v = Fraction(q)
    elif wt.kind == "i":
        v = Fraction(q - (1 << b) if q >= (1 << (b - 1)) else q)
    else:
        E, M = wt.exp, wt.man
        sgn = -1 if q >> (b - 1) else 1
        e = (q >> M) & ((1 << E) - 1)
        m = q & ((1 << M) - 1)
        bias = (1 << (E - 1)) - 1
        if e == 0:
            v = sgn * Fraction(2) ** (1 - bias) * Fraction(m, 1 << M)
        else:
            v = sgn * Fraction(2) ** (e - bias) * (1 + Fraction(m, 1 << M))
    return (v - Fraction(z)) * Fraction(float(s))


@pytest.mark.parametrize("wt", all_kernel_formats(), ids=lambda w: w.name)
def test_dequant_exact_and_fp32_representable(wt):
    """Every dequantized value equals the exact rational and is exact in fp32 (O5)."""
    rng = np.random.default_rng(wt.bits * 31 + wt.kind_code)
    nq = 1 << wt.bits
    # all codes x 64 random finite fp16 scales (positive and negative, normal and subnormal)
    raw = rng.integers(0, 0x7C00, size=64).astype(np.uint16)
    raw[::2] |= 0x8000
    scales = raw.view(np.float16)
    codes = np.tile(np.arange(nq, dtype=np.uint8), (64, 1)).T  # [nq, 64]
    G = nq
    zeros = None
    if wt.kind == "u":
        zeros = rng.integers(0, nq, size=(1, 64)).astype(np.float16)
    w = dequant(wt, codes, scales.reshape(1, 64), zeros, G)
    assert np.array_equal(w.astype(np.float32).astype(np.float64), w)
    for i in range(0, nq, max(1, nq // 16)):
        for j in range(0, 64, 7):
            z = 0 if zeros is None else int(zeros[0, j])
            exact = _fraction_dequant(wt, i, scales[j], z)
            assert Fraction(w[i, j]) == exact


def test_dequant_unit_scale_is_value_table():
    wt = parse_wtype("f6e3m2")
    codes = np.arange(64, dtype=np.uint8).reshape(64, 1)
    w = dequant(wt, codes, np.ones((1, 1), np.float16), None, 64)
    assert np.array_equal(w[:, 0], code_values(wt))


def test_dequant_groups_index_rows():
    """g = k // G (R8): row k uses scale row k // G."""
    wt = parse_wtype("u4")
    codes = np.ones((8, 2), dtype=np.uint8)
    scales = np.array([[1, 2], [3, 4]], dtype=np.float16)
    w = dequant(wt, codes, scales, np.zeros((2, 2), np.float16), 4)
    assert w[:4].tolist() == [[1, 2]] * 4 and w[4:].tolist() == [[3, 4]] * 4


def test_dequant_zero_points_uint_only():
    with pytest.raises(ValueError):
        dequant(parse_wtype("i4"), np.zeros((4, 1), np.uint8), np.ones((1, 1), np.float16),
                np.zeros((1, 1), np.float16), 4)


def test_dequant_negative_zero_sign():
    """R13: float -0 code times s keeps IEEE sign; (q - z) = 0 gives +0."""
    wt = parse_wtype("f4e2m1")
    w = dequant(wt, np.array([[8]], np.uint8), np.array([[0.5]], np.float16), None, 1)
    assert w[0, 0] == 0 and np.signbit(w[0, 0])
    wu = dequant(parse_wtype("u4"), np.array([[3]], np.uint8), np.array([[-0.5]], np.float16),
                 np.array([[3]], np.float16), 1)
    assert wu[0, 0] == 0


@pytest.mark.parametrize("fmt", ["u3", "i5", "f6e3m2", "u8", "i1", "f3e1m1"])
def test_matmul_vs_exact_rational(fmt):
    """fp64 matmul vs exact Fraction sums on tiny shapes: error within K * 2^-53 * sum|terms|."""
    wt = parse_wtype(fmt)
    M, K, N, G = 3, 64, 5, 32
    seed = wl.stable_seed("frac", fmt)
    A = wl.gen_activations(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    z = wl.gen_zeros(fmt, K, N, G, seed)
    Y = matmul_fp64(A, dequant(wt, codes, s, z, G))
    for m in range(M):
        for n in range(N):
            terms = []
            for k in range(K):
                zz = 0 if z is None else int(z[k // G, n])
                terms.append(Fraction(float(A[m, k])) * _fraction_dequant(wt, int(codes[k, n]), s[k // G, n], zz))
            exact = sum(terms, Fraction(0))
            bound = K * 2.0 ** -53 * float(sum(abs(t) for t in terms))
            assert abs(Fraction(Y[m, n]) - exact) <= Fraction(bound)


def test_matmul_special_cases():
    wt = parse_wtype("u4")
    K, N, G = 128, 16, 128
    A = wl.gen_activations(4, K, 1)
    s = wl.gen_scales("u4", K, N, G, 1)
    # W = 0 -> 0: code == zero point everywhere
    z = np.full((1, N), 5, np.float16)
    codes = np.full((K, N), 5, np.uint8)
    assert not matmul_fp64(A, dequant(wt, codes, s, z, G)).any()
    # M = K = 1 -> A * deq(W)
    w1 = dequant(wt, np.array([[7, 3]], np.uint8), np.array([[0.25, 0.5]], np.float16),
                 np.array([[1, 2]], np.float16), 1)
    assert matmul_fp64(np.array([[2.0]], np.float16), w1).tolist() == [[3.0, 1.0]]
    # A = I -> Y = w
    codes = wl.gen_codes("u4", 16, N, 2)
    w = dequant(wt, codes, wl.gen_scales("u4", 16, N, 16, 2), wl.gen_zeros("u4", 16, N, 16, 2), 16)
    assert np.array_equal(matmul_fp64(np.eye(16, dtype=np.float16), w), w)


def test_tolerance_comparator():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((4, 256)).astype(np.float16)
    w = rng.standard_normal((256, 64)) * 0.02
    Y64 = matmul_fp64(A, w)
    assert tolerance_check(Y64.astype(np.float16), Y64, A, w)["ok"]
    bad = (Y64 * 1.01).astype(np.float16)
    r = tolerance_check(bad, Y64, A, w)
    assert not r["ok"] and r["rel_fro"] > 5e-3
    one = Y64.astype(np.float16).copy()
    one[1, 3] += 100
    assert not tolerance_check(one, Y64, A, w)["ok"]
    nan = Y64.astype(np.float16).copy()
    nan[0, 0] = np.nan
    assert not tolerance_check(nan, Y64, A, w)["ok"]
    # bf16-rounded output fails the fp16 bound but passes the bf16 bound (R15)
    import ml_dtypes
    yb = Y64.astype(ml_dtypes.bfloat16)
    assert tolerance_check(yb, Y64, A, w, "bf16")["ok"]


def test_fp32_accumulation_fits_tolerance_fp16_chunks_do_not():
    """Reading R10: fp32 accumulation is required; long fp16 accumulation breaks O7."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((16, 4096)).astype(np.float16)
    w = (rng.standard_normal((4096, 256)) * 0.02).astype(np.float16).astype(np.float64)
    Y64 = matmul_fp64(A, w)
    y32 = (A.astype(np.float32) @ w.astype(np.float32)).astype(np.float16)
    assert tolerance_check(y32, Y64, A, w)["ok"]
    acc = np.zeros((16, 256), np.float16)
    for k in range(4096):
        acc = (acc + (A[:, k:k + 1].astype(np.float16) * w[k:k + 1].astype(np.float16))).astype(np.float16)
    assert not tolerance_check(acc, Y64, A, w)["ok"]


@pytest.mark.parametrize("wt", all_kernel_formats(), ids=lambda w: w.name)
def test_encode_inverts_decode(wt):
    """decode . encode is the identity on the code space."""
    v = code_values(wt)
    assert np.array_equal(encode(wt, v), np.arange(v.size))


@pytest.mark.parametrize("ex", GOLDEN["encode"], ids=lambda e: e["cite"])
def test_golden_encode(ex):
    assert int(encode(parse_wtype(ex["dtype"]), np.array([ex["value"]]))[0]) == ex["code"]


def test_encode_round_half_even_and_saturate():
    wt = parse_wtype("i4")
    assert encode(wt, np.array([2.5, 3.5, -2.5, 100.0, -100.0])).tolist() == [2, 4, 14, 7, 8]


def test_exact_instance_is_exact():
    """The generator's exact-integer instance makes fp32 accumulation order-independent."""
    fmt, M, K, N, G = "u8", 2, 8192, 8, 128
    A, codes, s, z = wl.gen_exact_instance(fmt, M, K, N, G, seed=3)
    w = dequant(parse_wtype(fmt), codes, s, z, G)
    y64 = matmul_fp64(A, w)
    fwd = np.zeros((M, N), np.float32)
    for k in range(K):
        fwd += A[:, k:k + 1].astype(np.float32) * w[k:k + 1].astype(np.float32)
    rev = np.zeros((M, N), np.float32)
    for k in reversed(range(K)):
        rev += A[:, k:k + 1].astype(np.float32) * w[k:k + 1].astype(np.float32)
    assert np.array_equal(fwd, y64) and np.array_equal(rev, y64)


def _elementwise_case():
    """A problem where rel-Frobenius stays far below 1e-3 while one element misses by more than
    1e-2 * ||A_m|| * ||w_n||: only O7's element-wise clause (north star) can reject it."""
    rng = np.random.default_rng(7)
    M, K, N = 64, 256, 4096
    A = rng.standard_normal((M, K)).astype(np.float16)
    w = rng.standard_normal((K, N)) * 0.02
    Y64 = matmul_fp64(A, w)
    bound = 1e-2 * np.linalg.norm(A.astype(np.float64), axis=1)[:, None] * np.linalg.norm(w, axis=0)[None, :]
    return A, w, Y64, bound


def test_tolerance_elementwise_clause_rejects_single_outlier():
    A, w, Y64, bound = _elementwise_case()
    Y = Y64.astype(np.float16)
    m, n = 37, 2049
    Y[m, n] = np.float16(Y64[m, n] + 1.5 * bound[m, n])
    d = Y.astype(np.float64) - Y64
    rel = np.linalg.norm(d) / np.linalg.norm(Y64)
    assert rel <= 1e-3                              # the Frobenius clause alone would accept it
    assert abs(d[m, n]) > bound[m, n]               # ... the element-wise clause must not
    r = tolerance_check(Y, Y64, A, w)
    assert not r["ok"] and r["rel_fro"] <= 1e-3
    # the clause is per (row, column): the same absolute error on an element whose row norm is
    # 4x larger is inside its own bound
    A2 = A.copy()
    A2[m] *= 4
    Y64b = matmul_fp64(A2, w)
    Yb = Y64b.astype(np.float16)
    Yb[m, n] = np.float16(Y64b[m, n] + 1.5 * bound[m, n])
    assert tolerance_check(Yb, Y64b, A2, w)["ok"]


def test_tolerance_elementwise_clause_uses_row_and_column_norms():
    """Mis-axing the bound (column norm of A, row norm of w) would change which element passes:
    a column of w 10x smaller than the rest tightens only that column's bound."""
    A, w, Y64, _ = _elementwise_case()
    w = w.copy()
    w[:, 5] *= 0.1
    Y64 = matmul_fp64(A, w)
    bcol = 1e-2 * np.linalg.norm(A[0].astype(np.float64)) * np.linalg.norm(w[:, 5])
    Y = Y64.astype(np.float16)
    Y[0, 5] = np.float16(Y64[0, 5] + 2.0 * bcol)       # outside column 5's (small) bound
    assert not tolerance_check(Y, Y64, A, w)["ok"]
    Y = Y64.astype(np.float16)
    Y[0, 6] = np.float16(Y64[0, 6] + 2.0 * bcol)       # same error, inside column 6's bound
    assert tolerance_check(Y, Y64, A, w)["ok"]


def test_tolerance_max_abs_ratio_is_the_guard_statistic():
    """max_abs_ratio = max |Y - Y64| / (||A_m|| ||w_n||): the statistic the GPU tests also hold to
    the 1e-3 internal regression guard (observed ~1.5e-5 for fp16 output)."""
    A, w, Y64, bound = _elementwise_case()
    Y = Y64.astype(np.float16)
    r = tolerance_check(Y, Y64, A, w)
    assert r["ok"] and r["max_abs_ratio"] < 1e-4
    Y[3, 3] = np.float16(Y64[3, 3] + 0.5 * bound[3, 3])   # 5e-3 of the norm product: inside O7
    r = tolerance_check(Y, Y64, A, w)
    assert r["ok"] and 4e-3 < r["max_abs_ratio"] < 6e-3   # ... but 5x over the 1e-3 guard
