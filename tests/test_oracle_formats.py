"""Pins for oracle O1/O2 (value of every code of every format) -- CPU only.

Each check compares the oracle with something other than itself:
  * integer formats: closed forms (identity; sign extension by arithmetic shift);
  * floats: ml_dtypes' own tables (float4_e2m1fn, float6_e2m3fn, float6_e3m2fn,
    float8_e4m3fn, float8_e3m4, float8_e4m3, float8_e5m2) where they exist, and
    the mantissa-embedding law value_{E,M}(c) == value_{E,M+1}(c with a 0
    mantissa bit appended), which chains every (E, M) to an ml_dtypes table or
    to the E=1 fixed-point closed form;
  * SPEC's worked examples (tests/golden/spec_examples.json).
"""

import json
import os

import ml_dtypes
import numpy as np
import pytest

from oracle import all_kernel_formats, code_values, oracle_only_formats, parse_wtype
from oracle.formats import WType

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _same(a, b):
    """Bit-level float equality including the sign of zero."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.array_equal(a, b) and np.array_equal(np.signbit(a), np.signbit(b))


def test_format_count():
    fmts = all_kernel_formats()
    assert len(fmts) == 37
    assert len({f.name for f in fmts}) == 37
    assert {f.name for f in oracle_only_formats()} == {"f6e5m0", "f7e5m1", "f7e6m0", "f8e5m2", "f8e6m1", "f8e7m0"}


@pytest.mark.parametrize("s", ["u1", "u8", "i1", "i6", "f3e1m1", "f6e3m2", "f8e4m3", "f3e2m0"])
def test_parse_roundtrip(s):
    assert parse_wtype(s).name == s


@pytest.mark.parametrize("s", ["u0", "u9", "f2e1m0", "f6e3m3", "f8e5m2", "x4", "i4e1m2"])
def test_parse_rejects(s):
    with pytest.raises(ValueError):
        parse_wtype(s)


@pytest.mark.parametrize("b", range(1, 9))
def test_uint_closed_form(b):
    assert _same(code_values(WType("u", b)), np.arange(1 << b))


@pytest.mark.parametrize("b", range(1, 9))
def test_int_sign_extension(b):
    # independent closed form: put the b-bit code in the top of an int8 and
    # arithmetic-shift it back down (sign extension by the hardware rule)
    c = np.arange(1 << b, dtype=np.int64)
    top = (c << (8 - b)).astype(np.uint8).view(np.int8).astype(np.int64)
    expect = top >> (8 - b)
    assert _same(code_values(WType("i", b)), expect)


def _ml_table(dt, bits):
    codes = np.arange(1 << bits, dtype=np.uint8)
    return codes.view(dt).astype(np.float64)


@pytest.mark.parametrize("name,dt", [("f4e2m1", ml_dtypes.float4_e2m1fn),
                                     ("f6e2m3", ml_dtypes.float6_e2m3fn),
                                     ("f6e3m2", ml_dtypes.float6_e3m2fn)])
def test_float_matches_ml_dtypes_exactly(name, dt):
    wt = parse_wtype(name)
    assert _same(code_values(wt), _ml_table(dt, wt.bits))


def test_f8e4m3_matches_e4m3fn_except_nan():
    ours = code_values(parse_wtype("f8e4m3"))
    ml = _ml_table(ml_dtypes.float8_e4m3fn, 8)
    nan = np.isnan(ml)
    assert np.flatnonzero(nan).tolist() == [0x7F, 0xFF]
    assert _same(ours[~nan], ml[~nan])
    # reading R3: no NaN; the all-ones code is the top of the last binade
    assert ours[0x7F] == 480.0 and ours[0xFF] == -480.0


@pytest.mark.parametrize("name,dt,E", [("f8e3m4", ml_dtypes.float8_e3m4, 3),
                                       ("f8e4m3", ml_dtypes.float8_e4m3, 4),
                                       ("f8e5m2", ml_dtypes.float8_e5m2, 5)])
def test_float8_ieee_like_below_top_binade(name, dt, E):
    wt = parse_wtype(name, kernel=False)
    ours = code_values(wt)
    ml = _ml_table(dt, 8)
    e = (np.arange(256) >> wt.man) & ((1 << E) - 1)
    keep = e < (1 << E) - 1  # IEEE-like types reserve the top binade for Inf/NaN
    assert _same(ours[keep], ml[keep])


def _append_mantissa_zero(wt: WType, c: int) -> int:
    s = c >> (wt.bits - 1)
    mag = c & ((1 << (wt.bits - 1)) - 1)
    return (s << wt.bits) | (mag << 1)


def _all_float_formats():
    return [f for f in all_kernel_formats() + oracle_only_formats() if f.kind == "f"]


@pytest.mark.parametrize("wt", [f for f in _all_float_formats() if f.bits < 8], ids=lambda w: w.name)
def test_mantissa_embedding(wt):
    """value_{E,M}(c) == value_{E,M+1}(c << 1): chains every format to a pinned table."""
    wider = WType("f", wt.bits + 1, wt.exp, wt.man + 1)
    a = code_values(wt)
    b = code_values(wider)
    idx = [_append_mantissa_zero(wt, c) for c in range(1 << wt.bits)]
    assert _same(a, b[idx])


@pytest.mark.parametrize("M", range(0, 7))
def test_e1_fixed_point_closed_form(M):
    """E=1 (bias 0) is fixed point: magnitudes are k * 2^(1-M), k = 0 .. 2^(M+1)-1."""
    if M == 0:
        pytest.skip("f2e1m0 is not a format (floats have >= 3 bits)")
    wt = WType("f", 2 + M, 1, M)
    v = code_values(wt)
    half = 1 << (wt.bits - 1)
    assert _same(v[:half], np.arange(half) * 2.0 ** (1 - M))
    assert _same(v[half:], -(np.arange(half) * 2.0 ** (1 - M)))


@pytest.mark.parametrize("wt", all_kernel_formats(), ids=lambda w: w.name)
def test_kernel_formats_are_fp16_exact(wt):
    """Reading R4: every code of every kernel format is exactly representable in fp16."""
    v = code_values(wt)
    assert _same(v.astype(np.float16).astype(np.float64), v)


def test_e5_not_fp16_exact():
    v = code_values(parse_wtype("f8e5m2", kernel=False))
    assert not _same(v.astype(np.float16).astype(np.float64), v)


@pytest.mark.parametrize("name,mx", [("f3e1m1", 3), ("f4e2m1", 6), ("f5e2m2", 7),
                                     ("f6e3m2", 28), ("f7e3m3", 30), ("f8e4m3", 480)])
def test_max_values(name, mx):
    v = code_values(parse_wtype(name))
    assert v.max() == mx and v.min() == -mx


@pytest.mark.parametrize("ex", GOLDEN["decode"], ids=lambda e: e["cite"])
def test_golden_decode(ex):
    assert code_values(parse_wtype(ex["dtype"]))[ex["code"]] == ex["value"]


@pytest.mark.parametrize("ex", GOLDEN["cast_f16"], ids=lambda e: e["cite"])
def test_golden_cast_f16(ex):
    v = code_values(parse_wtype(ex["dtype"]))[ex["codes"]].astype(np.float16)
    assert v.tolist() == ex["values"]


def test_negative_zero():
    v = code_values(parse_wtype("f6e3m2"))
    assert v[32] == 0.0 and np.signbit(v[32]) and not np.signbit(v[0])


@pytest.mark.parametrize("wt", _all_float_formats(), ids=lambda w: w.name)
def test_binade_is_evenly_spaced(wt):
    """Within each (sign, exponent) binade values are equally spaced, the subnormal binade
    shares the spacing of the first normal binade, and consecutive normal binades meet
    without a gap.  With the m=0 values anchored by the embedding chain to ml_dtypes, this
    pins the odd-mantissa codes of the widest formats (e.g. f8e2m5) too."""
    E, M = wt.exp, wt.man
    v = code_values(wt)
    pos = v[: 1 << (wt.bits - 1)]
    assert _same(v[1 << (wt.bits - 1):], -pos)
    steps = []
    for e in range(1 << E):
        b = pos[e << M:(e + 1) << M]
        d = np.diff(b)
        if M >= 1:
            assert np.allclose(d, d[0], rtol=0, atol=0)
            steps.append(d[0])
        if e >= 1 and e + 1 < (1 << E):
            nxt = pos[(e + 1) << M]
            step = (b[-1] - b[0]) / max((1 << M) - 1, 1) if M >= 1 else b[0]
            assert b[-1] + step == nxt
    if M >= 1 and E >= 1 and len(steps) >= 2:
        assert steps[0] == steps[1]
