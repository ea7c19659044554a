"""Pins of the MX oracle (row f4, reading R25) against an independent implementation:
ml_dtypes' OCP types float8_e8m0fnu (the scale), float4_e2m1fn / float6_e2m3fn / float6_e3m2fn /
float8_e4m3fn (the elements) and IEEE half bit patterns.  CPU only."""

import ml_dtypes
import numpy as np
import pytest

from oracle import e8m0_to_f16_scale, e8m0_value, mx_dequant, parse_wtype

ALL = np.arange(256, dtype=np.uint8)


def test_e8m0_value_matches_ml_dtypes_on_every_code():
    ref = ALL.view(ml_dtypes.float8_e8m0fnu).astype(np.float64)
    got = e8m0_value(ALL)
    assert np.isnan(got[255]) and np.isnan(ref[255])
    assert np.array_equal(got[:255], ref[:255])
    assert got[127] == 1.0 and got[0] == 2.0 ** -127 and got[254] == 2.0 ** 127


@pytest.mark.parametrize("adj", [0, -6, 10, -30])
def test_f16_scale_is_exact_in_range_and_nan_outside(adj):
    s = e8m0_to_f16_scale(ALL, adj)
    x = ALL.astype(np.int64) - 127 + adj
    for e in range(256):
        xe = int(x[e])
        if e == 255 or xe < -24 or xe > 15:
            assert np.isnan(s[e]), e
        else:
            bits = int(s[e:e + 1].view(np.uint16)[0])
            # IEEE binary16: normal 2^x has biased exponent x+15 and a zero fraction; subnormal
            # 2^x (x < -14) is fraction bit x+24 with a zero exponent field
            want = ((xe + 15) << 10) if xe >= -14 else (1 << (xe + 24))
            assert bits == want, (e, hex(bits), hex(want))
            assert float(s[e]) == 2.0 ** xe


@pytest.mark.parametrize("fmt,mlt,adj", [("f4e2m1", ml_dtypes.float4_e2m1fn, 0),
                                         ("f6e2m3", ml_dtypes.float6_e2m3fn, 0),
                                         ("f6e3m2", ml_dtypes.float6_e3m2fn, 0),
                                         ("f8e4m3", ml_dtypes.float8_e4m3fn, 0),
                                         ("i8", None, -6)])
def test_mx_dequant_matches_ocp_element_and_scale_types(fmt, mlt, adj):
    rng = np.random.default_rng(7)
    K, N = 128, 24
    b = int(fmt[1])
    codes = rng.integers(0, 1 << b, size=(K, N)).astype(np.uint8)
    e = rng.integers(100, 140, size=(K // 32, N)).astype(np.uint8)
    e[0, 0] = 255  # the NaN scale code poisons exactly its block of 32
    got = mx_dequant(parse_wtype(fmt), codes, e, adj)
    if mlt is None:
        elem = codes.view(np.int8).astype(np.float64)                 # MXINT8: two's complement
    else:
        elem = codes.view(mlt).astype(np.float64)
    scale = e.view(ml_dtypes.float8_e8m0fnu).astype(np.float64) * 2.0 ** adj
    ref = elem * np.repeat(scale, 32, axis=0)
    if fmt == "f8e4m3":
        # reading R3: codes S.1111.111 are +-480 here (no NaN), OCP e4m3fn makes them NaN
        nan_codes = (codes & 0x7F) == 0x7F
        assert np.isnan(ref[nan_codes]).all()
        ref = np.where(nan_codes, np.where(codes >= 128, -480.0, 480.0) * np.repeat(scale, 32, axis=0), ref)
    assert np.isnan(got[:32, 0]).all() and not np.isnan(got[32:, 0]).any()
    ok = ~np.isnan(ref)
    assert np.array_equal(got[ok], ref[ok])
    assert np.array_equal(np.isnan(got), np.isnan(ref))


def test_mx_dequant_rejects_bad_block_shape():
    with pytest.raises(ValueError):
        mx_dequant(parse_wtype("f4e2m1"), np.zeros((64, 8), np.uint8), np.zeros((1, 8), np.uint8))


@pytest.mark.parametrize("adj", [0, -6, -10, 3])
def test_bf16_scale_is_exact_in_range(adj):
    from oracle import e8m0_to_bf16_scale
    v = e8m0_to_bf16_scale(ALL, adj)
    x = ALL.astype(np.int64) - 127 + adj
    for e in range(256):
        xe = int(x[e])
        if e == 255 or xe < -133 or xe > 127:
            assert np.isnan(v[e]), e
        else:
            b = np.array([v[e]]).astype(ml_dtypes.bfloat16)
            assert float(b[0]) == 2.0 ** xe  # representable in bf16, hence exact
            bits = int(b.view(np.uint16)[0])
            # IEEE-style bf16: normal 2^x has biased exponent x+127, subnormal (x < -126) bit x+133
            assert bits == (((xe + 127) << 7) if xe >= -126 else (1 << (xe + 133))), (e, hex(bits))
    # with adj = 0 every finite E8M0 code is a bf16 number (the reason bf16 scales need no range check)
    if adj == 0:
        assert not np.isnan(v[:255]).any()
