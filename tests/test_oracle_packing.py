"""Pins for oracle O3/O4 (compact LSB-first storage) -- CPU only.

Independent references: numpy.packbits / numpy.unpackbits with
bitorder='little' applied to each code's bit expansion, the SPEC worked
examples, the length law ceil(count*b/8) and the store-locality law.
"""

import json
import os

import numpy as np
import pytest

from oracle import pack, packed_nbytes, parse_wtype, unpack

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _np_pack(codes, b):
    bits = np.unpackbits(codes.astype(np.uint8).reshape(-1, 1), axis=1, bitorder="little")[:, :b]
    return np.packbits(bits.reshape(-1), bitorder="little")


@pytest.mark.parametrize("b", range(1, 9))
def test_pack_matches_numpy_packbits(b):
    rng = np.random.default_rng(b)
    for n in [1, 2, 3, 7, 8, 9, 31, 128, 1000, 4097]:
        codes = rng.integers(0, 1 << b, size=n)
        assert np.array_equal(pack(codes, b), _np_pack(codes, b))


@pytest.mark.parametrize("b", range(1, 9))
def test_unpack_matches_numpy_unpackbits(b):
    rng = np.random.default_rng(100 + b)
    n = 777
    buf = rng.integers(0, 256, size=packed_nbytes(n, b), dtype=np.uint8)
    bits = np.unpackbits(buf, bitorder="little")[: n * b].reshape(n, b)
    expect = (bits.astype(np.int64) << np.arange(b)).sum(axis=1)
    assert np.array_equal(unpack(buf, n, b), expect)


@pytest.mark.parametrize("b", range(1, 9))
def test_roundtrip_10k_vectors(b):
    rng = np.random.default_rng(7 * b)
    total = 0
    while total < 10_000:
        n = int(rng.integers(1, 64))
        codes = rng.integers(0, 1 << b, size=n)
        buf = pack(codes, b)
        assert buf.size == packed_nbytes(n, b) == (n * b + 7) // 8
        assert np.array_equal(unpack(buf, n, b), codes)
        # trailing pad bits are zero
        pad = buf.size * 8 - n * b
        if pad:
            assert int(buf[-1]) >> (8 - pad) == 0
        total += 1


@pytest.mark.parametrize("b", range(1, 9))
def test_store_locality(b):
    """Changing element k changes only stream bits [k*b, (k+1)*b)."""
    rng = np.random.default_rng(b + 50)
    codes = rng.integers(0, 1 << b, size=40)
    base = np.unpackbits(pack(codes, b), bitorder="little")
    for k in [0, 1, 5, 17, 39]:
        c2 = codes.copy()
        c2[k] = (c2[k] + 1) % (1 << b)
        now = np.unpackbits(pack(c2, b), bitorder="little")
        changed = np.flatnonzero(base != now)
        assert changed.size and changed.min() >= k * b and changed.max() < (k + 1) * b


def test_u8_is_plain_bytes():
    codes = np.arange(256)
    assert np.array_equal(pack(codes, 8), codes.astype(np.uint8))


def test_pack_rejects_oversized():
    with pytest.raises(ValueError):
        pack(np.array([16]), 4)


@pytest.mark.parametrize("ex", GOLDEN["unpack"], ids=lambda e: e["cite"])
def test_golden_unpack(ex):
    b = parse_wtype(ex["dtype"]).bits
    assert unpack(np.array(ex["bytes"], dtype=np.uint8), ex["count"], b).tolist() == ex["codes"]


@pytest.mark.parametrize("ex", GOLDEN["pack"], ids=lambda e: e["cite"])
def test_golden_pack(ex):
    b = parse_wtype(ex["dtype"]).bits
    assert pack(np.array(ex["codes"]), b).tolist() == ex["bytes"]


@pytest.mark.parametrize("ex", GOLDEN["sizes"], ids=lambda e: e["cite"])
def test_golden_sizes(ex):
    b = parse_wtype(ex["dtype"]).bits
    assert packed_nbytes(ex["K"] * ex["N"], b) == ex["nbytes"]


def test_row_major_flattening():
    """Reading R2: [K,N] flattens row-major, so element (k, n) is stream element k*N+n."""
    codes = np.arange(12).reshape(3, 4) % 16
    flat = unpack(pack(codes, 4), 12, 4)
    assert flat.reshape(3, 4)[2, 1] == codes[2, 1]
