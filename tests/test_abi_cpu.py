"""The C-ABI library loads and exports every symbol include/tilus_b200.h declares,
and its host-only entry points (sizes, validation, error strings) behave -- CPU only,
no compute calls."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tilus_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tl_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import paper_2504_12984_b200 as P
    return P


def test_header_declares_the_boundary():
    names = _declared()
    for must in ["tl_pack", "tl_transform_weights", "tl_matmul", "tl_matmul_workspace_bytes", "tl_dequant",
                 "tl_packed_bytes", "tl_transformed_bytes", "tl_status_str", "tl_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    so = ctypes.CDLL(lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(so, n)]
    assert not missing, missing
    assert sorted(lib.EXPORTED) == _declared()


def test_sizes(lib):
    w = lib.wtype("i6")
    assert lib.tl_packed_bytes(w, 4, 8) == 24        # P:187 / S:468
    assert lib.tl_packed_bytes(lib.wtype("u3"), 3, 3) == 4  # ceil(27/8)
    assert lib.tl_transformed_bytes(w, 128, 256) == 128 * 256 * 6 // 8
    assert lib.tl_transformed_bytes(w, 100, 256) == 0  # K not a multiple of 128
    assert lib.tl_format_version() >= 1
    assert lib.tl_matmul_workspace_bytes(lib.wtype("u4"), 1, 512, 512, 128) > 0


def test_bad_arguments_rejected_before_any_launch(lib):
    import torch
    w = lib.wtype("u4")
    # descriptors that are not kernel formats
    for bad in [lib.tl_wtype(0, 9, 0, 0), lib.tl_wtype(2, 8, 5, 2), lib.tl_wtype(2, 6, 3, 3), lib.tl_wtype(3, 4, 0, 0)]:
        st = lib._lib._tl_matmul(bad, 0, 1, 128, 128, 128, 16, 128, 16, 16, None, 16, 128, 16, 1 << 20, None)
        assert lib._lib._tl_status_str(st).decode() == "TL_EINVAL_DTYPE"
    # shape / group / zeros / alignment / workspace checks
    cases = [
        (dict(N=100), "TL_EINVAL_SHAPE"),
        (dict(K=200), "TL_EINVAL_SHAPE"),
        (dict(G=48), "TL_EINVAL_GROUP"),
        (dict(G=96), "TL_EINVAL_GROUP"),
        (dict(A=0), "TL_ENULL"),
        (dict(A=8), "TL_EALIGN"),
        (dict(ws=1), "TL_EWORKSPACE"),
        (dict(lda=64), "TL_EINVAL_SHAPE"),
    ]
    for kw, expect in cases:
        a = dict(M=1, N=128, K=128, G=128, A=16, lda=None, ws=1 << 24)
        a.update(kw)
        st = lib._lib._tl_matmul(w, 0, a["M"], a["N"], a["K"], a["G"], a["A"] or None,
                                 a["lda"] if a["lda"] is not None else a["K"], 16, 16, None, 16, a["N"], 16,
                                 a["ws"], None)
        assert lib._lib._tl_status_str(st).decode() == expect, (kw, lib._lib._tl_last_error())
    st = lib._lib._tl_matmul(lib.wtype("i4"), 0, 1, 128, 128, 128, 16, 128, 16, 16, 16, 16, 128, 16, 1 << 24, None)
    assert lib._lib._tl_status_str(st).decode() == "TL_EZEROS"
    # M == 0 is a no-op
    st = lib._lib._tl_matmul(w, 0, 0, 128, 128, 128, 16, 128, 16, 16, None, 16, 128, 16, 1 << 24, None)
    assert st == 0
    st = lib._lib._tl_matmul(w, 0, 1, 128, 128, 128, 16, 128, 16, 16, None, 16, 128, 16, 64, None)
    assert lib._lib._tl_status_str(st).decode() == "TL_EWORKSPACE"
    assert "workspace" in lib._lib._tl_last_error().decode()
    # activation types: fp16 and bf16 are defined, anything else is rejected
    st = lib._lib._tl_matmul(w, 7, 1, 128, 128, 128, 16, 128, 16, 16, None, 16, 128, 16, 1 << 24, None)
    assert lib._lib._tl_status_str(st).decode() == "TL_EUNSUPPORTED"
    assert lib.tl_matmul_workspace_bytes(w, 1, 128, 128, 128, atype=7) == 0
    assert lib.tl_matmul_workspace_bytes(w, 1, 128, 128, 128, atype=lib.TL_ACT_BF16) > 0
    # int8 activations (row f4): the workspace grows by the staged fp16 copy of A (2*M*K bytes, 256-aligned)
    f16 = lib.tl_matmul_workspace_bytes(w, 3, 256, 512, 128)
    assert lib.tl_matmul_workspace_bytes(w, 3, 256, 512, 128, atype=lib.TL_ACT_I8) == (f16 + 255) // 256 * 256 + 2 * 3 * 512
    # int8 rows need 16-byte strides in BYTES: lda = 8 int8 elements is misaligned, 16 is fine (then NULL ws)
    st = lib._lib._tl_matmul(w, lib.TL_ACT_I8, 1, 128, 128, 128, 16, 136, 16, 16, None, 16, 128, 16, 1 << 24, None)
    assert lib._lib._tl_status_str(st).decode() == "TL_EALIGN"
    st = lib._lib._tl_matmul(w, lib.TL_ACT_I8, 1, 128, 128, 128, 16, 144, 16, 16, None, 16, 128, 0, 1 << 24, None)
    assert lib._lib._tl_status_str(st).decode() == "TL_EWORKSPACE"
    # MX scale conversion: argument checks only (no launch on CPU)
    assert lib._lib._tl_status_str(lib._lib._tl_mx_scales_to_f16(16, -1, 0, 16, None)).decode() == "TL_EINVAL_SHAPE"
    assert lib._lib._tl_status_str(lib._lib._tl_mx_scales_to_f16(None, 4, 0, 16, None)).decode() == "TL_ENULL"
    assert lib._lib._tl_status_str(lib._lib._tl_mx_scales_to_f16(16, 4, 65, 16, None)).decode() == "TL_EINVAL_SHAPE"
    assert lib._lib._tl_mx_scales_to_f16(16, 0, 0, 16, None) == 0
    # tl_matmul_ex: unknown flags / paths, negative splits
    def ex(path=0, splits=0, flags=0):
        return lib._lib._tl_status_str(lib._lib._tl_matmul_ex(w, 0, 1, 128, 128, 128, 16, 128, 16, 16, None, 16,
                                                              128, 16, 1 << 24, path, splits, flags,
                                                              None)).decode()
    assert ex(flags=2) == "TL_EINVAL_SHAPE"
    assert ex(path=7) == "TL_EUNSUPPORTED"
    assert ex(splits=-1) == "TL_EINVAL_SHAPE"
    del torch


def test_python_binding_raises_on_error(lib):
    with pytest.raises(lib.TilusError):
        lib._lib._check(2, "x")


def test_wtype_grammar(lib):
    assert lib.wtype("f6e3m2").name == "f6e3m2"
    assert (lib.wtype("i5").kind, lib.wtype("i5").bits) == (1, 5)
    with pytest.raises(ValueError):
        lib.wtype("q4")


def test_batch_hostio_argument_checks(lib):
    L = lib._lib
    items = (L.tl_batch_item * 1)()
    st = L._tl_matmul_batch_hostio(0, -1, items, 16, 16, 16, 16, 0, None)
    assert L._tl_status_str(st).decode() == "TL_EINVAL_SHAPE"
    assert L._tl_matmul_batch_hostio(0, 0, None, None, None, None, None, 0, None) == 0  # empty batch: no-op
    st = L._tl_matmul_batch_hostio(0, 1, items, None, 16, 16, 16, 0, None)
    assert L._tl_status_str(st).decode() == "TL_ENULL"
    st = L._tl_matmul_batch_hostio(9, 1, items, 16, 16, 16, 16, 0, None)
    assert L._tl_status_str(st).decode() == "TL_EUNSUPPORTED"
    items[0].M, items[0].N, items[0].K = 1, 0, 128
    st = L._tl_matmul_batch_hostio(0, 1, items, 16, 16, 16, 16, 0, None)
    assert L._tl_status_str(st).decode() == "TL_EINVAL_SHAPE"


def test_row_parallel_argument_checks(lib):
    L = lib._lib
    VP = L._vp * 8
    st = lambda x: L._tl_status_str(x).decode()
    assert st(L._tl_signal_peers(VP(*[16] * 8), 8, None)) == "TL_EINVAL_SHAPE"
    assert st(L._tl_signal_peers(VP(18), 1, None)) == "TL_EALIGN"
    assert L._tl_signal_peers(None, 0, None) == 0
    assert st(L._tl_reduce_scatter_peer(2, VP(16, 32), 2, 1, 128, 128, 16, 128, None)) == "TL_EUNSUPPORTED"
    assert st(L._tl_reduce_scatter_peer(0, VP(16, 32), 9, 1, 128, 128, 16, 128, None)) == "TL_EINVAL_SHAPE"
    assert st(L._tl_reduce_scatter_peer(0, VP(16, 32), 2, 1, 100, 128, 16, 128, None)) == "TL_EINVAL_SHAPE"
    assert st(L._tl_reduce_scatter_peer(0, VP(16, 32), 2, 1, 128, 64, 16, 128, None)) == "TL_EINVAL_SHAPE"
    assert st(L._tl_reduce_scatter_peer(0, VP(16, 40), 2, 1, 128, 128, 16, 128, None)) == "TL_EALIGN"
    assert L._tl_reduce_scatter_peer(0, VP(16, 32), 2, 0, 128, 128, 16, 128, None) == 0
