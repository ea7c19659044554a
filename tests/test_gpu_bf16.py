"""GPU parity with bf16 activations, scales, zero points and output (SURVEY §8(f) row f2,
PAPER.md:527 "we also support bfloat16").  The oracle takes the bf16 values exactly (fp64);
tolerance per reading R15: both O7 bounds x8 for a bf16 output (3 fewer mantissa bits)."""

import ml_dtypes
import numpy as np
import pytest

import workloads as wl
from helpers import make_problem, prepare_weights
from oracle import dequant, matmul_fp64, parse_wtype, tolerance_check

pytestmark = pytest.mark.gpu
BF = ml_dtypes.bfloat16
GEMV, TC, TCD, PREFILL = 1, 2, 3, 4


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2504_12984_b200 as P
    return P, torch


def _dev_bf16(x, torch):
    """numpy bf16 array -> CUDA torch.bfloat16 tensor (bit copy)."""
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).cuda().view(torch.bfloat16)


def _run(P, torch, fmt, A, codes, s, z, G, path, ldy=None):
    M, K = A.shape
    N = codes.shape[1]
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    ldy = ldy or N
    Y = torch.full((M, ldy), float("nan"), dtype=torch.bfloat16, device="cuda")
    ws = P.alloc_workspace(w, M, N, K, G)
    P.tl_matmul_ex(w, M, N, K, G, _dev_bf16(A, torch), wt, _dev_bf16(s, torch),
                   None if z is None else _dev_bf16(z, torch), Y, ws, path=path, ldy=ldy)
    torch.cuda.synchronize()
    full = Y.view(torch.int16).cpu().numpy().view(BF)
    return full[:, :N], full


def _bf16_problem(fmt, M, K, N, G, tag):
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag=tag)
    return (A.astype(np.float32).astype(BF), codes, s.astype(np.float32).astype(BF),
            None if z is None else z.astype(np.float32).astype(BF))


@pytest.mark.parametrize("path,M", [(TCD, 1), (TCD, 5), (TCD, 16), (TC, 24), (TC, 128), (TC, 200),
                                    (PREFILL, 600), (0, 1), (GEMV, 1)])
@pytest.mark.parametrize("fmt", ["u1", "u4", "i3", "i8", "u8", "f4e2m1", "f6e3m2", "f8e4m3"])
def test_bf16_parity(env, fmt, path, M):
    P, torch = env
    K, N, G = 1024, 384, 128
    A, codes, s, z = _bf16_problem(fmt, M, K, N, G, "bf16")
    Y, full = _run(P, torch, fmt, A, codes, s, z, G, path, ldy=N + 8)
    assert np.isnan(full[:, N:].astype(np.float32)).all()
    wd = dequant(parse_wtype(fmt), codes, s, z, G)
    r = tolerance_check(Y, matmul_fp64(A, wd), A, wd, "bf16")
    assert r["ok"], r
    assert r["max_abs_ratio"] <= 8e-3, r


@pytest.mark.parametrize("path,M", [(TCD, 1), (TCD, 4), (TC, 64), (PREFILL, 520)])
@pytest.mark.parametrize("fmt", ["u4", "i5", "f5e2m2"])
def test_bf16_exact_integer_instance(env, fmt, path, M):
    """A in {-1,0,1}, s = 2^-3: every fp32 partial sum is exact in any order, so the bf16 output
    must equal RN_bf16(Y64) bit for bit."""
    P, torch = env
    N, G = 256, 128
    wt_ = parse_wtype(fmt)
    K = 4096 if wt_.kind != "f" else 256
    A, codes, s, z = wl.gen_exact_instance(fmt, M, K, N, G, seed=wl.stable_seed("exact-bf16", fmt, M), j=3)
    A, s = A.astype(np.float32).astype(BF), s.astype(np.float32).astype(BF)
    z = None if z is None else z.astype(np.float32).astype(BF)
    Y, _ = _run(P, torch, fmt, A, codes, s, z, G, path)
    Y64 = matmul_fp64(A, dequant(wt_, codes, s, z, G))
    assert np.array_equal(Y.view(np.uint16), Y64.astype(np.float32).astype(BF).view(np.uint16))


def test_bf16_range_beyond_fp16(env):
    """bf16 activations far outside the fp16 range (|A| ~ 1e6) are handled without overflow: the
    weights are the converted operand, the activations are never narrowed to fp16."""
    P, torch = env
    fmt, M, K, N, G = "i4", 3, 512, 256, 128
    A, codes, s, z = _bf16_problem(fmt, M, K, N, G, "bf16-range")
    A = (A.astype(np.float32) * 1e6).astype(BF)
    s = (s.astype(np.float32) * 1e-3).astype(BF)
    for path in (TCD, TC):
        Y, _ = _run(P, torch, fmt, A, codes, s, z, G, path)
        wd = dequant(parse_wtype(fmt), codes, s, z, G)
        r = tolerance_check(Y, matmul_fp64(A, wd), A, wd, "bf16")
        assert r["ok"], (path, r)
