"""GPU parity for SURVEY §8(f) row f4: int8 activations (A8Wx, reading R24) and
microscaling block scales (reading R25), through the C ABI, against the oracle."""

import numpy as np
import pytest

import workloads as wl
from helpers import GUARD, prepare_weights, to_dev
from oracle import (dequant, e8m0_to_f16_scale, matmul_fp64, mx_dequant, parse_wtype, tolerance_check)

pytestmark = pytest.mark.gpu
GEMV, TC, TCD, PREFILL = 1, 2, 3, 4


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2504_12984_b200 as P
    return P, torch


def _run_a8(P, torch, fmt, A8, codes, s, z, G, path, lda=None, ldy=None, graph=False):
    M, K = A8.shape
    N = codes.shape[1]
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    lda = lda or K
    A_d = torch.full((M, lda), 127, dtype=torch.int8, device="cuda")   # padding past K must not be read
    A_d[:, :K] = to_dev(A8, torch)
    ldy = ldy or N
    Y = torch.full((M, ldy), float("nan"), dtype=torch.float16, device="cuda")
    ws = P.alloc_workspace(w, M, N, K, G, atype=P.TL_ACT_I8)
    P.tl_matmul_ex(w, M, N, K, G, A_d, wt, to_dev(s, torch), to_dev(z, torch), Y, ws, path=path, lda=lda,
                   ldy=ldy)
    torch.cuda.synchronize()
    full = Y.cpu().numpy()
    return full[:, :N], full


@pytest.mark.parametrize("path,M", [(0, 1), (TCD, 1), (TCD, 7), (TCD, 16), (GEMV, 1), (GEMV, 3), (TC, 64),
                                    (TC, 200), (PREFILL, 520)])
@pytest.mark.parametrize("fmt", ["u4", "i3", "u8", "i8", "f6e3m2", "f4e2m1"])
def test_a8_parity(env, fmt, path, M):
    P, torch = env
    K, N, G = 1024, 384, 128
    seed = wl.stable_seed("a8", fmt, M, path)
    A8 = wl.gen_activations_i8(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    z = wl.gen_zeros(fmt, K, N, G, seed, zero_range="full")
    Y, full = _run_a8(P, torch, fmt, A8, codes, s, z, G, path, lda=K + 16, ldy=N + 8)
    assert np.isnan(full[:, N:]).all()
    wd = dequant(parse_wtype(fmt), codes, s, z, G)
    r = tolerance_check(Y, matmul_fp64(A8, wd), A8, wd)
    assert r["ok"], r
    assert r["max_abs_ratio"] <= GUARD, r


@pytest.mark.parametrize("path,M", [(TCD, 1), (TCD, 16), (GEMV, 1), (TC, 48), (PREFILL, 600)])
@pytest.mark.parametrize("fmt", ["u3", "u7", "i5", "i8"])
def test_a8_exact_integer_instance(env, fmt, path, M):
    """Full-range int8 A, s = 2^-8, integer zeros, K = 256: every partial sum is an integer multiple
    of 2^-8 below 128*255*256 = 2^23 in magnitude, so fp32 accumulation is exact in any order and Y
    must equal RN_f16(Y64) bit for bit."""
    P, torch = env
    K, N, G = 256, 256, 128
    seed = wl.stable_seed("a8-exact", fmt, M, path)
    A8 = wl.gen_activations_i8(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = np.full((K // G, N), 2.0 ** -8, dtype=np.float16)
    z = wl.gen_zeros(fmt, K, N, G, seed, zero_range="full")
    wt_ = parse_wtype(fmt)
    Y64 = matmul_fp64(A8, dequant(wt_, codes, s, z, G))
    # precondition of exactness: sum_k |A||q - z| < 2^24 (in units of 2^-8)
    assert (np.abs(A8.astype(np.float64)) @ np.abs(dequant(wt_, codes, s, z, G))).max() * 256 < 2.0 ** 24
    assert np.abs(Y64).max() < 65504
    Y, _ = _run_a8(P, torch, fmt, A8, codes, s, z, G, path)
    assert np.array_equal(Y.view(np.uint16), Y64.astype(np.float16).view(np.uint16))


def test_a8_hostio_and_graph(env):
    """int8 activations through the host-buffer call, and inside a captured CUDA graph."""
    P, torch = env
    fmt, M, K, N, G = "i4", 2, 2048, 512, 128
    seed = wl.stable_seed("a8-hostio")
    A8 = wl.gen_activations_i8(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    s_d = to_dev(s, torch)
    ws = P.alloc_workspace(w, M, N, K, G, atype=P.TL_ACT_I8)
    A_host = torch.from_numpy(A8).pin_memory()
    A_dev = torch.empty((M, K), dtype=torch.int8, device="cuda")
    Y_dev = torch.empty((M, N), dtype=torch.float16, device="cuda")
    Y_host = torch.empty((M, N), dtype=torch.float16).pin_memory()
    P.tl_matmul_hostio(w, M, N, K, G, A_host, A_dev, wt, s_d, None, Y_dev, Y_host, ws)
    torch.cuda.synchronize()
    wd = dequant(parse_wtype(fmt), codes, s, None, G)
    Y64 = matmul_fp64(A8, wd)
    assert tolerance_check(Y_host.numpy(), Y64, A8, wd)["ok"]
    g = torch.cuda.CUDAGraph()
    Y2 = torch.full((M, N), float("nan"), dtype=torch.float16, device="cuda")
    s_ = torch.cuda.Stream()
    with torch.cuda.stream(s_):
        with torch.cuda.graph(g, stream=s_):
            P.tl_matmul(w, M, N, K, G, A_dev, wt, s_d, None, Y2, ws, stream=s_)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(Y2.cpu().numpy().view(np.uint16), Y_host.numpy().view(np.uint16))


@pytest.mark.parametrize("adj", [0, -6, 9])
def test_mx_scales_all_codes(env, adj):
    P, torch = env
    e = torch.arange(256, dtype=torch.int32).to(torch.uint8).cuda()
    got = P.tl_mx_scales_to_f16(e, adj).cpu().numpy()
    want = e8m0_to_f16_scale(np.arange(256, dtype=np.uint8), adj)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.array_equal(got[ok].view(np.uint16), want[ok].view(np.uint16))


@pytest.mark.parametrize("M", [1, 5, 40])
@pytest.mark.parametrize("fmt,adj,center", [("f4e2m1", 0, 119), ("f6e2m3", 0, 120), ("f6e3m2", 0, 117),
                                            ("f8e4m3", 0, 115), ("i8", -6, 121)])
def test_mx_matmul(env, fmt, adj, center, M):
    """MX weights = a kernel element format + group 32 + the converted E8M0 scales; the oracle is the
    MX definition value(code) * 2^(e-127+adj) (oracle/mx.py), independent of the fp16 conversion."""
    P, torch = env
    K, N = 1024, 256
    seed = wl.stable_seed("mx", fmt, M)
    A = wl.gen_activations(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    e = wl.gen_mx_exponents(K, N, seed, center)
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    s_d = P.tl_mx_scales_to_f16(to_dev(e, torch), adj)
    Y = torch.full((M, N), float("nan"), dtype=torch.float16, device="cuda")
    ws = P.alloc_workspace(w, M, N, K, 32)
    P.tl_matmul(w, M, N, K, 32, to_dev(A, torch), wt, s_d, None, Y, ws)
    torch.cuda.synchronize()
    wd = mx_dequant(parse_wtype(fmt), codes, e, adj)
    r = tolerance_check(Y.cpu().numpy(), matmul_fp64(A, wd), A, wd)
    assert r["ok"], r
    assert r["max_abs_ratio"] <= GUARD, r


@pytest.mark.parametrize("adj", [0, -6, -10])
def test_mx_scales_bf16_all_codes(env, adj):
    import ml_dtypes
    from oracle import e8m0_to_bf16_scale
    P, torch = env
    e = torch.arange(256, dtype=torch.int32).to(torch.uint8).cuda()
    got = P.tl_mx_scales_to_bf16(e, adj).view(torch.int16).cpu().numpy().view(ml_dtypes.bfloat16).astype(np.float64)
    want = e8m0_to_bf16_scale(np.arange(256, dtype=np.uint8), adj)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.array_equal(got[ok], want[ok])


@pytest.mark.parametrize("M", [1, 24])
@pytest.mark.parametrize("fmt,adj,center", [("f4e2m1", 0, 119), ("f8e4m3", 0, 115), ("i8", -6, 121)])
def test_mx_matmul_bf16(env, fmt, adj, center, M):
    """MX weights with bf16 activations: bf16 block scales from tl_mx_scales_to_bf16, group 32."""
    import ml_dtypes
    P, torch = env
    BF = ml_dtypes.bfloat16
    K, N = 1024, 256
    seed = wl.stable_seed("mx-bf16", fmt, M)
    A = wl.gen_activations(M, K, seed).astype(np.float32).astype(BF)
    codes = wl.gen_codes(fmt, K, N, seed)
    e = wl.gen_mx_exponents(K, N, seed, center)
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    s_d = P.tl_mx_scales_to_bf16(to_dev(e, torch), adj)
    A_d = torch.from_numpy(np.ascontiguousarray(A).view(np.int16)).cuda().view(torch.bfloat16)
    Y = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    ws = P.alloc_workspace(w, M, N, K, 32, atype=P.TL_ACT_BF16)
    P.tl_matmul(w, M, N, K, 32, A_d, wt, s_d, None, Y, ws)
    torch.cuda.synchronize()
    Yn = Y.view(torch.int16).cpu().numpy().view(BF)
    wd = mx_dequant(parse_wtype(fmt), codes, e, adj)
    r = tolerance_check(Yn, matmul_fp64(A, wd), A, wd, "bf16")
    assert r["ok"], r
