"""GPU parity of the decode kernel (tcd.cuh, M = 1 decode configuration) on every int / uint format:
three shapes incl. G = 256 and G = K, full-range zero points, activations spanning the whole fp16
range within one k-tile (an all-zero tile, +-2^-24, 6e4 next to 1e-3), and exact-integer instances
bit-exact under four stream-K splits."""

import numpy as np
import pytest

import workloads as wl
from helpers import check_oracle, run_matmul
from oracle import dequant, matmul_fp64, parse_wtype

pytestmark = pytest.mark.gpu
TCD = 3
INTS = [f"u{b}" for b in range(1, 9)] + [f"i{b}" for b in range(1, 9)]


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2504_12984_b200 as P
    return P, torch


@pytest.mark.parametrize("fmt", INTS)
@pytest.mark.parametrize("K,N,G", [(1024, 384, 128), (2048, 256, 256), (640, 512, 640)])
def test_i8_decode_parity(env, fmt, K, N, G):
    P, torch = env
    seed = wl.stable_seed("rawdec", fmt, K, N, G)
    A = wl.gen_activations(1, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    z = wl.gen_zeros(fmt, K, N, G, seed, zero_range="full")
    Y, full, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=TCD, ldy=N + 8)
    assert np.isnan(full[:, N:]).all()
    check_oracle(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("fmt", ["u4", "u8", "i5", "i8"])
def test_i8_decode_dynamic_range(env, fmt):
    """Tiles whose activations span the whole fp16 range (one element near 6e4 next to subnormals,
    an all-zero tile, a tile of +-2^-24): the error stays far inside O7."""
    P, torch = env
    K, N, G = 1024, 256, 128
    seed = wl.stable_seed("rawdr", fmt)
    A = wl.gen_activations(1, K, seed).astype(np.float32)
    A[0, 0:128] *= 1e-3
    A[0, 5] = 60000.0
    A[0, 128:256] = 0.0
    A[0, 256:384] = np.where(np.arange(128) % 2 == 0, 2.0 ** -24, -(2.0 ** -24))
    A[0, 384:512] *= 2.0 ** -14
    A = A.astype(np.float16)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    z = wl.gen_zeros(fmt, K, N, G, seed, zero_range="full")
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=TCD)
    check_oracle(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("fmt", ["u1", "u3", "u7", "u8", "i2", "i5", "i8"])
@pytest.mark.parametrize("splits", [0, 1, 7, 33])
def test_i8_decode_exact_integer_instance(env, fmt, splits):
    """A in {-1, 0, 1}, s = 2^-3, K = 4096: every per-tile sum is an exact integer and every partial
    sum an exact multiple of 2^-3 below 2^21, so Y must equal RN_f16(Y64) bit for bit under any
    stream-K split."""
    P, torch = env
    K, N, G = 4096, 384, 128
    A, codes, s, z = wl.gen_exact_instance(fmt, 1, K, N, G, seed=wl.stable_seed("rawexact", fmt), j=3)
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=TCD, splits=splits)
    Y64 = matmul_fp64(A, dequant(parse_wtype(fmt), codes, s, z, G))
    assert np.array_equal(Y.view(np.uint16), Y64.astype(np.float16).view(np.uint16))
