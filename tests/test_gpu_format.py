"""GPU parity of the one-time weight preparation (row a1) and of the unpack/dequant that
every kernel shares: bit-exact against the oracle for all 37 kernel formats."""

import numpy as np
import pytest

import workloads as wl
from helpers import prepare_weights, to_dev
from oracle import all_kernel_formats, dequant, pack, parse_wtype

pytestmark = pytest.mark.gpu
FORMATS = [f.name for f in all_kernel_formats()]


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2504_12984_b200 as P
    return P, torch


@pytest.mark.parametrize("fmt", FORMATS)
def test_pack_bit_exact(env, fmt):
    P, torch = env
    for (K, N) in [(1, 1), (3, 5), (7, 13), (128, 384), (37, 129)]:
        codes = wl.gen_codes(fmt, K, N, wl.stable_seed("pack", fmt, K, N))
        bs = P.tl_pack(P.wtype(fmt), K, N, to_dev(codes, torch)).cpu().numpy()
        assert np.array_equal(bs, pack(codes, parse_wtype(fmt).bits)), (K, N)
        back = P.tl_unpack(P.wtype(fmt), K, N, to_dev(bs, torch)).cpu().numpy()
        assert np.array_equal(back, codes)


@pytest.mark.parametrize("fmt", FORMATS)
def test_transform_roundtrip_and_size(env, fmt):
    P, torch = env
    for (K, N) in [(128, 128), (256, 384), (640, 256)]:
        codes = wl.gen_codes(fmt, K, N, wl.stable_seed("tr", fmt, K, N))
        w, bs, wt = prepare_weights(P, torch, fmt, K, N, codes)
        assert wt.numel() == P.tl_packed_bytes(w, K, N) == P.tl_transformed_bytes(w, K, N)
        back = P.tl_untransform_weights(w, K, N, wt).cpu().numpy()
        assert np.array_equal(back, bs.cpu().numpy())
        # the transform is a true permutation: it is not the identity for multi-tile shapes
        if fmt != "u8" and N > 128:
            assert not np.array_equal(wt.cpu().numpy(), bs.cpu().numpy())


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("G", [32, 64, 128, 256])
def test_dequant_bit_exact(env, fmt, G):
    """GPU tl_dequant(transform(x)) == oracle dequant, bit for bit in fp32 incl. the sign of zero."""
    P, torch = env
    K, N = 512, 256
    seed = wl.stable_seed("deq", fmt, G)
    codes = wl.gen_codes(fmt, K, N, seed)
    rng = np.random.default_rng(seed)
    # scales: random finite fp16 of both signs, normal and subnormal
    raw = rng.integers(0, 0x7C00, size=(K // G, N)).astype(np.uint16) | (rng.integers(0, 2, size=(K // G, N)) << 15).astype(np.uint16)
    scales = raw.view(np.float16)
    zeros = wl.gen_zeros(fmt, K, N, G, seed, zero_range="full")
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    out = P.tl_dequant(w, K, N, G, wt, to_dev(scales, torch), to_dev(zeros, torch)).cpu().numpy()
    ref = dequant(parse_wtype(fmt), codes, scales, zeros, G)
    assert np.array_equal(out.view(np.uint32), ref.astype(np.float32).view(np.uint32))


def test_dequant_per_channel_group(env):
    P, torch = env
    fmt, K, N = "u4", 1024, 128
    codes = wl.gen_codes(fmt, K, N, 5)
    s = wl.gen_scales(fmt, K, N, K, 5)
    z = wl.gen_zeros(fmt, K, N, K, 5)
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    out = P.tl_dequant(w, K, N, K, wt, to_dev(s, torch), to_dev(z, torch)).cpu().numpy()
    assert np.array_equal(out, dequant(parse_wtype(fmt), codes, s, z, K).astype(np.float32))
