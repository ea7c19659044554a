"""GPU parity of the batched tcgen05 path (tc2, M > 16) and of the edge cases every path shares,
against the fp64 oracle (O6/O7 + the App. F regression guard, helpers.check_oracle).

tc2 is the "Tensor Cores for 16 or more tokens" regime of PAPER.md:546: MMA-N = the batch tile
NB = 16..128 (instruction descriptor N, activation box rows, descriptor block stride NB*8, NB
accumulator columns and the multi-group epilogue all depend on it) and M > 128 is chunked.
"""

import numpy as np
import pytest

import workloads as wl
from helpers import check_oracle, make_problem, prepare_weights, run_matmul, to_dev
from oracle import all_kernel_formats, dequant, matmul_cols_fp64, matmul_fp64, parse_wtype, tolerance_check

pytestmark = pytest.mark.gpu
GEMV, TC, TCD = 1, 2, 3
BATCHES = [17, 31, 32, 48, 64, 100, 128, 129, 200, 256]
EIGHT = ["u1", "u4", "i3", "i8", "u8", "f4e2m1", "f6e3m2", "f8e4m3"]


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2504_12984_b200 as P
    return P, torch


@pytest.mark.parametrize("path", [TC, 0], ids=["tc", "auto"])
@pytest.mark.parametrize("M", BATCHES)
@pytest.mark.parametrize("fmt", EIGHT)
def test_batched_parity(env, fmt, M, path):
    P, torch = env
    K, N, G = 512, 384, 128 if fmt != "i3" else 64
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="batched")
    Y, full, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=path, ldy=N + 8)
    assert np.isnan(full[:, N:]).all()
    check_oracle(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("fmt", [f.name for f in all_kernel_formats()])
def test_tc_all_formats_m128(env, fmt):
    P, torch = env
    M, K, N, G = 128, 1024, 256, 128
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="m128")
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=TC)
    check_oracle(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("M", [64, 128, 160])
@pytest.mark.parametrize("fmt", ["u1", "u4", "i3", "u8", "i8", "f4e2m1", "f6e3m2", "f8e4m3", "f5e1m3"])
def test_tc_exact_integer_instance_bit_exact(env, fmt, M):
    """A in {-1,0,1}, s = 2^-3: every fp32 partial sum is exact in any order, so Y must equal
    RN_f16(Y64) bit for bit -- catches indexing / descriptor bugs the tolerance would hide."""
    P, torch = env
    N, G = 256, 128
    wt_ = parse_wtype(fmt)
    K = 8192 if wt_.kind != "f" else (4096 if wt_.exp <= 3 else 256)
    A, codes, s, z = wl.gen_exact_instance(fmt, M, K, N, G, seed=wl.stable_seed("exact-tc", fmt, M), j=3)
    w = dequant(wt_, codes, s, z, G)
    grid = 2.0 ** -3 * (2.0 ** (1 - ((1 << (wt_.exp - 1)) - 1) - wt_.man) if wt_.kind == "f" else 1.0)
    assert (np.abs(A).astype(np.float64) @ np.abs(w)).max() < 2.0 ** 24 * grid
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=TC)
    assert np.array_equal(Y.view(np.uint16), matmul_fp64(A, w).astype(np.float16).view(np.uint16))


@pytest.mark.parametrize("path", [GEMV, TC, TCD, 0], ids=["gemv", "tc", "tcd", "auto"])
@pytest.mark.parametrize("M", [1, 5, 16, 40])
@pytest.mark.parametrize("fmt", ["u3", "i5", "f6e3m2"])
def test_strided_activations(env, fmt, M, path):
    """lda > K: A rows padded with NaN past K; the kernels must read exactly K elements per row."""
    P, torch = env
    if path == GEMV and M > 16:
        M = 33  # the GEMV path runs 16 rows per launch: also exercise its row chunking
    K, N, G = 1024, 256, 128
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="lda")
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=path, lda=K + 72)
    check_oracle(fmt, A, codes, s, z, G, Y)


def _signed_subnormal_scales(shape, seed):
    """Scales with random sign, a quarter of them fp16 subnormals (|s| < 2^-14), the rest normal."""
    rng = np.random.Generator(np.random.PCG64(seed))
    mag = rng.uniform(0.5, 1.5, size=shape) * 0.02
    sub = rng.random(shape) < 0.25
    mag = np.where(sub, rng.integers(1, 1024, size=shape) * 2.0 ** -24, mag)
    sgn = np.where(rng.random(shape) < 0.5, -1.0, 1.0)
    return (sgn * mag).astype(np.float16)


@pytest.mark.parametrize("path", [GEMV, TC, TCD], ids=["gemv", "tc", "tcd"])
@pytest.mark.parametrize("fmt", ["u4", "i6", "f5e2m2", "u8"])
def test_negative_and_subnormal_scales(env, fmt, path):
    P, torch = env
    for M in ([1, 16] if path != TC else [24, 128]):
        K, N = 1024, 256
        G = 128 if path == TCD else 64
        A, codes, _, z = make_problem(fmt, M, K, N, G, seed_tag="negsub")
        s = _signed_subnormal_scales((K // G, N), wl.stable_seed("negsub", fmt, M))
        assert (s < 0).any() and (np.abs(s.astype(np.float32)) < 2.0 ** -14).any()
        Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=path)
        check_oracle(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("M", [17, 33, 130])
def test_gemv_row_chunking(env, M):
    """The CUDA-core path handles 16 rows per launch; M > 16 is chunked inside tl_matmul_ex."""
    P, torch = env
    fmt, K, N, G = "u4", 512, 256, 64
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="gemv-chunk")
    Y, full, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=GEMV, ldy=N + 16)
    assert np.isnan(full[:, N:]).all()
    check_oracle(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("M", [129, 257, 300])
def test_tc_m_chunks_ragged_ldy(env, M):
    """M > 128 is chunked by 128 rows (the last chunk ragged): every row written, nothing past N."""
    P, torch = env
    fmt, K, N, G = "i5", 1024, 384, 128
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="mchunk")
    Y, full, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=TC, ldy=N + 64)
    assert not np.isnan(Y).any() and np.isnan(full[:, N:]).all()
    check_oracle(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
@pytest.mark.parametrize("M", [1, 16, 64])
def test_transform_then_matmul_without_host_sync(env, M, graph):
    """The weights, scales and zeros are produced on the device by the kernels immediately
    preceding tl_matmul on the same stream (tl_pack -> tl_transform_weights -> a scale copy),
    with no host synchronisation in between: the matmul must see the fresh values (PDL rules:
    only griddepcontrol.wait guarantees the predecessor's writes are visible)."""
    P, torch = env
    fmt, K, N, G = "u4", 2048, 512, 128
    w = P.wtype(fmt)
    ws = torch.zeros(P.tl_matmul_workspace_bytes(w, M, N, K, G), dtype=torch.uint8, device="cuda")
    codes_d = torch.zeros((K, N), dtype=torch.uint8, device="cuda")
    bs = torch.zeros(P.tl_packed_bytes(w, K, N), dtype=torch.uint8, device="cuda")
    wt = torch.zeros(P.tl_transformed_bytes(w, K, N), dtype=torch.uint8, device="cuda")
    s_src = torch.zeros((K // G, N), dtype=torch.float16, device="cuda")
    z_src = torch.zeros((K // G, N), dtype=torch.float16, device="cuda")
    s_d, z_d = torch.zeros_like(s_src), torch.zeros_like(z_src)
    A_d = torch.zeros((M, K), dtype=torch.float16, device="cuda")
    Y = torch.zeros((M, N), dtype=torch.float16, device="cuda")

    def prepare_and_run():
        P.tl_pack(w, K, N, codes_d, bs)
        P.tl_transform_weights(w, K, N, bs, wt)
        s_d.copy_(s_src)
        z_d.copy_(z_src)
        P.tl_matmul(w, M, N, K, G, A_d, wt, s_d, z_d, Y, ws)

    g = None
    if graph:
        prepare_and_run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            prepare_and_run()
    for it in range(3):
        A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag=f"nosync{it}")
        # all new inputs land first (host->device), then the device-side chain runs
        codes_d.copy_(to_dev(codes, torch))
        s_src.copy_(to_dev(s, torch))
        z_src.copy_(to_dev(z, torch))
        A_d.copy_(to_dev(A, torch))
        if g is not None:
            g.replay()
        else:
            prepare_and_run()
        torch.cuda.synchronize()
        check_oracle(fmt, A, codes, s, z, G, Y.cpu().numpy())


@pytest.mark.slow
@pytest.mark.parametrize("M", [64, 128])
@pytest.mark.parametrize("fmt,layer", [("u4", "gate_up"), ("i5", "down"), ("f6e3m2", "qkv"), ("u3", "o")])
def test_full_size_sampled_columns_batched(env, fmt, layer, M):
    """Llama-3.3-70B layer shapes at the bench's batched launch configuration; oracle on a column
    sample (first/last column of every 128-tile and of every 8-way shard + random)."""
    P, torch = env
    K, N = wl.LLAMA33_70B[layer]
    G = 128
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="full")
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G)
    cols = wl.sample_columns(N)
    zc = None if z is None else z[:, cols]
    Y64 = matmul_cols_fp64(parse_wtype(fmt), A, codes[:, cols], s[:, cols], zc, G)
    w = dequant(parse_wtype(fmt), codes[:, cols], s[:, cols], zc, G)
    r = tolerance_check(Y[:, cols], Y64, A, w)
    assert r["ok"] and r["max_abs_ratio"] <= 1e-3, r


@pytest.mark.parametrize("path", [GEMV, TCD, 0], ids=["gemv", "tcd", "auto"])
@pytest.mark.parametrize("K,G", [(40960, 128), (2048, 256), (2048, 2048), (1536, 384)])
@pytest.mark.parametrize("fmt", ["u3", "i6", "f6e3m2", "u8"])
def test_decode_configurations(env, fmt, K, G, path):
    """M = 1 beyond the common shape: K*2 > 64 KB (the activation row no longer fits the decode
    kernels' shared-memory stash: tcd runs its 16-row configuration, the CUDA-core GEMV falls back
    to the staged kernel) and groups spanning several 128-k tiles (G = 256, 384, K)."""
    P, torch = env
    N = 256
    A, codes, s, z = make_problem(fmt, 1, K, N, G, seed_tag="decode-cfg")
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=path)
    check_oracle(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("splits", [1, 2, 5, 40, 148])
@pytest.mark.parametrize("fmt", ["u3", "f6e3m2"])
def test_gemv_m1_stream_k(env, fmt, splits):
    """The M = 1 CUDA-core kernel under every stream-K partition: n-tile segments shared by several
    CTAs, stages that span two n-tiles (their scale / zero boxes come from two n-tiles)."""
    P, torch = env
    K, N, G = 1536, 640, 128
    A, codes, s, z = make_problem(fmt, 1, K, N, G, seed_tag="gv1-sk")
    Y, full, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=GEMV, splits=splits, ldy=N + 8)
    assert np.isnan(full[:, N:]).all()
    check_oracle(fmt, A, codes, s, z, G, Y)


PREFILL = 4


@pytest.mark.parametrize("M", [200, 512, 700])
@pytest.mark.parametrize("fmt", ["u1", "u4", "i3", "i8", "f4e2m1", "f6e3m2", "u8"])
def test_prefill_parity(env, fmt, M):
    """Large-M path: the weight decoded to fp16 by the library, then a dense
    f16 x f16 GEMM with fp32 accumulation; ragged M, ldy > N, a group size below 128 for one
    format."""
    P, torch = env
    K, N = 1024, 384
    G = 64 if fmt == "i3" else 128
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="prefill")
    Y, full, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=PREFILL, ldy=N + 8)
    assert np.isnan(full[:, N:]).all()
    check_oracle(fmt, A, codes, s, z, G, Y)


def test_prefill_chunks_and_auto_dispatch(env):
    """N larger than one decode chunk (several dq16 + GEMM rounds) through the automatic dispatch
    at M = 640 (>= the prefill threshold)."""
    P, torch = env
    fmt, M, K, N, G = "u4", 640, 8192, 4608, 128
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="prefill-chunks")
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G)
    assert P.tl_matmul_plan(P.wtype(fmt), M, N, K, G)[0] == PREFILL
    cols = wl.sample_columns(N)
    Y64 = matmul_cols_fp64(parse_wtype(fmt), A, codes[:, cols], s[:, cols], z[:, cols], G)
    w = dequant(parse_wtype(fmt), codes[:, cols], s[:, cols], z[:, cols], G)
    r = tolerance_check(Y[:, cols], Y64, A, w)
    assert r["ok"] and r["max_abs_ratio"] <= 1e-3, r


@pytest.mark.parametrize("fmt,M,K,N", [("u3", 128, 2048, 1280), ("i5", 64, 4096, 1024), ("f6e3m2", 100, 1024, 2560),
                                       ("u8", 128, 8192, 512)])
def test_distributed_reduction_same_bits_as_last_arriver(env, fmt, M, K, N):
    """The batched kernel's distributed stream-K reduction (aligned split grids, every contributor
    reduces 1/S of the tile) sums the contributors in the same CTA order as the last-arriver
    reduction (TL_TC2_DIST=0): the outputs must be bit-identical, and identical run to run."""
    import os
    P, torch = env
    G = 128
    A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="dist")
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    outs = []
    for dist in ("1", "0", "1"):
        old = os.environ.get("TL_TC2_DIST")
        os.environ["TL_TC2_DIST"] = dist
        try:
            Y, _, ws = run_matmul(P, torch, fmt, A, codes, s, z, G, path=2, wt=wt)
        finally:
            if old is None:
                os.environ.pop("TL_TC2_DIST", None)
            else:
                os.environ["TL_TC2_DIST"] = old
        assert int(ws[: 64 * 1024].view(torch.int32).abs().sum().item()) == 0  # semaphores back at zero
        outs.append(Y.view(np.uint16).copy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    check_oracle(fmt, A, codes, s, z, G, outs[0].view(np.float16))
