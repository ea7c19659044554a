"""GPU parity of the hot path tl_matmul (rows a2-a11) against the fp64 oracle.

Tolerance (north star / oracle O7): rel-Frobenius <= 1e-3 and |err| <= 1e-2*||A_m||*||w_n||.
Exact-integer instances (A in {-1,0,1}, s = 2^-j) must match RN_f16(Y64) bit for bit.
"""

import numpy as np
import pytest

import workloads as wl
from helpers import check_oracle, make_problem, prepare_weights, run_matmul, to_dev
from oracle import all_kernel_formats, dequant, matmul_cols_fp64, matmul_fp64, parse_wtype, tolerance_check

pytestmark = pytest.mark.gpu
FORMATS = [f.name for f in all_kernel_formats()]
PATHS = {"gemv": 1, "tc": 2, "tcd": 3}


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2504_12984_b200 as P
    return P, torch


_check = check_oracle


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("fmt", FORMATS)
def test_matmul_all_formats(env, fmt, path):
    P, torch = env
    for (M, K, N, G) in [(1, 512, 384, 128), (3, 640, 256, 64), (16, 256, 128, 32)]:
        A, codes, s, z = make_problem(fmt, M, K, N, G)
        Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=PATHS[path])
        _check(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("fmt", ["u1", "u4", "i3", "u8", "i8", "f4e2m1", "f6e3m2", "f8e4m3", "f5e1m3"])
def test_matmul_exact_integer_instance_bit_exact(env, fmt, path):
    P, torch = env
    M, N, G = 4, 256, 128
    wt_ = parse_wtype(fmt)
    # floats: keep every partial sum exact in fp32 (values are multiples of 2^(1-bias-M))
    K = 8192 if wt_.kind != "f" else (4096 if wt_.exp <= 3 else 256)
    A, codes, s, z = wl.gen_exact_instance(fmt, M, K, N, G, seed=wl.stable_seed("exact", fmt), j=3)
    w = dequant(wt_, codes, s, z, G)
    # precondition: every partial sum, in ANY order, is a multiple of the value grid and
    # below 2^24 grid steps, so fp32 accumulation is exact whatever the kernel's order
    grid = 2.0 ** -3 * (2.0 ** (1 - ((1 << (wt_.exp - 1)) - 1) - wt_.man) if wt_.kind == "f" else 1.0)
    assert (np.abs(A).astype(np.float64) @ np.abs(w)).max() < 2.0 ** 24 * grid
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=PATHS[path])
    Y64 = matmul_fp64(A, w)
    assert np.array_equal(Y.view(np.uint16), Y64.astype(np.float16).view(np.uint16))


@pytest.mark.parametrize("path", list(PATHS))
def test_matmul_grid_sweep_stream_k(env, path):
    """Every stream-K partition (1 CTA ... one CTA per tile) is within O7 of the oracle.  Different
    partitions sum the K range in different orders, so they agree within tolerance, not in bits
    (run-to-run identity of ONE partition is test_matmul_deterministic_and_fully_written)."""
    P, torch = env
    fmt, M, K, N, G = "u4", 2, 1024, 512, 128
    A, codes, s, z = make_problem(fmt, M, K, N, G)
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    for grid in [1, 3, 5, 7, 8, 13, 31, 32]:
        Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=PATHS[path], splits=grid, wt=wt)
        _check(fmt, A, codes, s, z, G, Y)


@pytest.mark.parametrize("path", list(PATHS))
def test_matmul_deterministic_and_fully_written(env, path):
    P, torch = env
    fmt, M, K, N, G = "i5", 5, 2048, 1024, 128
    A, codes, s, z = make_problem(fmt, M, K, N, G)
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    outs = []
    for _ in range(3):
        Y, full, _ = run_matmul(P, torch, fmt, A, codes, s, z, G, path=PATHS[path], wt=wt, ldy=N + 64)
        assert not np.isnan(Y).any()                  # every element written (NaN poison)
        assert np.isnan(full[:, N:]).all()            # nothing written past N (ldy > N)
        outs.append(Y.view(np.uint16).copy())
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    _check(fmt, A, codes, s, z, G, outs[0].view(np.float16))


@pytest.mark.parametrize("path", list(PATHS))
def test_matmul_no_zeros_and_per_channel(env, path):
    P, torch = env
    fmt, M, K, N = "u3", 2, 1024, 256
    A, codes, s, _ = make_problem(fmt, M, K, N, K, with_zeros=False)
    Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, None, K, path=PATHS[path])
    _check(fmt, A, codes, s, None, K, Y)


@pytest.mark.parametrize("path", list(PATHS))
def test_workspace_reuse_across_shapes(env, path):
    """Semaphores self-reset: one zeroed workspace serves many calls."""
    P, torch = env
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    for (fmt, M, K, N) in [("u4", 1, 1024, 256), ("i6", 3, 512, 640), ("f6e3m2", 2, 2048, 128)]:
        A, codes, s, z = make_problem(fmt, M, K, N, 128)
        w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
        Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
        for grid in [0, 7]:
            P.tl_matmul_ex(w, M, N, K, 128, to_dev(A, torch), wt, to_dev(s, torch), to_dev(z, torch), Y, ws,
                           path=PATHS[path], splits=grid)
            _check(fmt, A, codes, s, z, 128, Y.cpu().numpy())
    assert int(ws[:65536].view(torch.int32).abs().sum()) == 0


@pytest.mark.slow
@pytest.mark.parametrize("fmt,layer", [("u4", "gate_up"), ("i5", "down"), ("f6e3m2", "qkv"), ("u3", "o")])
def test_matmul_full_size_sampled_columns(env, fmt, layer):
    """Llama-3.3-70B layer shapes at the bench's launch configuration; oracle on a column sample."""
    P, torch = env
    K, N = wl.LLAMA33_70B[layer]
    G = 128
    for M in [1, 16]:
        A, codes, s, z = make_problem(fmt, M, K, N, G, seed_tag="full")
        Y, _, _ = run_matmul(P, torch, fmt, A, codes, s, z, G)
        cols = wl.sample_columns(N)
        Y64 = matmul_cols_fp64(parse_wtype(fmt), A, codes[:, cols], s[:, cols], None if z is None else z[:, cols], G)
        w = dequant(parse_wtype(fmt), codes[:, cols], s[:, cols], None if z is None else z[:, cols], G)
        r = tolerance_check(Y[:, cols], Y64, A, w)
        assert r["ok"], r


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("fmt", ["u4", "i5", "f6e3m2"])
def test_dependent_chain_programmatic_launch(env, fmt, graph):
    """The decode path is launched with programmatic dependent launch: its weight stream starts
    before the previous kernel finishes, everything that reads A or writes Y / the workspace waits
    (griddepcontrol.wait).  Chain Y1 = A W1, Y2 = Y1 W2, Y3 = Y2 W3 back to back on one stream
    (eager and captured in a CUDA graph), with one shared workspace: each step must match the
    oracle applied to the GPU's own previous output."""
    P, torch = env
    M, K, G = 1, 2048, 128
    A, _, _, _ = make_problem(fmt, M, K, K, G, seed_tag="chain")
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    layers = []
    for i in range(3):
        _, codes, s, z = make_problem(fmt, M, K, K, G, seed_tag=f"chain{i}")
        w, _, wt = prepare_weights(P, torch, fmt, K, K, codes)
        layers.append((codes, s, z, w, wt, to_dev(s, torch), to_dev(z, torch)))
    X = [to_dev(A, torch)] + [torch.full((M, K), float("nan"), dtype=torch.float16, device="cuda") for _ in range(3)]

    def chain():
        for i, (_, _, _, w, wt, s_d, z_d) in enumerate(layers):
            P.tl_matmul(w, M, K, K, G, X[i], wt, s_d, z_d, X[i + 1], ws)

    if graph:
        chain()
        torch.cuda.synchronize()
        for x in X[1:]:
            x.fill_(float("nan"))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            chain()
        g.replay()
    else:
        chain()
    torch.cuda.synchronize()
    for i, (codes, s, z, *_rest) in enumerate(layers):
        Ain = X[i].cpu().numpy().astype(np.float16)
        Yi = X[i + 1].cpu().numpy()
        assert not np.isnan(Yi).any()
        _check(fmt, Ain, codes, s, z, G, Yi)
    assert int(ws[:65536].view(torch.int32).abs().sum()) == 0
