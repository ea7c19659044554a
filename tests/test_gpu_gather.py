"""GPU parity for SURVEY §8(f) row f3: the gathered-output column-sharded matmul with the all-gather
fused into the epilogue (include/tilus_b200.h tl_matmul_gathered / tl_gather_wait).

One GPU, `world` virtual ranks in one process: each rank's gathered buffer and flag array are
separate device allocations, and rank r's call stores into the other ranks' buffers through their
device addresses -- the same code path as NVLink peer addresses, minus the link.  The ranks' calls
run one after another on one stream and every wait is issued after all of them, so no kernel ever
waits on another (the waits return at once); the bounded wait itself is checked in a subprocess."""

import os
import subprocess
import sys

import numpy as np
import pytest

import workloads as wl
from helpers import GUARD, prepare_weights, to_dev
from oracle import dequant, matmul_fp64, parse_wtype, tolerance_check

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2504_12984_b200 as P
    from paper_2504_12984_b200 import dist
    return P, torch, dist


def _problem(fmt, M, K, N, G, tag):
    seed = wl.stable_seed("gather", fmt, M, K, N, G, tag)
    return (wl.gen_activations(M, K, seed), wl.gen_codes(fmt, K, N, seed), wl.gen_scales(fmt, K, N, G, seed),
            wl.gen_zeros(fmt, K, N, G, seed, zero_range="full"))


# (world, M, fmt, K, N, G): decode kernel (M <= 16), batched kernel incl. M > 128 chunks (one signal
# per call), prefill (cuBLAS, replicate-and-signal kernel), the CUDA-core GEMV for G = 64
CASES = [(2, 1, "u4", 1024, 512, 128), (4, 1, "i6", 1024, 1024, 128), (2, 16, "u4", 1024, 768, 128),
         (3, 64, "i6", 1024, 768, 128), (2, 300, "f6e3m2", 512, 512, 128), (2, 600, "u4", 512, 512, 128),
         (2, 1, "i3", 512, 512, 64), (8, 4, "u3", 512, 2048, 128)]


@pytest.mark.parametrize("world,M,fmt,K,N,G", CASES)
def test_gathered_virtual_ranks(env, world, M, fmt, K, N, G):
    P, torch, dist = env
    w = P.wtype(fmt)
    Yg = [torch.full((M, N), float("nan"), dtype=torch.float16, device="cuda") for _ in range(world)]
    flags = [torch.zeros(world, dtype=torch.int32, device="cuda") for _ in range(world)]
    shards = []
    for r in range(world):
        n0, n1 = dist.column_shard(N, world, r)
        shards.append((n0, n1))
    for epoch in (1, 2):
        A, codes, s, z = _problem(fmt, M, K, N, G, f"e{epoch}")
        A_d = to_dev(A, torch)
        for r in range(world):
            n0, n1 = shards[r]
            Ns = n1 - n0
            _, _, wt = prepare_weights(P, torch, fmt, K, Ns, np.ascontiguousarray(codes[:, n0:n1]))
            ws = P.alloc_workspace(w, M, Ns, K, G)
            y_peers, f_peers = dist.peer_pointers([t.data_ptr() for t in Yg], [t.data_ptr() for t in flags], r, n0)
            P.tl_matmul_gathered(w, M, Ns, K, G, A_d, wt, to_dev(np.ascontiguousarray(s[:, n0:n1]), torch),
                                 None if z is None else to_dev(np.ascontiguousarray(z[:, n0:n1]), torch),
                                 Yg[r][:, n0:], N, y_peers, f_peers, ws)
        for r in range(world):
            P.tl_gather_wait(flags[r], world, r, epoch)
        torch.cuda.synchronize()
        for r in range(world):
            f = flags[r].cpu().numpy()
            assert f[r] == 0 and all(f[q] == epoch for q in range(world) if q != r), (r, f)
        Y0 = Yg[0].cpu().numpy()
        for r in range(1, world):
            assert np.array_equal(Yg[r].cpu().numpy().view(np.uint16), Y0.view(np.uint16)), r
        wd = dequant(parse_wtype(fmt), codes, s, z, G)
        rr = tolerance_check(Y0, matmul_fp64(A, wd), A, wd)
        assert rr["ok"], rr
        assert rr["max_abs_ratio"] <= GUARD, rr


def test_gather_wait_is_bounded():
    """A peer that never arrives: the wait kernel traps after TL_GATHER_TIMEOUT_MS instead of hanging
    (run in a subprocess: the trap ends that process's CUDA context)."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import torch, paper_2504_12984_b200 as P\n"
            "f = torch.zeros(2, dtype=torch.int32, device='cuda')\n"
            "P.tl_gather_wait(f, 2, 0, 1)\n"
            "try:\n    torch.cuda.synchronize()\n    print('NO-TRAP')\n"
            "except Exception as e:\n    print('TRAPPED', type(e).__name__)\n") % ROOT
    env = dict(os.environ, TL_GATHER_TIMEOUT_MS="200")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, env=env)
    assert "TRAPPED" in p.stdout, (p.stdout, p.stderr[-2000:])


def test_gathered_argument_checks(env):
    P, torch, _ = env
    w = P.wtype("u4")
    L = P._lib
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    x = torch.zeros(4096, dtype=torch.float16, device="cuda")
    VP = L._vp * 8
    bad = L._tl_matmul_gathered(w, 0, 1, 128, 128, 128, x.data_ptr(), 128, x.data_ptr(), x.data_ptr(), None,
                                x.data_ptr(), 128, VP(*[x.data_ptr()] * 8), VP(*[x.data_ptr()] * 8), 8,
                                ws.data_ptr(), ws.numel(), 0, None)
    assert L._tl_status_str(bad).decode() == "TL_EINVAL_SHAPE"
    bad = L._tl_matmul_gathered(w, 0, 1, 128, 128, 128, x.data_ptr(), 128, x.data_ptr(), x.data_ptr(), None,
                                x.data_ptr(), 128, VP(x.data_ptr() + 2), VP(x.data_ptr()), 1,
                                ws.data_ptr(), ws.numel(), 0, None)
    assert L._tl_status_str(bad).decode() == "TL_EALIGN"
    assert L._tl_status_str(L._tl_gather_wait(x.data_ptr(), 9, 0, 1, None)).decode() == "TL_EINVAL_SHAPE"
    assert L._tl_status_str(L._tl_gather_wait(x.data_ptr(), 2, 2, 1, None)).decode() == "TL_EINVAL_SHAPE"
    assert L._tl_gather_wait(x.data_ptr(), 1, 0, 1, None) == 0


@pytest.mark.parametrize("world,M,fmt,K,N,G", [(2, 1, "u4", 1024, 512, 128), (4, 1, "i6", 2048, 1024, 128),
                                              (3, 16, "f6e3m2", 1536, 768, 128), (2, 64, "u3", 1024, 256, 128),
                                              (4, 3, "i3", 2048, 512, 256)])
def test_row_parallel_reduce_scatter_virtual_ranks(env, world, M, fmt, K, N, G):
    """Row-parallel: rank r computes the partial of its K rows; after every rank signalled, each rank
    reduces its column block of all partials.  Bit-exact against the same fixed-order fp32 sum of
    the fp16 partials done in numpy, and within O7 of the oracle."""
    P, torch, dist = env
    w = P.wtype(fmt)
    A, codes, s, z = _problem(fmt, M, K, N, G, "rowpar")
    parts = [torch.full((M, N), float("nan"), dtype=torch.float16, device="cuda") for _ in range(world)]
    flags = [torch.zeros(world, dtype=torch.int32, device="cuda") for _ in range(world)]
    for r in range(world):
        k0, k1 = dist.row_shard(K, world, r, G)
        _, _, wt = prepare_weights(P, torch, fmt, k1 - k0, N, np.ascontiguousarray(codes[k0:k1]))
        ws = P.alloc_workspace(w, M, N, k1 - k0, G)
        zr = None if z is None else to_dev(np.ascontiguousarray(z[k0 // G:k1 // G]), torch)
        P.tl_matmul(w, M, N, k1 - k0, G, to_dev(np.ascontiguousarray(A[:, k0:k1]), torch), wt,
                    to_dev(np.ascontiguousarray(s[k0 // G:k1 // G]), torch), zr, parts[r], ws)
        _, fs = dist.peer_pointers([0] * world, [f.data_ptr() for f in flags], r, 0)
        P.tl_signal_peers(fs)
    ys = []
    for r in range(world):
        P.tl_gather_wait(flags[r], world, r, 1)
        n0, n1 = dist.column_shard(N, world, r)
        Y = torch.full((M, n1 - n0), float("nan"), dtype=torch.float16, device="cuda")
        P.tl_reduce_scatter_peer(dist.reduce_pointers([p.data_ptr() for p in parts], n0), M, n1 - n0, N, Y)
        ys.append(Y)
    torch.cuda.synchronize()
    for r in range(world):
        f = flags[r].cpu().numpy()
        assert f[r] == 0 and all(f[q] == 1 for q in range(world) if q != r), (r, f)
    Yg = np.concatenate([y.cpu().numpy() for y in ys], axis=1)
    ref = np.zeros((M, N), np.float32)
    for p in parts:
        ref = ref + p.cpu().numpy().astype(np.float32)       # rank order, fp32, one rounding
    assert np.array_equal(Yg.view(np.uint16), ref.astype(np.float16).view(np.uint16))
    wd = dequant(parse_wtype(fmt), codes, s, z, G)
    rr = tolerance_check(Yg, matmul_fp64(A, wd), A, wd)
    assert rr["ok"], rr


@pytest.mark.parametrize("act,M", [("bf16", 1), ("bf16", 64), ("i8", 1), ("i8", 40)])
def test_gathered_other_activation_types(env, act, M):
    """The fused gathered epilogue with bf16 activations / outputs and with int8 activations (staged
    to fp16 before the fused kernel), two virtual ranks."""
    import ml_dtypes
    P, torch, dist = env
    world, fmt, K, N, G = 2, "u4", 1024, 512, 128
    w = P.wtype(fmt)
    seed = wl.stable_seed("gather-act", act, M)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    z = wl.gen_zeros(fmt, K, N, G, seed, zero_range="full")
    if act == "bf16":
        BF = ml_dtypes.bfloat16
        A = wl.gen_activations(M, K, seed).astype(np.float32).astype(BF)
        s, z = s.astype(np.float32).astype(BF), z.astype(np.float32).astype(BF)
        dev_t = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).cuda().view(torch.bfloat16)
        ydt, atype, out_kind = torch.bfloat16, P.TL_ACT_BF16, "bf16"
    else:
        A = wl.gen_activations_i8(M, K, seed)
        dev_t = lambda x: to_dev(x, torch)
        ydt, atype, out_kind = torch.float16, P.TL_ACT_I8, "f16"
    Yg = [torch.full((M, N), float("nan"), dtype=ydt, device="cuda") for _ in range(world)]
    flags = [torch.zeros(world, dtype=torch.int32, device="cuda") for _ in range(world)]
    for r in range(world):
        n0, n1 = dist.column_shard(N, world, r)
        _, _, wt = prepare_weights(P, torch, fmt, K, n1 - n0, np.ascontiguousarray(codes[:, n0:n1]))
        ys, fs = dist.peer_pointers([t.data_ptr() for t in Yg], [t.data_ptr() for t in flags], r, n0)
        P.tl_matmul_gathered(w, M, n1 - n0, K, G, dev_t(A), wt, dev_t(s[:, n0:n1]), dev_t(z[:, n0:n1]), Yg[r][:, n0:],
                             N, ys, fs, P.alloc_workspace(w, M, n1 - n0, K, G, atype=atype))
    for r in range(world):
        P.tl_gather_wait(flags[r], world, r, 1)
    torch.cuda.synchronize()
    outs = [(Yg[r].view(torch.int16).cpu().numpy().view(ml_dtypes.bfloat16) if act == "bf16" else Yg[r].cpu().numpy())
            for r in range(world)]
    assert np.array_equal(outs[0].view(np.uint16), outs[1].view(np.uint16))
    wd = dequant(parse_wtype(fmt), codes, s, z, G)
    rr = tolerance_check(outs[0], matmul_fp64(A, wd), A, wd, out_kind)
    assert rr["ok"], rr


def test_fused_classes_single_rank(env):
    """dist.FusedGather / dist.FusedReduceScatter at world size 1 (no peers, no IPC): the plumbing of
    epochs, buffers and waits around tl_matmul_gathered / tl_signal_peers / tl_reduce_scatter_peer."""
    P, torch, dist = env
    fmt, M, K, N, G = "u4", 2, 1024, 512, 128
    A, codes, s, z = _problem(fmt, M, K, N, G, "fused-classes")
    wd = dequant(parse_wtype(fmt), codes, s, z, G)
    Y64 = matmul_fp64(A, wd)
    layer = dist.ShardedA16WxLinear(fmt, K, N, G, to_dev(codes, torch), to_dev(s, torch), to_dev(z, torch), 1, 0)
    fg = dist.FusedGather(M, N, 1, 0)
    for _ in range(3):  # three epochs over two alternating buffers
        Y = fg(layer, to_dev(A, torch))
        torch.cuda.synchronize()
        assert tolerance_check(Y.cpu().numpy(), Y64, A, wd)["ok"]
    rs = dist.FusedReduceScatter(M, N, 1, 0)
    w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    ws = P.alloc_workspace(w, M, N, K, G)
    for _ in range(3):
        Y = rs(w, K, G, to_dev(A, torch), wt, to_dev(s, torch), to_dev(z, torch), ws)
        torch.cuda.synchronize()
        assert tolerance_check(Y.cpu().numpy(), Y64, A, wd)["ok"]
