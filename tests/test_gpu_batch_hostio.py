"""GPU: tl_matmul_batch_hostio (one H2D of all items' activations, the items' matmuls, one D2H of all
outputs) returns exactly what the per-item tl_matmul calls return, for a mix of formats, shapes,
batch sizes (decode, batched and CUDA-core paths) and activation types, with one shared workspace."""

import numpy as np
import pytest

import workloads as wl
from helpers import prepare_weights, to_dev
from oracle import dequant, matmul_fp64, parse_wtype, tolerance_check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2504_12984_b200 as P
    return P, torch


@pytest.mark.parametrize("act", ["f16", "i8"])
def test_batch_hostio_matches_single_calls(env, act):
    P, torch = env
    specs = [("u3", 1, 1024, 384, 128), ("i5", 1, 2048, 256, 128), ("f6e3m2", 16, 1024, 512, 128),
             ("u8", 40, 512, 256, 128), ("i3", 1, 512, 384, 64), ("u4", 3, 1024, 128, 128)]
    atype = P.TL_ACT_I8 if act == "i8" else P.TL_ACT_F16
    adt = torch.int8 if act == "i8" else torch.float16
    probs, a_parts = [], []
    ws_bytes = 0
    for fmt, M, K, N, G in specs:
        seed = wl.stable_seed("batch", fmt, M, K, N, act)
        A = wl.gen_activations_i8(M, K, seed) if act == "i8" else wl.gen_activations(M, K, seed)
        codes = wl.gen_codes(fmt, K, N, seed)
        s = wl.gen_scales(fmt, K, N, G, seed)
        z = wl.gen_zeros(fmt, K, N, G, seed)
        w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
        ws_bytes = max(ws_bytes, P.tl_matmul_workspace_bytes(w, M, N, K, G, atype))
        probs.append(dict(fmt=fmt, w=w, group=G, M=M, N=N, K=K, w_t=wt, scales=to_dev(s, torch),
                          zeros=to_dev(z, torch), A=A, codes=codes, s=s, z=z))
        a_parts.append(A.reshape(-1))
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
    for p in probs:
        p["workspace"] = ws
    A_all = np.concatenate(a_parts)
    A_host = torch.from_numpy(A_all).pin_memory()
    A_dev = torch.empty(A_all.size, dtype=adt, device="cuda")
    y_elems = sum(p["M"] * p["N"] for p in probs)
    Y_dev = torch.full((y_elems,), float("nan"), dtype=torch.float16, device="cuda")
    Y_host = torch.full((y_elems,), float("nan"), dtype=torch.float16).pin_memory()
    items = P.batch_items(probs)
    P.tl_matmul_batch_hostio(items, len(probs), A_host, A_dev, Y_dev, Y_host, atype=atype)
    torch.cuda.synchronize()
    off = 0
    for p in probs:
        M, N = p["M"], p["N"]
        got = Y_host[off:off + M * N].numpy().reshape(M, N)
        Y1 = torch.empty((M, N), dtype=torch.float16, device="cuda")
        P.tl_matmul(p["w"], M, N, p["K"], p["group"], torch.from_numpy(p["A"]).cuda(), p["w_t"], p["scales"],
                    p["zeros"], Y1, ws)
        torch.cuda.synchronize()
        assert np.array_equal(got.view(np.uint16), Y1.cpu().numpy().view(np.uint16)), p["fmt"]
        wd = dequant(parse_wtype(p["fmt"]), p["codes"], p["s"], p["z"], p["group"])
        assert tolerance_check(got, matmul_fp64(p["A"], wd), p["A"], wd)["ok"], p["fmt"]
        off += M * N
