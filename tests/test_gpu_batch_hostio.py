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


@pytest.mark.parametrize("act", ["f16", "i8", "bf16"])
def test_batch_hostio_matches_single_calls(env, act):
    P, torch = env
    specs = [("u3", 1, 1024, 384, 128), ("i5", 1, 2048, 256, 128), ("f6e3m2", 16, 1024, 512, 128),
             ("u8", 40, 512, 256, 128), ("i3", 1, 512, 384, 64), ("u4", 3, 1024, 128, 128)]
    import ml_dtypes
    atype = {"f16": P.TL_ACT_F16, "i8": P.TL_ACT_I8, "bf16": P.TL_ACT_BF16}[act]
    adt = {"f16": torch.float16, "i8": torch.int8, "bf16": torch.bfloat16}[act]
    BF = ml_dtypes.bfloat16
    probs, a_parts = [], []
    ws_bytes = 0
    for fmt, M, K, N, G in specs:
        seed = wl.stable_seed("batch", fmt, M, K, N, act)
        A = wl.gen_activations_i8(M, K, seed) if act == "i8" else wl.gen_activations(M, K, seed)
        codes = wl.gen_codes(fmt, K, N, seed)
        s = wl.gen_scales(fmt, K, N, G, seed)
        z = wl.gen_zeros(fmt, K, N, G, seed)
        if act == "bf16":
            A = A.astype(np.float32).astype(BF)
            s = s.astype(np.float32).astype(BF)
            z = None if z is None else z.astype(np.float32).astype(BF)
        w, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
        ws_bytes = max(ws_bytes, P.tl_matmul_workspace_bytes(w, M, N, K, G, atype))
        dv = (lambda x: None if x is None else torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).cuda()
              .view(torch.bfloat16)) if act == "bf16" else (lambda x: to_dev(x, torch))
        probs.append(dict(fmt=fmt, w=w, group=G, M=M, N=N, K=K, w_t=wt, scales=dv(s),
                          zeros=dv(z), A=A, codes=codes, s=s, z=z))
        a_parts.append(A.reshape(-1))
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
    for p in probs:
        p["workspace"] = ws
    A_all = np.concatenate(a_parts)
    A_host = (torch.from_numpy(A_all.view(np.int16)).view(torch.bfloat16) if act == "bf16"
              else torch.from_numpy(A_all)).pin_memory()
    A_dev = torch.empty(A_all.size, dtype=adt, device="cuda")
    y_elems = sum(p["M"] * p["N"] for p in probs)
    ydt = torch.bfloat16 if act == "bf16" else torch.float16
    Y_dev = torch.full((y_elems,), float("nan"), dtype=ydt, device="cuda")
    Y_host = torch.full((y_elems,), float("nan"), dtype=ydt).pin_memory()
    items = P.batch_items(probs)
    P.tl_matmul_batch_hostio(items, len(probs), A_host, A_dev, Y_dev, Y_host, atype=atype)
    torch.cuda.synchronize()
    off = 0
    for p in probs:
        M, N = p["M"], p["N"]
        got = Y_host[off:off + M * N].view(torch.int16).numpy().reshape(M, N)
        Y1 = torch.empty((M, N), dtype=ydt, device="cuda")
        A1 = (torch.from_numpy(np.ascontiguousarray(p["A"]).view(np.int16)).cuda().view(torch.bfloat16)
              if act == "bf16" else torch.from_numpy(p["A"]).cuda())
        P.tl_matmul(p["w"], M, N, p["K"], p["group"], A1, p["w_t"], p["scales"], p["zeros"], Y1, ws)
        torch.cuda.synchronize()
        assert np.array_equal(got, Y1.view(torch.int16).cpu().numpy()), p["fmt"]
        wd = dequant(parse_wtype(p["fmt"]), p["codes"], p["s"], p["z"], p["group"])
        gotv = got.view(BF) if act == "bf16" else got.view(np.float16)
        assert tolerance_check(gotv, matmul_fp64(p["A"], wd), p["A"], wd, "bf16" if act == "bf16" else "f16")["ok"], \
            p["fmt"]
        off += M * N
