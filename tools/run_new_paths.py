"""One small call of each round-2 path (for compute-sanitizer): int8 activations (decode and batched),
MX scales + group-32 matmul, the gathered epilogue over two virtual ranks, the row-parallel
reduce-scatter, the batched host-I/O call.  Prints ' ok ' per case when the result is within O7."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2504_12984_b200 as P  # noqa: E402
import workloads as wl  # noqa: E402
from oracle import dequant, matmul_fp64, parse_wtype, tolerance_check, mx_dequant  # noqa: E402
from paper_2504_12984_b200 import dist  # noqa: E402


def dev(x):
    return None if x is None else torch.from_numpy(np.ascontiguousarray(x)).cuda()


def prep(fmt, K, N, codes):
    w = P.wtype(fmt)
    return w, P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, dev(codes)))


def check(name, Y, A, wd):
    r = tolerance_check(Y, matmul_fp64(A, wd), A, wd)
    print(f"{name}: {' ok ' if r['ok'] else 'FAIL'} rel_fro={r['rel_fro']:.2e}", flush=True)


K, N, G = 512, 256, 128
for M in (1, 40):
    fmt = "u4"
    A8 = wl.gen_activations_i8(M, K, 1)
    codes = wl.gen_codes(fmt, K, N, 1)
    s = wl.gen_scales(fmt, K, N, G, 1)
    z = wl.gen_zeros(fmt, K, N, G, 1)
    w, wt = prep(fmt, K, N, codes)
    Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
    ws = P.alloc_workspace(w, M, N, K, G, atype=P.TL_ACT_I8)
    P.tl_matmul(w, M, N, K, G, dev(A8), wt, dev(s), dev(z), Y, ws)
    torch.cuda.synchronize()
    check(f"a8 M={M}", Y.cpu().numpy(), A8, dequant(parse_wtype(fmt), codes, s, z, G))

fmt, M = "f4e2m1", 3
A = wl.gen_activations(M, K, 2)
codes = wl.gen_codes(fmt, K, N, 2)
e = wl.gen_mx_exponents(K, N, 2, 119)
w, wt = prep(fmt, K, N, codes)
sc = P.tl_mx_scales_to_f16(dev(e), 0)
Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
P.tl_matmul(w, M, N, K, 32, dev(A), wt, sc, None, Y, P.alloc_workspace(w, M, N, K, 32))
torch.cuda.synchronize()
check("mx", Y.cpu().numpy(), A, mx_dequant(parse_wtype(fmt), codes, e, 0))

world, fmt, M = 2, "i6", 1
A = wl.gen_activations(M, K, 3)
codes = wl.gen_codes(fmt, K, N, 3)
s = wl.gen_scales(fmt, K, N, G, 3)
Yg = [torch.full((M, N), float("nan"), dtype=torch.float16, device="cuda") for _ in range(world)]
flags = [torch.zeros(world, dtype=torch.int32, device="cuda") for _ in range(world)]
for r in range(world):
    n0, n1 = dist.column_shard(N, world, r)
    w, wt = prep(fmt, K, n1 - n0, codes[:, n0:n1])
    ys, fs = dist.peer_pointers([t.data_ptr() for t in Yg], [t.data_ptr() for t in flags], r, n0)
    P.tl_matmul_gathered(w, M, n1 - n0, K, G, dev(A), wt, dev(s[:, n0:n1]), None, Yg[r][:, n0:], N, ys, fs,
                         P.alloc_workspace(w, M, n1 - n0, K, G))
for r in range(world):
    P.tl_gather_wait(flags[r], world, r, 1)
torch.cuda.synchronize()
check("gathered", Yg[1].cpu().numpy(), A, dequant(parse_wtype(fmt), codes, s, None, G))

parts = [torch.empty((M, N), dtype=torch.float16, device="cuda") for _ in range(world)]
flags = [torch.zeros(world, dtype=torch.int32, device="cuda") for _ in range(world)]
for r in range(world):
    k0, k1 = dist.row_shard(K, world, r, G)
    w, wt = prep(fmt, k1 - k0, N, codes[k0:k1])
    P.tl_matmul(w, M, N, k1 - k0, G, dev(A[:, k0:k1]), wt, dev(s[k0 // G:k1 // G]), None, parts[r],
                P.alloc_workspace(w, M, N, k1 - k0, G))
    _, fs = dist.peer_pointers([0] * world, [f.data_ptr() for f in flags], r, 0)
    P.tl_signal_peers(fs)
ys = []
for r in range(world):
    P.tl_gather_wait(flags[r], world, r, 1)
    n0, n1 = dist.column_shard(N, world, r)
    Y = torch.empty((M, n1 - n0), dtype=torch.float16, device="cuda")
    P.tl_reduce_scatter_peer(dist.reduce_pointers([p.data_ptr() for p in parts], n0), M, n1 - n0, N, Y)
    ys.append(Y)
torch.cuda.synchronize()
check("row-parallel", np.concatenate([y.cpu().numpy() for y in ys], axis=1), A,
      dequant(parse_wtype(fmt), codes, s, None, G))

probs = []
for fmt, M in (("u3", 1), ("i5", 24)):
    codes = wl.gen_codes(fmt, K, N, 4)
    s = wl.gen_scales(fmt, K, N, G, 4)
    z = wl.gen_zeros(fmt, K, N, G, 4)
    w, wt = prep(fmt, K, N, codes)
    probs.append(dict(w=w, group=G, M=M, N=N, K=K, w_t=wt, scales=dev(s), zeros=dev(z),
                      workspace=P.alloc_workspace(w, M, N, K, G), A=wl.gen_activations(M, K, 4), codes=codes, s=s, z=z,
                      fmt=fmt))
A_host = torch.from_numpy(np.concatenate([p["A"].reshape(-1) for p in probs])).pin_memory()
A_dev = torch.empty(A_host.numel(), dtype=torch.float16, device="cuda")
Y_dev = torch.empty(sum(p["M"] * N for p in probs), dtype=torch.float16, device="cuda")
Y_host = torch.empty(Y_dev.numel(), dtype=torch.float16).pin_memory()
P.tl_matmul_batch_hostio(P.batch_items(probs), len(probs), A_host, A_dev, Y_dev, Y_host)
torch.cuda.synchronize()
off = 0
for p in probs:
    check(f"batch {p['fmt']}", Y_host[off:off + p["M"] * N].numpy().reshape(p["M"], N), p["A"],
          dequant(parse_wtype(p["fmt"]), p["codes"], p["s"], p["z"], G))
    off += p["M"] * N
