"""GPU: every rank's column shard computed through ShardedA16WxLinear equals the oracle on
its columns, and the concatenation of the shards equals the single-GPU matmul.
All shards run on the one GPU of the test box (world is simulated; no collective needed)."""

import numpy as np
import pytest

import workloads as wl
from oracle import dequant, matmul_fp64, parse_wtype, tolerance_check

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("fmt", ["u4", "i6"])
def test_sharded_linear_matches_single_gpu(fmt, world):
    import torch

    import paper_2504_12984_b200 as P
    from paper_2504_12984_b200.dist import ShardedA16WxLinear, column_shard
    M, K, N, G = 3, 1024, 2048, 128
    seed = wl.stable_seed("gdist", fmt)
    A = wl.gen_activations(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    z = wl.gen_zeros(fmt, K, N, G, seed)
    Ad = torch.from_numpy(A).cuda()
    parts = []
    for r in range(world):
        n0, n1 = column_shard(N, world, r)
        lin = ShardedA16WxLinear(fmt, K, N, G, torch.from_numpy(np.ascontiguousarray(codes[:, n0:n1])).cuda(),
                                 torch.from_numpy(np.ascontiguousarray(s[:, n0:n1])).cuda(),
                                 None if z is None else torch.from_numpy(np.ascontiguousarray(z[:, n0:n1])).cuda(),
                                 world, r)
        y = lin(Ad).cpu().numpy()
        w = dequant(parse_wtype(fmt), codes[:, n0:n1], s[:, n0:n1], None if z is None else z[:, n0:n1], G)
        assert tolerance_check(y, matmul_fp64(A, w), A, w)["ok"]
        parts.append(y)
    Ys = np.concatenate(parts, axis=1)
    # single-GPU reference through the same library
    wv = P.wtype(fmt)
    wt = P.tl_transform_weights(wv, K, N, P.tl_pack(wv, K, N, torch.from_numpy(codes).cuda()))
    Y1 = torch.empty((M, N), dtype=torch.float16, device="cuda")
    P.tl_matmul(wv, M, N, K, G, Ad, wt, torch.from_numpy(s).cuda(), None if z is None else torch.from_numpy(z).cuda(),
                Y1, P.alloc_workspace(wv, M, N, K, G))
    wfull = dequant(parse_wtype(fmt), codes, s, z, G)
    r = tolerance_check(Ys, Y1.cpu().numpy().astype(np.float64), A, wfull)
    assert r["rel_fro"] < 1e-3
