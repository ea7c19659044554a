"""Shared test plumbing: build one problem from the seeded generators, run the CUDA path
through the C-ABI binding and the oracle on the SAME inputs."""

from __future__ import annotations

import numpy as np

import workloads as wl


def make_problem(fmt: str, M: int, K: int, N: int, G: int, seed_tag: str = "", zero_range: str = "mid",
                 with_zeros: bool = True):
    seed = wl.stable_seed("parity", fmt, M, K, N, G, seed_tag)
    A = wl.gen_activations(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    scales = wl.gen_scales(fmt, K, N, G, seed)
    zeros = wl.gen_zeros(fmt, K, N, G, seed, zero_range=zero_range) if with_zeros else None
    return A, codes, scales, zeros


def to_dev(x, torch):
    return None if x is None else torch.from_numpy(np.ascontiguousarray(x)).cuda()


def prepare_weights(P, torch, fmt: str, K: int, N: int, codes: np.ndarray):
    """codes (host) -> device bitstream (tl_pack) -> transformed (tl_transform_weights)."""
    w = P.wtype(fmt)
    codes_d = to_dev(codes, torch)
    bs = P.tl_pack(w, K, N, codes_d)
    wt = P.tl_transform_weights(w, K, N, bs)
    return w, bs, wt


def run_matmul(P, torch, fmt, A, codes, scales, zeros, G, path=0, splits=0, wt=None, ldy=None, poison=True,
               lda=None):
    """Runs tl_matmul_ex.  ldy > N: Y rows are NaN-poisoned past N (nothing may be written there);
    lda > K: A rows are padded with NaN past K (nothing may be read there)."""
    M, K = A.shape
    N = codes.shape[1]
    w = P.wtype(fmt)
    if wt is None:
        _, _, wt = prepare_weights(P, torch, fmt, K, N, codes)
    s_d, z_d = to_dev(scales, torch), to_dev(zeros, torch)
    lda = lda or K
    A_d = torch.full((M, lda), float("nan"), dtype=torch.float16, device="cuda")
    A_d[:, :K] = to_dev(A, torch)
    ldy = ldy or N
    Y = torch.full((M, ldy), float("nan") if poison else 0.0, dtype=torch.float16, device="cuda")
    ws = P.alloc_workspace(w, M, N, K, G)
    P.tl_matmul_ex(w, M, N, K, G, A_d, wt, s_d, z_d, Y, ws, path=path, splits=splits, lda=lda, ldy=ldy)
    torch.cuda.synchronize()
    return Y[:, :N].cpu().numpy(), Y.cpu().numpy(), ws


# the element-wise O7 bound (1e-2) is ~500x looser than what fp32 accumulation
# with an fp16 output achieves (~1.5e-5); the GPU tests also hold max|err|/(|A_m||w_n|) to this
# internal regression guard so a 100x local error regression cannot hide under O7.
GUARD = 1e-3


def check_oracle(fmt, A, codes, scales, zeros, G, Y):
    """O7 against the fp64 oracle on the same inputs, plus the internal regression guard."""
    from oracle import dequant, matmul_fp64, parse_wtype, tolerance_check
    w = dequant(parse_wtype(fmt), codes, scales, zeros, G)
    r = tolerance_check(Y, matmul_fp64(A, w), A, w)
    assert r["ok"], r
    assert r["max_abs_ratio"] <= GUARD, r
    return r
