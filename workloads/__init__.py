"""Seeded synthetic inputs and the BASELINE.json workload shapes.

Shared by the tests (which feed the oracle and the CUDA path the SAME arrays)
and by bench.py.  This module holds none of the method's arithmetic: it only
draws random codes / scales / zeros / activations and lists layer shapes.  It
imports neither ``oracle`` nor ``paper_2504_12984_b200``.

Input recipe:
  * codes   uniform over all 2^b codes (floats therefore include +-0,
            subnormals and the top binade);
  * scales  fp16, U[0.5, 1.5) * 0.02 / 2^(b-1) per (group, column) -- an
            LLM-like weight magnitude that needs no value table;
  * zeros   (unsigned formats only) integers uniform in {2^(b-1)-1, 2^(b-1)},
            or full range [0, 2^b-1] with ``zero_range="full"``;
  * A       fp16 ~ N(0, 1);
  * "exact-integer instance": A in {-1, 0, 1}, s = 2^-j, integer zeros, so
            every partial sum is a multiple of 2^-j below 2^24 and fp32
            accumulation in any order is exact.
The paper uses dummy weights too: performance is content-independent.
"""

from __future__ import annotations

import hashlib

import numpy as np

# --------------------------------------------------------------------------
# layer shapes (K -> N) of the models BASELINE.json names
# --------------------------------------------------------------------------
LLAMA3_8B = {  # hidden 4096, kv 1024 (GQA), ffn 14336
    "q": (4096, 4096), "k": (4096, 1024), "v": (4096, 1024), "o": (4096, 4096),
    "gate_up": (4096, 28672), "down": (14336, 4096),
}
LLAMA33_70B = {  # hidden 8192, q+k+v = 8192+1024+1024, ffn 28672 (reading R21)
    "qkv": (8192, 10240), "o": (8192, 8192), "gate_up": (8192, 57344), "down": (28672, 8192),
}
QWEN25_32B = {  # hidden 5120, q+k+v = 5120+1024+1024, ffn 27648
    "qkv": (5120, 7168), "o": (5120, 5120), "gate_up": (5120, 55296), "down": (27648, 5120),
}

# BASELINE.json configs[0..4]
CONFIG0 = {"name": "c0_u4_gemv_512", "layers": {"l": (512, 512)}, "M": [1], "formats": ["u4"], "group": 128}
CONFIG1_FORMATS = ["u1", "u2", "u3", "u4", "u5", "u6", "u7", "u8",
                   "i1", "i2", "i3", "i4", "i5", "i6", "i7", "i8",
                   "f3e1m1", "f4e2m1", "f5e2m2", "f6e3m2", "f7e3m3", "f8e4m3"]
CONFIG1 = {"name": "c1_llama3_8b_decode", "layers": LLAMA3_8B, "M": [1, 16], "formats": CONFIG1_FORMATS, "group": 128}
CONFIG2 = {"name": "c2_llama33_70b", "layers": LLAMA33_70B, "M": [1, 16, 64, 128],
           "formats": ["u3", "i5", "f6e3m2", "u8"], "group": 128}
CONFIG3 = {"name": "c3_qwen25_32b_sweep", "layers": QWEN25_32B,
           "M": [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128, 160, 192, 224, 256],
           "formats": ["i4", "f6e3m2"], "group": 128}
CONFIG4 = {"name": "c4_llama33_70b_gate_up_sharded", "layers": {"gate_up": (8192, 57344)},
           "M": [1, 16, 128], "formats": ["u4", "i6"], "group": 128, "world": [1, 2, 4, 8]}
CONFIGS = [CONFIG0, CONFIG1, CONFIG2, CONFIG3, CONFIG4]


def stable_seed(*parts) -> int:
    """Seed = stable hash of the config string (same on every host / Python run)."""
    h = hashlib.sha256("|".join(str(p) for p in parts).encode()).digest()
    return int.from_bytes(h[:8], "little")


def _bits_of(fmt: str) -> int:
    # 'u4' / 'i6' / 'f6e3m2' -> bit width (naming grammar only)
    return int(fmt[1])


def _kind_of(fmt: str) -> str:
    return fmt[0]


def gen_codes(fmt: str, K: int, N: int, seed: int) -> np.ndarray:
    """Uniform codes [K, N] uint8 over all 2^b values."""
    b = _bits_of(fmt)
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, 1 << b, size=(K, N), dtype=np.uint8)


def gen_scales(fmt: str, K: int, N: int, group: int, seed: int) -> np.ndarray:
    """fp16 scales [K/G, N] = U[0.5,1.5) * 0.02 / 2^(b-1)."""
    b = _bits_of(fmt)
    rng = np.random.Generator(np.random.PCG64(seed + 1))
    u = rng.random(size=(K // group, N)) + 0.5
    return (u * (0.02 / (1 << (b - 1)))).astype(np.float16)


def gen_zeros(fmt: str, K: int, N: int, group: int, seed: int, zero_range: str = "mid") -> np.ndarray | None:
    """fp16 integer zero points [K/G, N] for unsigned formats, else None."""
    if _kind_of(fmt) != "u":
        return None
    b = _bits_of(fmt)
    rng = np.random.Generator(np.random.PCG64(seed + 2))
    if zero_range == "full":
        z = rng.integers(0, 1 << b, size=(K // group, N))
    else:
        lo = max((1 << (b - 1)) - 1, 0)
        z = rng.integers(lo, (1 << (b - 1)) + 1, size=(K // group, N))
    return z.astype(np.float16)


def gen_activations(M: int, K: int, seed: int) -> np.ndarray:
    """A [M, K] fp16 ~ N(0, 1)."""
    rng = np.random.Generator(np.random.PCG64(seed + 3))
    return rng.standard_normal(size=(M, K)).astype(np.float16)


def gen_activations_i8(M: int, K: int, seed: int) -> np.ndarray:
    """A [M, K] int8, uniform over all 256 values (row f4: int8 activations)."""
    rng = np.random.Generator(np.random.PCG64(seed + 6))
    return rng.integers(-128, 128, size=(M, K), dtype=np.int8)


def gen_mx_exponents(K: int, N: int, seed: int, center: int, spread: int = 3) -> np.ndarray:
    """E8M0 block-scale codes [K/32, N] uint8, uniform in [center - spread, center + spread]
    (row f4: microscaling, one code per block of 32 weights along K)."""
    rng = np.random.Generator(np.random.PCG64(seed + 7))
    return rng.integers(center - spread, center + spread + 1, size=(K // 32, N)).astype(np.uint8)


def gen_exact_instance(fmt: str, M: int, K: int, N: int, group: int, seed: int, j: int = 0):
    """Exact-integer instance: A in {-1,0,1}, s = 2^-j, integer zeros.

    Returns (A, codes, scales, zeros).  With K <= 8192 and |q - z| <= 255 every
    partial sum is an integer multiple of 2^-j of magnitude < 2^24 * 2^-j, so
    fp32 accumulation in ANY order is exact and the fp16 output must equal the
    round-to-nearest-even of the fp64 result bit for bit.  (Float formats with
    E <= 4 have values that are multiples of 2^-9 at most: j is raised
    accordingly by the caller when needed.)
    """
    rng = np.random.Generator(np.random.PCG64(seed + 4))
    A = rng.integers(-1, 2, size=(M, K)).astype(np.float16)
    codes = gen_codes(fmt, K, N, seed)
    scales = np.full((K // group, N), 2.0 ** (-j), dtype=np.float16)
    zeros = gen_zeros(fmt, K, N, group, seed, zero_range="full")
    return A, codes, scales, zeros


def sample_columns(N: int, n_tile: int = 128, shards: int = 8, extra: int = 64, seed: int = 0) -> np.ndarray:
    """Column sample for full-size parity: first/last column of every N-tile and shard + random."""
    cols = set()
    for t in range(0, N, n_tile):
        cols.add(t)
        cols.add(min(t + n_tile - 1, N - 1))
    for s in range(shards):
        lo = s * N // shards
        cols.add(lo)
        cols.add(max(lo - 1, 0))
    rng = np.random.Generator(np.random.PCG64(seed + 5))
    cols.update(rng.integers(0, N, size=extra).tolist())
    return np.array(sorted(cols), dtype=np.int64)


# --------------------------------------------------------------------------
# device-side generators (same recipe, torch's Philox RNG) for bench-size layers
# --------------------------------------------------------------------------
def torch_generator(seed: int, device="cuda"):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed & ((1 << 63) - 1))
    return g


def gen_codes_torch(fmt: str, K: int, N: int, seed: int, device="cuda"):
    import torch
    b = _bits_of(fmt)
    return torch.randint(0, 1 << b, (K, N), generator=torch_generator(seed, device), device=device, dtype=torch.uint8)


def gen_scales_torch(fmt: str, K: int, N: int, group: int, seed: int, device="cuda"):
    import torch
    b = _bits_of(fmt)
    u = torch.rand((K // group, N), generator=torch_generator(seed + 1, device), device=device) + 0.5
    return (u * (0.02 / (1 << (b - 1)))).to(torch.float16)


def gen_zeros_torch(fmt: str, K: int, N: int, group: int, seed: int, device="cuda"):
    import torch
    if _kind_of(fmt) != "u":
        return None
    b = _bits_of(fmt)
    lo = max((1 << (b - 1)) - 1, 0)
    z = torch.randint(lo, (1 << (b - 1)) + 1, (K // group, N), generator=torch_generator(seed + 2, device),
                      device=device)
    return z.to(torch.float16)


def gen_activations_torch(M: int, K: int, seed: int, device="cuda"):
    import torch
    return torch.randn((M, K), generator=torch_generator(seed + 3, device), device=device).to(torch.float16)
