"""O3/O4 -- compact storage of low-bit codes.  TEST INFRASTRUCTURE ONLY.

Paper: low-precision data are stored "compactly within bytes ...
a single value [may span] two uint8 entries"; loading "extract[s] relevant bits
using bitwise AND, adjust[s] their position with bitwise SHIFT operations, and
finally combine[s] separated parts using bitwise OR if the value spans multiple
bytes"; storing "clear[s] the target bit positions using a bitwise mask, then
insert[s] the new value using bitwise OR".  SPEC PackedBuffer:
element k occupies stream bits [k*b, (k+1)*b), LSB-first; length
ceil(count*b/8); trailing pad bits zero.

Readings: R1 LSB-first stream (bit t of element i is stream bit
i*b+t; stream bit j is bit j&7 of byte j>>3).  R2 a [K,N] weight is flattened
row-major (i = k*N + n), n fastest ("i6[K, N]").
"""

from __future__ import annotations

import numpy as np


def packed_nbytes(count: int, bits: int) -> int:
    """Length of the packed buffer, ceil(count*bits/8)."""
    return (count * bits + 7) // 8


def pack(codes: np.ndarray, bits: int) -> np.ndarray:
    """Store every code with the paper's mask-then-OR procedure.

    ``codes`` is any integer array (flattened row-major, R2); returns uint8.
    """
    c = np.ascontiguousarray(codes).reshape(-1).astype(np.int64)
    if c.size and (c.min() < 0 or c.max() >= (1 << bits)):
        raise ValueError("code does not fit in the bit width")
    n = c.size
    buf = np.zeros(packed_nbytes(n, bits) + 1, dtype=np.int64)  # +1: room for the spill byte
    start = np.arange(n, dtype=np.int64) * bits
    j0 = start >> 3
    off = start & 7
    # first byte: clear the target bits, then OR the low part of the value in
    low = (c << off) & 0xFF
    mask0 = (((1 << bits) - 1) << off) & 0xFF
    # elements never share bits, so clearing then OR-ing element by element is
    # the same as doing it for all elements at once
    np.bitwise_and.at(buf, j0, ~mask0 & 0xFF)
    np.bitwise_or.at(buf, j0, low)
    # second byte, only where the value spans the byte boundary
    span = off + bits > 8
    if span.any():
        hi = c[span] >> (8 - off[span])
        mask1 = ((1 << bits) - 1) >> (8 - off[span])
        np.bitwise_and.at(buf, j0[span] + 1, ~mask1 & 0xFF)
        np.bitwise_or.at(buf, j0[span] + 1, hi)
    return buf[:-1].astype(np.uint8)


def unpack(buf: np.ndarray, count: int, bits: int) -> np.ndarray:
    """Load ``count`` codes with AND / SHIFT / OR across byte boundaries."""
    b = np.ascontiguousarray(buf).reshape(-1).astype(np.int64)
    if b.size < packed_nbytes(count, bits):
        raise ValueError("buffer too short")
    b = np.concatenate([b, np.zeros(1, dtype=np.int64)])
    start = np.arange(count, dtype=np.int64) * bits
    j0 = start >> 3
    off = start & 7
    lo = b[j0] >> off  # SHIFT the first byte's bits down
    hi = np.where(off + bits > 8, b[j0 + 1] << (8 - off), 0)  # part in the next byte
    return ((lo | hi) & ((1 << bits) - 1)).astype(np.uint8)  # OR, then AND the field
