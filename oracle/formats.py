"""O1/O2 -- weight formats and the value of every code.  TEST INFRASTRUCTURE ONLY.

Paper: "Supported types include int2 to int8, uint1 to uint8, and float3 to
float8, with arbitrary exponent and mantissa distribution for floating-point
types"; the evaluation uses e4m3, e3m3, e3m2, e2m2, e2m1, e1m1.
SPEC: ScalarType{kind, bits, exponent_bits, mantissa_bits}, decode
semantics, no Inf/NaN and bias 2^(E-1)-1 with subnormals
(S:267-268).

Readings:
  R3  minifloats: bias = 2^(E-1)-1, subnormals at e=0, no Inf/NaN (the all-ones
      exponent is an ordinary binade).  s=1,e=0,m=0 is -0.0.
  R4  kernel formats: float E in [1,4], M = b-1-E >= 0 (21 formats; every code
      is exactly representable in fp16).  E in [5,7] exists here only.
  R5  int1 (BASELINE config 2) is two's complement: code 0 -> 0, code 1 -> -1.
"""

from __future__ import annotations

import re
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class WType:
    """Weight element type.  kind: 'u' (unsigned int), 'i' (signed int), 'f' (float).

    The 4-byte descriptor (kind, bits, exp, man) follows SPEC's dtype code.
    """

    kind: str
    bits: int
    exp: int = 0
    man: int = 0

    @property
    def name(self) -> str:
        if self.kind == "f":
            return f"f{self.bits}e{self.exp}m{self.man}"
        return f"{self.kind}{self.bits}"

    @property
    def kind_code(self) -> int:
        return {"u": 0, "i": 1, "f": 2}[self.kind]

    @property
    def has_zeros(self) -> bool:
        """Zero points exist for unsigned formats only (north star; reading R6)."""
        return self.kind == "u"

    def validate(self, kernel: bool = True) -> None:
        if self.kind not in ("u", "i", "f"):
            raise ValueError(f"bad kind {self.kind!r}")
        if not 1 <= self.bits <= 8:
            raise ValueError(f"bits must be in [1,8], got {self.bits}")
        if self.kind == "f":
            if self.bits < 3:
                raise ValueError("float formats have 3..8 bits (P:162)")
            if self.exp < 1 or self.man < 0 or 1 + self.exp + self.man != self.bits:
                raise ValueError(f"bad float split e{self.exp}m{self.man} for {self.bits} bits")
            if kernel and self.exp > 4:
                raise ValueError("kernel float formats need E <= 4 (reading R4)")
        elif self.exp or self.man:
            raise ValueError("integer formats carry no exponent/mantissa split")

    def __str__(self) -> str:  # pragma: no cover - cosmetic
        return self.name


_GRAMMAR = re.compile(r"^(?:(u|i)(\d)|f(\d)e(\d)m(\d))$")


def parse_wtype(s: str, kernel: bool = True) -> WType:
    """Parse the dtype grammar u<b> / i<b> / f<b>e<E>m<M>."""
    m = _GRAMMAR.match(s.strip())
    if not m:
        raise ValueError(f"cannot parse dtype {s!r}")
    if m.group(1):
        wt = WType(m.group(1), int(m.group(2)))
    else:
        wt = WType("f", int(m.group(3)), int(m.group(4)), int(m.group(5)))
    wt.validate(kernel=kernel)
    return wt


def all_kernel_formats() -> list[WType]:
    """The 37 formats the kernels support: u1..u8, i1..i8, 21 floats with E<=4 (reading R4)."""
    out = [WType("u", b) for b in range(1, 9)] + [WType("i", b) for b in range(1, 9)]
    for b in range(3, 9):
        for e in range(1, 5):
            m = b - 1 - e
            if m >= 0:
                out.append(WType("f", b, e, m))
    return out


def oracle_only_formats() -> list[WType]:
    """Float formats with E >= 5: defined by the oracle, not fp16-exact, no kernel."""
    out = []
    for b in range(6, 9):
        for e in range(5, 8):
            m = b - 1 - e
            if m >= 0:
                out.append(WType("f", b, e, m))
    return out


def code_value(wt: WType, c: int) -> float:
    """Value of one code, written out as the definition (R3, R5)."""
    b = wt.bits
    if not 0 <= c < (1 << b):
        raise ValueError("code out of range")
    if wt.kind == "u":
        return float(c)
    if wt.kind == "i":
        # two's complement: codes >= 2^(b-1) are negative
        return float(c - (1 << b)) if c >= (1 << (b - 1)) else float(c)
    E, M = wt.exp, wt.man
    s = c >> (b - 1)
    e = (c >> M) & ((1 << E) - 1)
    m = c & ((1 << M) - 1)
    bias = (1 << (E - 1)) - 1
    sign = -1.0 if s else 1.0
    if e == 0:  # subnormal: 2^(1-bias) * m / 2^M
        return sign * (2.0 ** (1 - bias)) * (m / float(1 << M))
    return sign * (2.0 ** (e - bias)) * (1.0 + m / float(1 << M))


def code_values(wt: WType) -> np.ndarray:
    """float64 table value[code] for all 2^b codes."""
    return np.array([code_value(wt, c) for c in range(1 << wt.bits)], dtype=np.float64)
