"""CPU oracle for the Tilus A16Wx low-bit-weight matmul (arXiv 2504.12984).

TEST INFRASTRUCTURE ONLY.  This package is the plain, slow, obviously-correct
reference that the CUDA path is checked against.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2504_12984_b200``) never imports, calls or links anything in here, and
this package never imports the product path; the two share no code.  The only
module both sides use is ``workloads`` (seeded input generators, no method
arithmetic).

Citations: ``P:L`` = line L of the paper text, ``S:L`` = line L of
SPEC.md.  Every reading of a passage the paper leaves open is listed in
DESIGN.md's "Readings" table (R-numbers) and quoted next to the code.

Modules
  formats  -- O1/O2: the 37 weight formats and the value of every code
              
  packing  -- O3/O4: compact LSB-first bitstream pack / unpack
  dequant  -- O5: group-wise dequantization, exact (S:248-256 + zero points)
  matmul   -- O6/O7: fp64 matmul C = A x B and the tolerance
              comparator the north star states
  quantize -- O9: round-to-nearest-even encoder used only to build test data
  mx       -- row f4: E8M0 microscaling block scales and MX dequant (reading R25)

Every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against something other than itself (ml_dtypes
value tables, numpy.packbits, exact rational brute force, closed forms and the
paper's / SPEC's worked examples).  No function is "parity unpinned".
"""

from .formats import WType, parse_wtype, all_kernel_formats, oracle_only_formats, code_values
from .packing import pack, unpack, packed_nbytes
from .dequant import dequant
from .matmul import matmul_fp64, matmul_cols_fp64, tolerance_check
from .quantize import encode
from .mx import e8m0_value, e8m0_to_f16_scale, e8m0_to_bf16_scale, mx_dequant, MX_BLOCK

__all__ = [
    "WType", "parse_wtype", "all_kernel_formats", "oracle_only_formats", "code_values",
    "pack", "unpack", "packed_nbytes", "dequant", "matmul_fp64", "matmul_cols_fp64",
    "tolerance_check", "encode", "e8m0_value", "e8m0_to_f16_scale", "e8m0_to_bf16_scale", "mx_dequant", "MX_BLOCK",
]
