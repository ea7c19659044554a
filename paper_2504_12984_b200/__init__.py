"""B200-native A16Wx low-bit-weight matmul (the hot path of Tilus, arXiv 2504.12984).

Y[M,N] = A[M,K] (fp16, bf16 or int8) x dequant(Wq[K,N]) with Wq in any of 37 weight formats
(uint1..8, int1..8, float3..8 with E <= 4), group-wise fp16 scales and, for
unsigned formats, zero points.  The product is the C-ABI library
``libtilus_b200.so`` (include/tilus_b200.h); this package is its thin ctypes
binding (``_lib``) plus the N-sharded multi-GPU wrapper (``dist``).

The library must be built (``python paper_2504_12984_b200/build.py``); there is
no CPU fallback.
"""

from ._lib import (TL_PATH_AUTO, TL_PATH_GEMV, TL_PATH_TC, TL_PATH_TCD, TL_PATH_PREFILL, TL_ACT_F16, TL_ACT_BF16, TL_ACT_I8, TL_FLAG_STATIC_WEIGHTS, EXPORTED, LIB_PATH, TilusError, alloc_workspace,
                   tl_dequant, tl_format_version, tl_matmul, tl_matmul_ex, tl_matmul_hostio, tl_matmul_batch_hostio, batch_items, tl_matmul_plan,
                   tl_matmul_workspace_bytes, tl_matmul_gathered, tl_gather_wait, tl_signal_peers, tl_reduce_scatter_peer, tl_mx_scales_to_f16, tl_mx_scales_to_bf16, tl_pack, tl_packed_bytes, tl_transform_weights,
                   tl_transformed_bytes, tl_unpack, tl_untransform_weights, tl_wtype, wtype)

__all__ = [
    "TL_PATH_AUTO", "TL_PATH_GEMV", "TL_PATH_TC", "TL_PATH_TCD", "TL_PATH_PREFILL", "TL_ACT_F16", "TL_ACT_BF16", "TL_ACT_I8", "TL_FLAG_STATIC_WEIGHTS", "EXPORTED", "LIB_PATH", "TilusError", "alloc_workspace",
    "tl_dequant", "tl_format_version", "tl_matmul", "tl_matmul_ex", "tl_matmul_hostio", "tl_matmul_batch_hostio", "batch_items", "tl_matmul_plan",
    "tl_matmul_workspace_bytes", "tl_matmul_gathered", "tl_gather_wait", "tl_signal_peers", "tl_reduce_scatter_peer", "tl_mx_scales_to_f16", "tl_mx_scales_to_bf16", "tl_pack", "tl_packed_bytes", "tl_transform_weights", "tl_transformed_bytes",
    "tl_unpack", "tl_untransform_weights", "tl_wtype", "wtype",
]
