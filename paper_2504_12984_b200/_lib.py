"""ctypes binding of libtilus_b200.so -- argument marshalling only.

Every function here has the name of the C entry point it wraps
(include/tilus_b200.h) and does nothing but turn torch tensors into device
pointers / sizes and the current CUDA stream into a ``cudaStream_t``.  All of
the method's work runs in the CUDA kernels of the library.  There is no CPU
fallback: if the library is missing, importing this module raises.
"""

from __future__ import annotations

import ctypes
import os
import re

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TL_LIB_PATH") or os.path.join(_HERE, "libtilus_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build it with `python paper_2504_12984_b200/build.py` "
        "(there is no CPU fallback for the A16Wx matmul)")

_lib = ctypes.CDLL(LIB_PATH)


class tl_wtype(ctypes.Structure):  # noqa: N801 -- C name
    _fields_ = [("kind", ctypes.c_uint8), ("bits", ctypes.c_uint8),
                ("exp_bits", ctypes.c_uint8), ("man_bits", ctypes.c_uint8)]

    @property
    def name(self) -> str:
        if self.kind == 2:
            return f"f{self.bits}e{self.exp_bits}m{self.man_bits}"
        return ("u" if self.kind == 0 else "i") + str(self.bits)

    def __repr__(self) -> str:
        return f"tl_wtype({self.name})"


_DT = re.compile(r"^(?:(u|i)(\d)|f(\d)e(\d)m(\d))$")


def wtype(name: str) -> tl_wtype:
    """Dtype grammar u<b> / i<b> / f<b>e<E>m<M> -> the 4-byte descriptor."""
    m = _DT.match(name)
    if not m:
        raise ValueError(f"bad weight dtype {name!r}")
    if m.group(1):
        return tl_wtype(0 if m.group(1) == "u" else 1, int(m.group(2)), 0, 0)
    return tl_wtype(2, int(m.group(3)), int(m.group(4)), int(m.group(5)))


TL_PATH_AUTO, TL_PATH_GEMV, TL_PATH_TC, TL_PATH_TCD, TL_PATH_PREFILL = 0, 1, 2, 3, 4
TL_ACT_F16, TL_ACT_BF16, TL_ACT_I8 = 0, 1, 2
TL_FLAG_STATIC_WEIGHTS = 1

_c_size = ctypes.c_size_t
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_vp = ctypes.c_void_p
_W = tl_wtype


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_tl_packed_bytes = _sig("tl_packed_bytes", _c_size, [_W, _i64, _i64])
_tl_transformed_bytes = _sig("tl_transformed_bytes", _c_size, [_W, _i64, _i64])
_tl_format_version = _sig("tl_format_version", ctypes.c_uint32, [])
_tl_pack = _sig("tl_pack", ctypes.c_int, [_W, _i64, _i64, _vp, _vp, _vp])
_tl_unpack = _sig("tl_unpack", ctypes.c_int, [_W, _i64, _i64, _vp, _vp, _vp])
_tl_transform_weights = _sig("tl_transform_weights", ctypes.c_int, [_W, _i64, _i64, _vp, _vp, _vp])
_tl_untransform_weights = _sig("tl_untransform_weights", ctypes.c_int, [_W, _i64, _i64, _vp, _vp, _vp])
_A = ctypes.c_int  # tl_atype
_u32 = ctypes.c_uint32
_tl_matmul_workspace_bytes = _sig("tl_matmul_workspace_bytes", _c_size, [_W, _A, _i64, _i64, _i64, _i32])
_tl_matmul = _sig("tl_matmul", ctypes.c_int,
                  [_W, _A, _i64, _i64, _i64, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _c_size, _vp])
_tl_matmul_ex = _sig("tl_matmul_ex", ctypes.c_int,
                     [_W, _A, _i64, _i64, _i64, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _c_size, _i32, _i32,
                      _u32, _vp])
_tl_matmul_hostio = _sig("tl_matmul_hostio", ctypes.c_int,
                         [_W, _A, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_size, _u32,
                          _vp])
_tl_matmul_plan = _sig("tl_matmul_plan", ctypes.c_int,
                       [_W, _A, _i64, _i64, _i64, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32)])
_tl_matmul_gathered = _sig("tl_matmul_gathered", ctypes.c_int,
                           [_W, _A, _i64, _i64, _i64, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _i64,
                            ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i32, _vp, _c_size, _u32, _vp])
class tl_batch_item(ctypes.Structure):
    _fields_ = [("w", tl_wtype), ("group", ctypes.c_int32), ("M", ctypes.c_int64), ("N", ctypes.c_int64),
                ("K", ctypes.c_int64), ("w_t", ctypes.c_void_p), ("scales", ctypes.c_void_p),
                ("zeros", ctypes.c_void_p), ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t)]


_tl_matmul_batch_hostio = _sig("tl_matmul_batch_hostio", ctypes.c_int,
                               [ctypes.c_int, ctypes.c_int32, ctypes.POINTER(tl_batch_item), _vp, _vp, _vp, _vp,
                                _u32, _vp])
_tl_signal_peers = _sig("tl_signal_peers", ctypes.c_int, [ctypes.POINTER(_vp), _i32, _vp])
_tl_reduce_scatter_peer = _sig("tl_reduce_scatter_peer", ctypes.c_int,
                               [ctypes.c_int, ctypes.POINTER(_vp), _i32, _i64, _i64, _i64, _vp, _i64, _vp])
_tl_gather_wait = _sig("tl_gather_wait", ctypes.c_int, [_vp, _i32, _i32, _u32, _vp])
_tl_mx_scales_to_f16 = _sig("tl_mx_scales_to_f16", ctypes.c_int, [_vp, _i64, _i32, _vp, _vp])
_tl_mx_scales_to_bf16 = _sig("tl_mx_scales_to_bf16", ctypes.c_int, [_vp, _i64, _i32, _vp, _vp])
_tl_dequant = _sig("tl_dequant", ctypes.c_int, [_W, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp])
_tl_status_str = _sig("tl_status_str", ctypes.c_char_p, [ctypes.c_int])
_tl_last_error = _sig("tl_last_error", ctypes.c_char_p, [])

EXPORTED = ["tl_packed_bytes", "tl_transformed_bytes", "tl_format_version", "tl_pack", "tl_unpack",
            "tl_transform_weights", "tl_untransform_weights", "tl_matmul_workspace_bytes", "tl_matmul",
            "tl_matmul_ex", "tl_matmul_hostio", "tl_matmul_batch_hostio", "tl_matmul_plan", "tl_matmul_gathered", "tl_gather_wait", "tl_signal_peers", "tl_reduce_scatter_peer", "tl_mx_scales_to_f16", "tl_mx_scales_to_bf16", "tl_dequant", "tl_status_str",
            "tl_last_error"]


class TilusError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {_tl_status_str(status).decode()} ({_tl_last_error().decode()})")


def _check(st: int, where: str) -> None:
    if st != 0:
        raise TilusError(st, where)


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ---- sizes -----------------------------------------------------------------------------
def tl_packed_bytes(w: tl_wtype, K: int, N: int) -> int:
    return _tl_packed_bytes(w, K, N)


def tl_transformed_bytes(w: tl_wtype, K: int, N: int) -> int:
    return _tl_transformed_bytes(w, K, N)


def tl_format_version() -> int:
    return _tl_format_version()


def tl_matmul_workspace_bytes(w: tl_wtype, M: int, N: int, K: int, group: int, atype: int = TL_ACT_F16) -> int:
    return _tl_matmul_workspace_bytes(w, atype, M, N, K, group)


# ---- weight preparation ------------------------------------------------------------------
def tl_pack(w: tl_wtype, K: int, N: int, codes: torch.Tensor, bitstream: torch.Tensor | None = None,
            stream=None) -> torch.Tensor:
    if bitstream is None:
        bitstream = torch.empty(tl_packed_bytes(w, K, N), dtype=torch.uint8, device=codes.device)
    _check(_tl_pack(w, K, N, _ptr(codes), _ptr(bitstream), _stream(stream)), "tl_pack")
    return bitstream


def tl_unpack(w: tl_wtype, K: int, N: int, bitstream: torch.Tensor, codes: torch.Tensor | None = None,
              stream=None) -> torch.Tensor:
    if codes is None:
        codes = torch.empty((K, N), dtype=torch.uint8, device=bitstream.device)
    _check(_tl_unpack(w, K, N, _ptr(bitstream), _ptr(codes), _stream(stream)), "tl_unpack")
    return codes


def tl_transform_weights(w: tl_wtype, K: int, N: int, bitstream: torch.Tensor, w_t: torch.Tensor | None = None,
                         stream=None) -> torch.Tensor:
    if w_t is None:
        w_t = torch.empty(max(tl_transformed_bytes(w, K, N), 16), dtype=torch.uint8, device=bitstream.device)
    _check(_tl_transform_weights(w, K, N, _ptr(bitstream), _ptr(w_t), _stream(stream)), "tl_transform_weights")
    return w_t


def tl_untransform_weights(w: tl_wtype, K: int, N: int, w_t: torch.Tensor, bitstream: torch.Tensor | None = None,
                           stream=None) -> torch.Tensor:
    if bitstream is None:
        bitstream = torch.empty(tl_packed_bytes(w, K, N), dtype=torch.uint8, device=w_t.device)
    _check(_tl_untransform_weights(w, K, N, _ptr(w_t), _ptr(bitstream), _stream(stream)), "tl_untransform_weights")
    return bitstream


def tl_dequant(w: tl_wtype, K: int, N: int, group: int, w_t: torch.Tensor, scales: torch.Tensor,
               zeros: torch.Tensor | None = None, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    if out is None:
        out = torch.empty((K, N), dtype=torch.float32, device=w_t.device)
    _check(_tl_dequant(w, K, N, group, _ptr(w_t), _ptr(scales), _ptr(zeros), _ptr(out), _stream(stream)),
           "tl_dequant")
    return out


# ---- the hot path ---------------------------------------------------------------------------
def alloc_workspace(w: tl_wtype, M: int, N: int, K: int, group: int, device="cuda",
                    atype: int = TL_ACT_F16) -> torch.Tensor:
    """Zero-filled workspace (the kernels keep its semaphores at zero between calls)."""
    return torch.zeros(tl_matmul_workspace_bytes(w, M, N, K, group, atype), dtype=torch.uint8, device=device)


def tl_matmul_gathered(w: tl_wtype, M: int, N: int, K: int, group: int, A: torch.Tensor, w_t: torch.Tensor,
                       scales: torch.Tensor, zeros: torch.Tensor | None, Y: torch.Tensor, ldy: int,
                       Y_peers: list[int], flag_peers: list[int], workspace: torch.Tensor, lda: int | None = None,
                       flags: int = 0, stream=None) -> None:
    """Row f3.  Y: a view whose data_ptr is &Yg_local[0, n0] (row stride ldy); Y_peers / flag_peers:
    integer device addresses (peer-mapped) of &Yg_peer[0, n0] and &flags_peer[rank]."""
    n = len(Y_peers)
    if len(flag_peers) != n:
        raise ValueError("Y_peers and flag_peers differ in length")
    yp = (_vp * max(n, 1))(*Y_peers)
    fp = (_vp * max(n, 1))(*flag_peers)
    _check(_tl_matmul_gathered(w, _atype(A), M, N, K, group, _ptr(A), lda if lda is not None else K, _ptr(w_t),
                               _ptr(scales), _ptr(zeros), Y.data_ptr(), ldy, yp, fp, n, _ptr(workspace),
                               workspace.numel(), flags, _stream(stream)), "tl_matmul_gathered")


def tl_gather_wait(flags: torch.Tensor, nranks: int, rank: int, epoch: int, stream=None) -> None:
    """Row f3: enqueue the wait for every other rank's `epoch`-th gathered call into this rank."""
    if flags.dtype not in (torch.int32, torch.uint32) or flags.numel() < nranks:
        raise ValueError("flags must be an int32/uint32 device tensor with nranks entries")
    _check(_tl_gather_wait(_ptr(flags), nranks, rank, epoch & 0xFFFFFFFF, _stream(stream)), "tl_gather_wait")


def tl_signal_peers(flag_peers: list[int], stream=None) -> None:
    """Row f3 (row-parallel): release +1 on every peer's flag slot for this rank after the stream's work."""
    n = len(flag_peers)
    fp = (_vp * max(n, 1))(*flag_peers)
    _check(_tl_signal_peers(fp, n, _stream(stream)), "tl_signal_peers")


def tl_reduce_scatter_peer(parts: list[int], M: int, N: int, ldp: int, Y: torch.Tensor, ldy: int | None = None,
                           atype: int = TL_ACT_F16, stream=None) -> torch.Tensor:
    """Row f3 (row-parallel): Y[M, N] = sum over ranks (rank order, fp32) of the partials at `parts`
    (device addresses of each rank's partial at this rank's column block, row stride ldp)."""
    n = len(parts)
    pa = (_vp * max(n, 1))(*parts)
    _check(_tl_reduce_scatter_peer(atype, pa, n, M, N, ldp, Y.data_ptr(), ldy if ldy is not None else N,
                                   _stream(stream)), "tl_reduce_scatter_peer")
    return Y


def tl_mx_scales_to_bf16(e8m0: torch.Tensor, exp_adjust: int = 0, out: torch.Tensor | None = None,
                         stream=None) -> torch.Tensor:
    """E8M0 block-scale codes (uint8) -> bf16 scales 2^(e-127+exp_adjust) (exact for every finite code)."""
    if e8m0.dtype != torch.uint8:
        raise ValueError("e8m0 must be uint8")
    out = out if out is not None else torch.empty(e8m0.shape, dtype=torch.bfloat16, device=e8m0.device)
    _check(_tl_mx_scales_to_bf16(_ptr(e8m0), e8m0.numel(), exp_adjust, _ptr(out), _stream(stream)),
           "tl_mx_scales_to_bf16")
    return out


def tl_mx_scales_to_f16(e8m0: torch.Tensor, exp_adjust: int = 0, out: torch.Tensor | None = None,
                        stream=None) -> torch.Tensor:
    """E8M0 block-scale codes (uint8, any shape) -> fp16 scales 2^(e-127+exp_adjust) (NaN if not fp16)."""
    if e8m0.dtype != torch.uint8:
        raise ValueError("e8m0 must be uint8")
    out = out if out is not None else torch.empty(e8m0.shape, dtype=torch.float16, device=e8m0.device)
    _check(_tl_mx_scales_to_f16(_ptr(e8m0), e8m0.numel(), exp_adjust, _ptr(out), _stream(stream)),
           "tl_mx_scales_to_f16")
    return out


def _atype(A: torch.Tensor) -> int:
    if A.dtype == torch.float16:
        return TL_ACT_F16
    if A.dtype == torch.bfloat16:
        return TL_ACT_BF16
    if A.dtype == torch.int8:
        return TL_ACT_I8
    raise ValueError(f"activations must be fp16, bf16 or int8, got {A.dtype}")


def tl_matmul(w: tl_wtype, M: int, N: int, K: int, group: int, A: torch.Tensor, w_t: torch.Tensor,
              scales: torch.Tensor, zeros: torch.Tensor | None, Y: torch.Tensor, workspace: torch.Tensor,
              lda: int | None = None, ldy: int | None = None, stream=None) -> torch.Tensor:
    _check(_tl_matmul(w, _atype(A), M, N, K, group, _ptr(A), lda if lda is not None else K, _ptr(w_t),
                      _ptr(scales), _ptr(zeros), _ptr(Y), ldy if ldy is not None else N, _ptr(workspace),
                      workspace.numel(), _stream(stream)), "tl_matmul")
    return Y


def tl_matmul_ex(w: tl_wtype, M: int, N: int, K: int, group: int, A: torch.Tensor, w_t: torch.Tensor,
                 scales: torch.Tensor, zeros: torch.Tensor | None, Y: torch.Tensor, workspace: torch.Tensor,
                 path: int = TL_PATH_AUTO, splits: int = 0, lda: int | None = None, ldy: int | None = None,
                 flags: int = 0, stream=None) -> torch.Tensor:
    _check(_tl_matmul_ex(w, _atype(A), M, N, K, group, _ptr(A), lda if lda is not None else K, _ptr(w_t),
                         _ptr(scales), _ptr(zeros), _ptr(Y), ldy if ldy is not None else N, _ptr(workspace),
                         workspace.numel(), path, splits, flags, _stream(stream)), "tl_matmul_ex")
    return Y


def tl_matmul_hostio(w: tl_wtype, M: int, N: int, K: int, group: int, A_host: torch.Tensor, A_dev: torch.Tensor,
                     w_t: torch.Tensor, scales: torch.Tensor, zeros: torch.Tensor | None, Y_dev: torch.Tensor,
                     Y_host: torch.Tensor, workspace: torch.Tensor, flags: int = 0, stream=None) -> torch.Tensor:
    if A_host.is_cuda or Y_host.is_cuda:
        raise ValueError("A_host / Y_host must be host tensors")
    _check(_tl_matmul_hostio(w, _atype(A_dev), M, N, K, group, A_host.data_ptr(), _ptr(A_dev), _ptr(w_t),
                             _ptr(scales), _ptr(zeros), _ptr(Y_dev), Y_host.data_ptr(), _ptr(workspace),
                             workspace.numel(), flags, _stream(stream)), "tl_matmul_hostio")
    return Y_host


def batch_items(problems: list[dict]) -> "ctypes.Array":
    """problems: dicts with w, group, M, N, K, w_t, scales, zeros (tensor or None), workspace (tensor)."""
    arr = (tl_batch_item * max(len(problems), 1))()
    for i, p in enumerate(problems):
        arr[i] = tl_batch_item(p["w"], p["group"], p["M"], p["N"], p["K"], _ptr(p["w_t"]), _ptr(p["scales"]),
                               _ptr(p.get("zeros")), _ptr(p["workspace"]), p["workspace"].numel())
    return arr


def tl_matmul_batch_hostio(items, count: int, A_host: torch.Tensor, A_dev: torch.Tensor, Y_dev: torch.Tensor,
                           Y_host: torch.Tensor, atype: int = TL_ACT_F16, flags: int = 0, stream=None) -> torch.Tensor:
    """One H2D of the concatenated activations, the items' matmuls in order, one D2H of the outputs."""
    if A_host.is_cuda or Y_host.is_cuda:
        raise ValueError("A_host / Y_host must be host tensors")
    _check(_tl_matmul_batch_hostio(atype, count, items, A_host.data_ptr(), _ptr(A_dev), _ptr(Y_dev),
                                   Y_host.data_ptr(), flags, _stream(stream)), "tl_matmul_batch_hostio")
    return Y_host


def tl_matmul_plan(w: tl_wtype, M: int, N: int, K: int, group: int, atype: int = TL_ACT_F16) -> tuple[int, int]:
    p, s = _i32(0), _i32(0)
    _check(_tl_matmul_plan(w, atype, M, N, K, group, ctypes.byref(p), ctypes.byref(s)), "tl_matmul_plan")
    return p.value, s.value
