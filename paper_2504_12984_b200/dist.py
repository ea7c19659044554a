"""Column (N) sharding of the A16Wx matmul across the GPUs of one box.

Output column n depends only on W[:, n], s[:, n], z[:, n] and all of A (the paper's
independent output tiles), so a column shard needs no communication
to compute.  Rank r owns columns [n0, n1) = column_shard(N, world, r): contiguous,
multiples of 128 (the transformed layout's tile width).  Each rank transforms its own
shard once (tl_transform_weights) and runs tl_matmul on it; only the *gathered* variant
exchanges data: either one all-gather of the Y shards after the matmul (NCCL over NVLink on B200;
any torch.distributed backend works, the CPU tests use gloo), or -- row f3 -- no collective at all:
``FusedGather`` maps every rank's gathered buffer into every other rank (CUDA IPC handles,
exchanged once over the process group) and the matmul kernel's epilogue stores each finished
element straight into all of them over NVLink (``tl_matmul_gathered``), then signals per-rank
flags that the consumer waits on (``tl_gather_wait``).  The row-parallel (K-sharded) variant,
``FusedReduceScatter``, sums the ranks' partials over NVLink with this library's reduce-scatter
kernel (``tl_signal_peers`` / ``tl_gather_wait`` / ``tl_reduce_scatter_peer``) instead of NCCL.

This module holds shard arithmetic and the collective only; every matmul runs in the
CUDA library through ``_lib``.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L

TILE = 128


def column_shard(N: int, world: int, rank: int, align: int = TILE) -> tuple[int, int]:
    """Columns [n0, n1) of rank `rank`: contiguous, `align`-multiples, sizes differ by <= align."""
    if N % align:
        raise ValueError(f"N={N} is not a multiple of {align}")
    if not 0 <= rank < world:
        raise ValueError("bad rank")
    tiles = N // align
    t0 = rank * tiles // world
    t1 = (rank + 1) * tiles // world
    return t0 * align, t1 * align


def gather_columns(Y_shard: torch.Tensor, N: int, world: int, group=None) -> torch.Tensor:
    """All-gather the [M, n1-n0] shards of every rank into Y [M, N] (column order by rank).

    Shards must have equal width (N divisible by world*128) so all_gather_into_tensor can
    be used; the result is a [world, M, Ns] buffer viewed/permuted to [M, N].
    """
    M, Ns = Y_shard.shape
    if Ns * world != N:
        raise ValueError("gather_columns needs equal shard widths (N % (world*128) == 0)")
    buf = torch.empty((world * M, Ns), dtype=Y_shard.dtype, device=Y_shard.device)
    dist.all_gather_into_tensor(buf, Y_shard.contiguous(), group=group)
    buf = buf.view(world, M, Ns)
    if M == 1:
        return buf.view(1, N)            # rank-major columns are already contiguous
    return buf.permute(1, 0, 2).reshape(M, N)


def peer_pointers(y_bases: list[int], flag_bases: list[int], rank: int, n0: int,
                  elem_bytes: int = 2) -> tuple[list[int], list[int]]:
    """Addresses rank `rank` passes to tl_matmul_gathered (row f3): for every OTHER rank q, the
    address of column n0 of q's gathered buffer (row 0; the row stride is the full N) and of q's
    flag slot `rank`.  `y_bases` / `flag_bases` are the ranks' buffer base addresses as mapped in
    this process."""
    if len(y_bases) != len(flag_bases) or not 0 <= rank < len(y_bases):
        raise ValueError("one gathered buffer and one flag array per rank")
    ys = [b + n0 * elem_bytes for q, b in enumerate(y_bases) if q != rank]
    fs = [f + 4 * rank for q, f in enumerate(flag_bases) if q != rank]
    return ys, fs


def exchange(obj, world: int, group=None) -> list:
    """All ranks' `obj` (picklable), rank order (one torch.distributed all_gather_object)."""
    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj, group=group)
    return out


class FusedGather:
    """Row f3: gathered outputs of an [M, N] column-sharded layer with the all-gather fused into the
    matmul epilogue.  Holds `nbuf` gathered buffers [M, N] and one flag array [world] per rank,
    mapped into every rank through CUDA IPC handles exchanged once over `group`.  Successive calls
    alternate the buffers (the ordering contract of tl_matmul_gathered): the Y a call returns stays
    valid until the call `nbuf` calls later, whose peers write into the same buffer."""

    def __init__(self, M: int, N: int, world: int, rank: int, group=None, nbuf: int = 2,
                 dtype=torch.float16):
        from torch.multiprocessing.reductions import reduce_tensor
        self.M, self.N, self.world, self.rank, self.nbuf = M, N, world, rank, nbuf
        self.Yg = [torch.empty((M, N), dtype=dtype, device="cuda") for _ in range(nbuf)]
        self.flags = torch.zeros(world, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        mine = [reduce_tensor(t) for t in self.Yg + [self.flags]] if world > 1 else None
        self._peer_tensors = []     # keeps the IPC mappings alive
        y_bases = [[0] * world for _ in range(nbuf)]
        f_bases = [0] * world
        for q, payload in enumerate(exchange(mine, world, group)):
            ts = self.Yg + [self.flags] if q == rank else [fn(*args) for fn, args in payload]
            self._peer_tensors.append(ts)
            for b in range(nbuf):
                y_bases[b][q] = ts[b].data_ptr()
            f_bases[q] = ts[nbuf].data_ptr()
        self.y_bases, self.f_bases = y_bases, f_bases
        self.epoch = 0

    def __call__(self, layer: "ShardedA16WxLinear", A: torch.Tensor) -> torch.Tensor:
        """Y = the gathered [M, N] output of `layer` (this rank's shard) for activations A."""
        self.epoch += 1
        b = self.epoch % self.nbuf
        ys, fs = peer_pointers(self.y_bases[b], self.f_bases, self.rank, layer.n0)
        Y = self.Yg[b]
        L.tl_matmul_gathered(layer.w, A.shape[0], layer.Ns, layer.K, layer.G, A, layer.w_t, layer.scales,
                             layer.zeros, Y[:, layer.n0:], self.N, ys, fs, layer._workspace(A.shape[0]))
        L.tl_gather_wait(self.flags, self.world, self.rank, self.epoch)
        return Y


def row_shard(K: int, world: int, rank: int, group: int) -> tuple[int, int]:
    """Rows [k0, k1) of rank `rank` for the row-parallel (K-sharded) variant: contiguous, multiples
    of lcm(128, group) so that no scale group and no 128-row tile straddles two ranks."""
    import math
    align = 128 * group // math.gcd(128, group)
    if K % align:
        raise ValueError(f"K={K} is not a multiple of lcm(128, group)={align}")
    return column_shard(K, world, rank, align)


def reduce_pointers(part_bases: list[int], n0: int, elem_bytes: int = 2) -> list[int]:
    """Addresses tl_reduce_scatter_peer takes on a rank owning columns [n0, n1): every rank's partial
    (base addresses as mapped in this process, row stride = the full N) at column n0."""
    return [b + n0 * elem_bytes for b in part_bases]


class FusedReduceScatter:
    """Row f3, row-parallel: every rank's fp16 partial [M, N] (its K-slice's contribution) is mapped
    into every other rank (CUDA IPC); after its matmul a rank signals the others, waits for them and
    reduces its column block of all partials over NVLink (tl_reduce_scatter_peer, fixed rank order).
    `nbuf` partial buffers alternate between calls."""

    def __init__(self, M: int, N: int, world: int, rank: int, group=None, nbuf: int = 2, dtype=torch.float16):
        from torch.multiprocessing.reductions import reduce_tensor
        self.M, self.N, self.world, self.rank, self.nbuf = M, N, world, rank, nbuf
        self.parts = [torch.empty((M, N), dtype=dtype, device="cuda") for _ in range(nbuf)]
        self.flags = torch.zeros(world, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        mine = [reduce_tensor(t) for t in self.parts + [self.flags]] if world > 1 else None
        self._peer_tensors = []
        self.p_bases = [[0] * world for _ in range(nbuf)]
        self.f_bases = [0] * world
        for q, payload in enumerate(exchange(mine, world, group)):
            ts = self.parts + [self.flags] if q == rank else [fn(*args) for fn, args in payload]
            self._peer_tensors.append(ts)
            for b in range(nbuf):
                self.p_bases[b][q] = ts[b].data_ptr()
            self.f_bases[q] = ts[nbuf].data_ptr()
        self.n0, self.n1 = column_shard(N, world, rank)
        self.epoch = 0

    def __call__(self, w, K_shard: int, G: int, A_shard: torch.Tensor, w_t, scales, zeros, workspace,
                 out: torch.Tensor | None = None) -> torch.Tensor:
        """This rank's [M, n1-n0] block of sum_r A[:, K_r] x W[K_r, :]."""
        self.epoch += 1
        b = self.epoch % self.nbuf
        P = self.parts[b]
        L.tl_matmul(w, self.M, self.N, K_shard, G, A_shard, w_t, scales, zeros, P, workspace)
        _, fs = peer_pointers([0] * self.world, self.f_bases, self.rank, 0)
        L.tl_signal_peers(fs)
        L.tl_gather_wait(self.flags, self.world, self.rank, self.epoch)
        Y = out if out is not None else torch.empty((self.M, self.n1 - self.n0), dtype=P.dtype, device=P.device)
        L.tl_reduce_scatter_peer(reduce_pointers(self.p_bases[b], self.n0), self.M, self.n1 - self.n0, self.N, Y)
        return Y


class ShardedA16WxLinear:
    """One rank's column shard of an A16Wx linear layer Y = A x dequant(W)."""

    def __init__(self, fmt: str, K: int, N: int, group: int, codes_shard: torch.Tensor, scales_shard: torch.Tensor,
                 zeros_shard: torch.Tensor | None, world: int, rank: int, pg=None):
        self.w = L.wtype(fmt)
        self.K, self.N, self.G = K, N, group
        self.world, self.rank, self.pg = world, rank, pg
        self.n0, self.n1 = column_shard(N, world, rank)
        Ns = self.n1 - self.n0
        if tuple(codes_shard.shape) != (K, Ns):
            raise ValueError("codes_shard must be [K, n1-n0]")
        bs = L.tl_pack(self.w, K, Ns, codes_shard.contiguous())
        self.w_t = L.tl_transform_weights(self.w, K, Ns, bs)
        self.scales = scales_shard.contiguous()
        self.zeros = None if zeros_shard is None else zeros_shard.contiguous()
        self.Ns = Ns
        self._ws = {}

    def _workspace(self, M: int) -> torch.Tensor:
        if M not in self._ws:
            self._ws[M] = L.alloc_workspace(self.w, M, self.Ns, self.K, self.G, device=self.w_t.device)
        return self._ws[M]

    def forward(self, A: torch.Tensor, gather: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
        M = A.shape[0]
        Y = out if out is not None else torch.empty((M, self.Ns), dtype=torch.float16, device=A.device)
        L.tl_matmul(self.w, M, self.Ns, self.K, self.G, A, self.w_t, self.scales, self.zeros, Y, self._workspace(M))
        if not gather:
            return Y
        return gather_columns(Y, self.N, self.world, self.pg)

    __call__ = forward
