"""Host logic of the N-sharded multi-GPU path on CPU with world_size-2 gloo.

Each rank computes its column shard with the oracle (the CPU stand-in for tl_matmul on
its GPU), gather_columns reassembles Y, and the result must equal the full oracle output
bit for bit (column independence)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as wl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _column_shard(N, world, rank):
    # imported lazily inside the worker so the spawn start-up stays light
    from paper_2504_12984_b200.dist import column_shard
    return column_shard(N, world, rank)


def _worker(rank, world, port, fmt, M, K, N, G, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import dequant, matmul_fp64, parse_wtype
    from paper_2504_12984_b200.dist import column_shard, gather_columns
    seed = wl.stable_seed("dist", fmt, M, K, N)
    A = wl.gen_activations(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    z = wl.gen_zeros(fmt, K, N, G, seed)
    n0, n1 = column_shard(N, world, rank)
    w = dequant(parse_wtype(fmt), codes[:, n0:n1], s[:, n0:n1], None if z is None else z[:, n0:n1], G)
    y_shard = torch.from_numpy(matmul_fp64(A, w).astype(np.float16))
    Y = gather_columns(y_shard, N, world)
    if rank == 0:
        np.save(os.path.join(out_dir, "Y.npy"), Y.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M", [1, 3])
def test_gather_two_ranks_matches_full_oracle(tmp_path, M):
    world, fmt, K, N, G = 2, "u4", 256, 1024, 128
    mp.spawn(_worker, args=(world, _free_port(), fmt, M, K, N, G, str(tmp_path)), nprocs=world, join=True)
    Y = np.load(tmp_path / "Y.npy")
    from oracle import dequant, matmul_fp64, parse_wtype
    seed = wl.stable_seed("dist", fmt, M, K, N)
    A = wl.gen_activations(M, K, seed)
    full = matmul_fp64(A, dequant(parse_wtype(fmt), wl.gen_codes(fmt, K, N, seed), wl.gen_scales(fmt, K, N, G, seed),
                                  wl.gen_zeros(fmt, K, N, G, seed), G)).astype(np.float16)
    assert np.array_equal(Y.view(np.uint16), full.view(np.uint16))


@pytest.mark.parametrize("N,world", [(57344, 8), (57344, 2), (1024, 8), (384, 2), (10240, 8), (640, 3)])
def test_column_shards_partition_and_align(N, world):
    spans = [_column_shard(N, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == N
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    widths = [b - a for a, b in spans]
    assert all(w % 128 == 0 and w > 0 for w in widths)
    assert max(widths) - min(widths) <= 128


def test_column_shard_rejects_bad_inputs():
    from paper_2504_12984_b200.dist import column_shard
    with pytest.raises(ValueError):
        column_shard(1000, 2, 0)
    with pytest.raises(ValueError):
        column_shard(1024, 2, 2)


def test_bench_relaunches_itself_with_one_process_per_gpu():
    """`python bench.py --gpus N` (no WORLD_SIZE) re-executes under torch.distributed.run with N ranks
    on 127.0.0.1 and the same arguments (the driver's own launch form)."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    argv = b.torchrun_argv(4, ["--gpus", "4", "--steps", "7"], 29555)
    assert argv[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv and "--master-port=29555" in argv
    assert argv[-4:] == ["--gpus", "4", "--steps", "7"] and argv[-5].endswith("bench.py")


def _fused_worker(rank, world, port, M, N, out_dir):
    """Row f3 host logic: exchange fake buffer bases, derive the peer addresses with peer_pointers,
    and 'store' this rank's shard into every rank's buffer at those addresses (a byte-addressed
    numpy arena stands in for the mapped device memory).  Every rank's buffer must end up equal to
    the full Y, and every flag slot must be hit once by its owner rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_12984_b200.dist import column_shard, exchange, peer_pointers
    ybytes = M * N * 2
    y_base = (1 << 24) * (rank + 1)                               # disjoint fake address ranges
    f_base = (1 << 30) + 64 * rank
    bases = exchange((y_base, f_base), world)
    y_bases = [b[0] for b in bases]
    f_bases = [b[1] for b in bases]
    assert y_bases[rank] == y_base and len(set(y_bases)) == world
    n0, n1 = column_shard(N, world, rank)
    ys, fs = peer_pointers(y_bases, f_bases, rank, n0)
    assert len(ys) == world - 1
    Yfull = (np.arange(M * N, dtype=np.float64).reshape(M, N) % 2039).astype(np.float16)
    writes = []
    for q_addr, f_addr in zip(ys, fs):
        q = [i for i, b in enumerate(y_bases) if b <= q_addr < b + ybytes][0]
        assert f_bases[q] + 4 * rank == f_addr
        col0 = (q_addr - y_bases[q]) // 2
        assert col0 == n0
        writes.append((q, col0))
    allw = exchange(writes, world)
    if rank == 0:
        bufs = [np.full((M, N), np.nan, np.float16) for _ in range(world)]
        for r, ws_ in enumerate(allw):
            a, b = column_shard(N, world, r)
            bufs[r][:, a:b] = Yfull[:, a:b]                       # the rank's local store
            for q, c0 in ws_:
                bufs[q][:, c0:c0 + (b - a)] = Yfull[:, a:b]       # the replicated epilogue stores
        for q in range(world):
            assert np.array_equal(bufs[q].view(np.uint16), Yfull.view(np.uint16)), q
        np.save(os.path.join(out_dir, "ok.npy"), np.ones(1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_gather_peer_addresses(tmp_path, world):
    mp.spawn(_fused_worker, args=(world, _free_port(), 3, 1024, str(tmp_path)), nprocs=world, join=True)
    assert (tmp_path / "ok.npy").exists()


def test_row_shard_and_reduce_pointers():
    from paper_2504_12984_b200.dist import reduce_pointers, row_shard
    K, G = 8192, 128
    for world in (2, 3, 4, 8):
        spans = [row_shard(K, world, r, G) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == K
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert all((k1 - k0) % 128 == 0 and k0 % G == 0 for k0, k1 in spans)
    assert all(k0 % 384 == 0 for k0, _ in (row_shard(3 * 384 * 4, 4, r, 384) for r in range(4)))  # lcm(128, 384)
    with pytest.raises(ValueError):
        row_shard(8192 + 128, 2, 0, 256)
    assert reduce_pointers([1000, 5000], 64) == [1128, 5128]


def _rowpar_worker(rank, world, port, out_dir):
    """Row-parallel host logic with gloo: every rank's partial is the oracle on its K rows; an
    all_gather of the partials stands in for the peer mapping; each rank reduces its column block
    in rank order in fp32 -- the concatenation must equal the same reduction done centrally."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import dequant, matmul_fp64, parse_wtype
    from paper_2504_12984_b200.dist import column_shard, exchange, row_shard
    fmt, M, K, N, G = "u4", 2, 1024, 512, 128
    seed = wl.stable_seed("rowpar-cpu", fmt, M, K, N)
    A = wl.gen_activations(M, K, seed)
    codes = wl.gen_codes(fmt, K, N, seed)
    s = wl.gen_scales(fmt, K, N, G, seed)
    z = wl.gen_zeros(fmt, K, N, G, seed)
    k0, k1 = row_shard(K, world, rank, G)
    wd = dequant(parse_wtype(fmt), codes[k0:k1], s[k0 // G:k1 // G], z[k0 // G:k1 // G], G)
    part = matmul_fp64(A[:, k0:k1], wd).astype(np.float16)
    parts = exchange(part, world)
    n0, n1 = column_shard(N, world, rank)
    acc = np.zeros((M, n1 - n0), np.float32)
    for p in parts:
        acc = acc + p[:, n0:n1].astype(np.float32)
    blocks = exchange(acc.astype(np.float16), world)
    if rank == 0:
        Y = np.concatenate(blocks, axis=1)
        ref = np.zeros((M, N), np.float32)
        for p in parts:
            ref = ref + p.astype(np.float32)
        assert np.array_equal(Y.view(np.uint16), ref.astype(np.float16).view(np.uint16))
        np.save(os.path.join(out_dir, "ok.npy"), np.ones(1))
    dist.barrier()
    dist.destroy_process_group()


def test_row_parallel_two_ranks(tmp_path):
    mp.spawn(_rowpar_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok.npy").exists()
