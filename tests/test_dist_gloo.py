"""Multi-process (world_size 2, gloo, CPU) tests of the sharding logic (-m "not gpu").

The per-rank GEMM is the CPU oracle, so the test checks the distribution
scheme itself: column-sharded + all-gathered C must equal the single-process
oracle C bitwise (per-column exponents make slabs independent),
and batch shards must partition the batch.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2603_29975_b200 import dist as zd

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, k, n, s = 48, 40, 300, 6
        A = synth.spread(m, k, seed=1, phi=2.0)
        B = synth.spread(k, n, seed=2, phi=2.0)

        def gemm(At, Bt, Ct):   # oracle as the local GEMM: Ct = op(A) op(B)
            Ct.copy_(torch.from_numpy(oracle.dgemm("N", "N", 1.0, At.numpy(), Bt.numpy(), 0.0, None, s)))

        ref = oracle.dgemm("N", "N", 1.0, A, B, 0.0, None, s)
        bitexact = True
        for chunks in (1, 2, 3):   # one block per rank, and the chunked (overlapped) ownership
            Ct = torch.zeros((n, m), dtype=torch.float64).t()      # column-major m x n
            zd.sharded_gemm_columns(gemm, torch.from_numpy(A), torch.from_numpy(B), Ct, rank, world,
                                    chunks=chunks)
            bitexact = bitexact and bool((Ct.numpy() == ref).all())
        # batch shards and max-over-ranks
        shards = [zd.batch_shard(30, r, world) for r in range(world)]
        mx = zd.max_over_ranks(float(rank + 1))
        q.put((rank, bitexact, shards, mx))
    finally:
        dist.destroy_process_group()


def test_column_sharding_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, bitexact, shards, mx in res:
        assert bitexact, f"rank {rank}: gathered C != single-process oracle"
        assert mx == 2.0
        assert shards[0] == (0, 15) and shards[1] == (15, 30)


def test_shard_arithmetic():
    from paper_2603_29975_b200 import dist as zd
    for total in (0, 1, 7, 30, 256):
        for world in (1, 2, 3, 4, 8):
            rs = [zd.batch_shard(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    for n in (1, 100, 128, 1000, 32768):
        for world in (1, 2, 4, 8):
            sl = [zd.column_slab(n, r, world) for r in range(world)]
            assert sl[0][0] == 0 and max(b for a, b in sl) == n
            cover = np.zeros(n, int)
            for a, b in sl:
                cover[a:b] += 1
                assert a % zd.TILE_N == 0 or a == n
            assert (cover == 1).all()
            for chunks in (1, 2, 4):
                cover = np.zeros(n, int)
                for r in range(world):
                    width, bl = zd.column_blocks(n, r, world, chunks)
                    for c, (a, b) in enumerate(bl):
                        cover[a:b] += 1
                        if b > a:   # block g = c * world + r at offset r * width inside chunk c
                            assert a == (c * world + r) * width and a % zd.TILE_N == 0
                assert (cover == 1).all()
                if chunks == 1:
                    assert all(zd.column_blocks(n, r, world, 1)[1][0] == zd.column_slab(n, r, world)
                               for r in range(world))
