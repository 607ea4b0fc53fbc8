"""GPU: the column-sharded GEMM with the chunked all-gather (dist.sharded_gemm_columns) on the
real library, 2 ranks sharing this box's GPU over gloo (NCCL refuses two ranks per device; on
an 8-GPU box the same code takes the in-place NCCL path).  The gathered C must equal the
single-process GPU C bitwise (per-row / per-column exponents)."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2603_29975_b200 as oz
    import synth
    from paper_2603_29975_b200 import dist as zd

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, k, n, s = 300, 200, 1100, 7
        A = oz.colmajor(torch.from_numpy(np.asfortranarray(synth.spread(m, k, seed=1, phi=2.0))).cuda())
        B = oz.colmajor(torch.from_numpy(np.asfortranarray(synth.spread(k, n, seed=2, phi=2.0))).cuda())
        ref = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        oz.dgemm("N", "N", 1.0, A, B, 0.0, ref, s)

        def gemm(a, b, c):
            oz.dgemm("N", "N", 1.0, a, b, 0.0, c, s)

        ok = []
        for chunks in (1, 2, 4):
            C = torch.full((n, m), float("nan"), dtype=torch.float64, device="cuda").t()
            zd.sharded_gemm_columns(gemm, A, B, C, rank, world, chunks=chunks)
            torch.cuda.synchronize()
            ok.append(bool(torch.equal(C, ref)))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_sharded_gemm_columns_two_ranks_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok in res:
        assert all(ok), f"rank {rank}: gathered C != single-process C for chunks (1, 2, 4): {ok}"
