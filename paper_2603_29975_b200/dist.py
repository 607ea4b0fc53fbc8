"""Multi-GPU sharding of the Ozaki path (one process per GPU, torch.distributed).

Two ways the path shards:

* batch entries (config C4: independent energy-point / atom-block ZGEMMs): rank
  r computes entries [start, stop) of the batch -- no data-path collective;
* output column slabs of one large GEMM (config C5): rank r computes
  C[:, j0:j1] from all of op(A) and its column slab of op(B), then one
  all-gather reassembles C.  Row exponents come from full rows of op(A) and
  column exponents are per column, so every element is computed exactly as on
  one GPU: the gathered C is bitwise identical to the single-GPU result.

The GEMM itself is passed in as a callable (the library's ``dgemm`` on GPUs);
this module only does the index arithmetic and the collectives.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

TILE_N = 128   # slab widths are multiples of the GEMM's N tile


def batch_shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced partition of `total` batch entries (sizes differ by <= 1)."""
    q, r = divmod(total, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def column_slab(n: int, rank: int, world: int, align: int = TILE_N) -> tuple[int, int]:
    """Column range of C owned by `rank` with one block per rank: equal widths rounded up to
    `align` (the last slab takes the remainder; trailing ranks may get an empty slab)."""
    width = -(-n // world)
    width = -(-width // align) * align
    j0 = min(n, rank * width)
    return j0, min(n, j0 + width)


def column_blocks(n: int, rank: int, world: int, chunks: int = 1, align: int = TILE_N):
    """Column ownership for the chunked (overlapped) all-gather: the n columns are cut into
    world * chunks blocks of equal width (rounded up to `align`); block g = c * world + r
    belongs to rank r, so chunk c = blocks [c * world, (c + 1) * world) is one contiguous
    column range in which rank r's block sits at offset r * width.  Returns (width,
    [(j0, j1) for each chunk c]) -- empty blocks have j0 == j1.  chunks = 1 is column_slab."""
    nb = world * chunks
    width = -(-n // nb)
    width = -(-width // align) * align
    blocks = []
    for c in range(chunks):
        j0 = min(n, (c * world + rank) * width)
        blocks.append((j0, min(n, j0 + width)))
    return width, blocks


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (timing rule: max over ranks)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sharded_gemm_columns(gemm, A, B, C, rank: int, world: int, device=None, chunks: int = 4):
    """C = op(A) B column-sharded with the all-gather overlapped with the GEMM (SURVEY.md
    §8(e)): rank r computes its block of every chunk c (`gemm(A, B_block, C_block)` in place,
    column_blocks), and after each chunk's GEMM an asynchronous all-gather of that chunk runs
    on the communicator's stream while the next chunk's GEMM runs on the compute stream.
    Chunk c's blocks are adjacent in column-major C, so with NCCL the gather is in place
    (input = this rank's block inside the output range, no staging copies); ragged last
    chunks and other backends go through padded staging buffers.  A: m x k, B: k x n,
    C: m x n column-major tensors (stride(0) == 1) on `device`.  Every element is computed
    exactly as on one GPU (per-row / per-column exponents), so the gathered C is bitwise the
    single-GPU C.  Returns C."""
    m, n = C.shape
    if world == 1:
        gemm(A, B, C)
        return C
    width, blocks = column_blocks(n, rank, world, chunks)
    nccl = dist.get_backend() == "nccl" and hasattr(dist, "all_gather_into_tensor")
    flat = C.t().view(-1) if (C.stride(0) == 1 and C.stride(1) == m) else None
    works = []
    for c, (j0, j1) in enumerate(blocks):
        c0 = c * world * width                        # first column of chunk c
        if c0 >= n:
            break
        if j1 > j0:
            gemm(A, B[:, j0:j1], C[:, j0:j1])
        full = c0 + world * width <= n                # every rank's block of this chunk is full width
        if nccl and full and flat is not None:
            out = flat[c0 * m:(c0 + world * width) * m]
            inp = out[rank * width * m:(rank + 1) * width * m]
            works.append(dist.all_gather_into_tensor(out, inp, async_op=True))
            continue
        # staging path: padded blocks (ragged chunk, non-NCCL backend or strided C)
        send = torch.zeros((width, m), dtype=C.dtype, device=C.device)
        if j1 > j0:
            send[: j1 - j0].copy_(C[:, j0:j1].t())
        recv = torch.empty((world * width, m), dtype=C.dtype, device=C.device)
        if nccl:
            dist.all_gather_into_tensor(recv, send)
        else:   # gloo (CPU tests, the 2-ranks-on-one-GPU hook): gather through host memory
            rh = torch.empty((world * width, m), dtype=C.dtype)
            dist.all_gather(list(rh.chunk(world)), send.cpu())
            recv.copy_(rh)
        for r in range(world):
            a = min(n, c0 + r * width)
            b = min(n, a + width)
            if b > a and r != rank:
                C[:, a:b].copy_(recv[r * width: r * width + (b - a)].t())
    for w in works:
        w.wait()
    return C
