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
    """Column range of C owned by `rank`: equal widths rounded up to `align`
    (the last slab takes the remainder; trailing ranks may get an empty slab)."""
    width = -(-n // world)
    width = -(-width // align) * align
    j0 = min(n, rank * width)
    return j0, min(n, j0 + width)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (timing rule: max over ranks)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sharded_gemm_columns(gemm, A, B, C, rank: int, world: int, device=None):
    """C = op(A) B column-sharded: `gemm(A, B_slab, C_slab)` computes this rank's
    slab in place, then an all-gather of the (column-major, contiguous) slabs
    fills all of C on every rank.  A: m x k, B: k x n, C: m x n column-major
    tensors (stride(0) == 1) on `device`.  Returns C."""
    m, n = C.shape
    j0, j1 = column_slab(n, rank, world)
    width = column_slab(n, 0, world)[1] - column_slab(n, 0, world)[0]
    if j1 > j0:
        gemm(A, B[:, j0:j1], C[:, j0:j1])
    if world == 1:
        return C
    # every rank contributes a padded slab of `width` columns (column-major, contiguous)
    send = torch.zeros((width, m), dtype=C.dtype, device=C.device)
    if j1 > j0:
        send[: j1 - j0].copy_(C[:, j0:j1].t())
    recv = torch.empty((world * width, m), dtype=C.dtype, device=C.device)
    if hasattr(dist, "all_gather_into_tensor") and dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(recv, send)
    else:
        dist.all_gather(list(recv.chunk(world)), send)
    for r in range(world):
        a, b = column_slab(n, r, world)
        if b > a:
            C[:, a:b].copy_(recv[r * width: r * width + (b - a)].t())
    return C
