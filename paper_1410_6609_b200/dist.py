"""Multi-process plumbing (torch.distributed): NCCL id exchange, slab
ownership, max-over-ranks timing.  No compute happens here."""
from __future__ import annotations

from typing import Tuple


def share_nccl_id(rank: int, make_id) -> bytes:
    """Rank 0 creates the NCCL unique id (mg_nccl_unique_id), every rank gets
    it through torch.distributed (any backend, gloo included)."""
    import torch.distributed as dist
    box = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    uid = box[0]
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128
    return bytes(uid)


def slab_range(nx: int, nranks: int, rank: int) -> Tuple[int, int]:
    """x-planes [lo, hi) owned by `rank` on every distributed level of the
    finest grid (include/mg.h: rank r owns [r nx/P, (r+1) nx/P))."""
    if nx % nranks:
        raise ValueError("nx=%d not divisible by %d ranks" % (nx, nranks))
    n = nx // nranks
    return rank * n, (rank + 1) * n


def max_over_ranks(value: float, device=None) -> float:
    """MAX all-reduce of a per-rank timing."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
