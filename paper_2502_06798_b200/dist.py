"""Multi-GPU plumbing around libpas (one process per GPU, torch.distributed for the bootstrap only).

The data path's single collective (the all-gather of every rank's [N x k] candidates) runs inside
libpas on NCCL; this module only
  * bootstraps the NCCL communicator: rank 0 asks libpas for an ncclUniqueId, torch.distributed
    broadcasts the bytes, every rank passes them to pas_create;
  * states the round-robin shard arithmetic (gid g lives on rank g % G at local row g // G) used to
    size each rank's store;
  * reduces a timing to the max over ranks (bench.py).
"""
from __future__ import annotations


def shard_rows(total_rows: int, world: int, rank: int) -> int:
    """Rows of a ``total_rows`` cache that rank ``rank`` of ``world`` holds (gids g with g % world == rank)."""
    return (total_rows - rank + world - 1) // world if total_rows > rank else 0


def local_to_global(local_row: int, world: int, rank: int) -> int:
    return local_row * world + rank


def bootstrap_nccl_id(rank: int, make_id=None) -> bytes:
    """Broadcast an NCCL unique id from rank 0 over the default torch.distributed group."""
    import torch.distributed as dist
    if make_id is None:
        from . import pas
        make_id = pas.pas_nccl_unique_id
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank float over the default group (identity when not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
