"""Multi-GPU partitioning of independent GALA layer invocations.

The GALA dot product has no cross-ciphertext exchange step: independent
inputs (and independent output-channel groups of a convolution) are
partitioned across ranks, one process per GPU, with no data-path collective
("replicas", weak scaling).  The only collectives are control-plane: the
max-over-ranks of the timed region and gathering small per-rank results.
"""
from __future__ import annotations


def shard_range(n_items: int, world: int, rank: int) -> range:
    """Contiguous, balanced block of item indices owned by `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    """Maximum of a per-rank scalar (elapsed time) across the process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_objects(obj):
    """All ranks' small result objects (e.g. output shares) on every rank."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
