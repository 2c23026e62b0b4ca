"""Multi-GPU layout of the batched transforms: independent
columns sharded contiguously over ranks, no data-path collective. The only
communication is the timing protocol (barrier + max over ranks)."""
from __future__ import annotations


def column_shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first column, column count) of `rank`: contiguous blocks of
    ceil(total / world) columns; trailing ranks may get fewer (or none)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("column_shard: bad world/rank")
    per = (total + world - 1) // world
    first = min(rank * per, total)
    return first, max(0, min(per, total - first))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Maximum of a per-rank scalar (device timings are reported as the max
    over ranks); identity without a process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
