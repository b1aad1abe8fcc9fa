"""Multi-GPU partitioning of the detector workload (DESIGN.md §"Multi-GPU").

H-units are independent (north_star "partitioned across the 8
B200s of one box by slot with no collective beyond result placement"): each
rank detects a contiguous block of slots on its own GPU with its own plan and
stream. There is no exchange step, so the data path has no collective; the
only torch.distributed traffic is the barrier around the timed region, the
max-over-ranks reduction of the elapsed time, and (outside any timed region)
optional result placement for verification.
"""
from __future__ import annotations


def slot_partition(n_slots: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous [start, stop) slot ranges, one per rank (sizes differ by <= 1)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(n_slots, world)
    out, s = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((s, s + n))
        s += n
    return out


def weak_slots(slots_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: rank r owns slots [r*S, (r+1)*S) of an (N*S)-slot job."""
    return rank * slots_per_rank, (rank + 1) * slots_per_rank


def shard_seed(base_seed: int, rank: int) -> int:
    """Seed of rank r's shard (each rank's slots are an independent seeded draw)."""
    return base_seed + 7919 * rank


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over all ranks (identity when torch.distributed is not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_slot_blocks(local, world: int, dst: int = 0):
    """Result placement for verification: gather each rank's [slots...] block to rank dst and
    concatenate along the slot axis (None on other ranks). Never inside a timed region."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or world == 1:
        return local
    objs = [None] * world if dist.get_rank() == dst else None
    dist.gather_object(local, objs, dst=dst)
    if dist.get_rank() != dst:
        return None
    import numpy as np
    return np.concatenate(objs, axis=0)
