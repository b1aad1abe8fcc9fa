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


SC_PER_PRB = 12


def block_partition(n_slots: int, n_prb: int, world: int) -> list[dict]:
    """2-D (slot x PRB) block partition of one configured job over `world` ranks.

    a = gcd(n_slots, world) slot groups x b = world / a PRB groups; both splits are contiguous
    and balanced (sizes differ by <= 1: 273 PRBs over 4 groups -> 69/68/68/68). Rank r owns slot
    group r // b and PRB group r % b. Every (slot, PRB) is owned by exactly one rank, and each
    block is a whole number of H-units for per-subcarrier and per-PRB channels alike, so the
    shards need no exchange step. C5 (40 slots) over 8 ranks: 8 x 1, five slots per GPU -- the
    north_star's "sharded by slot across 8 GPUs"; C2 (10 slots) over 8: 2 x 4.
    Returns per rank {"slots": (s0, s1), "prbs": (p0, p1), "grid": (a, b)}."""
    import math
    if world < 1:
        raise ValueError("world must be >= 1")
    a = math.gcd(n_slots, world)
    b = world // a
    if b > n_prb:
        raise ValueError(f"cannot split {n_prb} PRBs into {b} groups")
    sl = slot_partition(n_slots, a)
    pr = slot_partition(n_prb, b)
    return [{"slots": sl[r // b], "prbs": pr[r % b], "grid": (a, b)} for r in range(world)]


def shard_arrays(H, y, n_slots: int, sc_per_h: int, block: dict, sym_per_slot: int = 14):
    """Contiguous copies of one rank's block of H [n_slots][n_fb][nr][nl] and y [n_sym][n_sc][nr]
    (numpy or torch; indexing only). Returns (H_blk, y_blk, n_sc_blk, n_slots_blk)."""
    s0, s1 = block["slots"]
    p0, p1 = block["prbs"]
    c0, c1 = p0 * SC_PER_PRB, p1 * SC_PER_PRB
    f0, f1 = c0 // sc_per_h, c1 // sc_per_h
    Hb = H[s0:s1, f0:f1]
    yb = y[s0 * sym_per_slot:s1 * sym_per_slot, c0:c1]
    if hasattr(Hb, "contiguous"):
        return Hb.contiguous(), yb.contiguous(), c1 - c0, s1 - s0
    import numpy as np
    return np.ascontiguousarray(Hb), np.ascontiguousarray(yb), c1 - c0, s1 - s0


def place_block(full, part, block: dict, sym_per_slot: int = 14):
    """Result placement: write one rank's [sym][sc][...] output block into the full grid."""
    s0, s1 = block["slots"]
    p0, p1 = block["prbs"]
    full[s0 * sym_per_slot:s1 * sym_per_slot, p0 * SC_PER_PRB:p1 * SC_PER_PRB] = part
    return full


def block_llr_shape(block: dict, full_shape, sym_per_slot: int = 14) -> tuple:
    """Shape of one rank's [sym][sc][...] output block inside the full grid `full_shape`."""
    s0, s1 = block["slots"]
    p0, p1 = block["prbs"]
    return ((s1 - s0) * sym_per_slot, (p1 - p0) * SC_PER_PRB) + tuple(full_shape[2:])


def place_blocks_p2p(local, blocks: list[dict], full_shape, dst: int = 0, sym_per_slot: int = 14):
    """Result placement (north_star: "no collective beyond result placement"): every rank sends
    its contiguous output block (torch tensor, e.g. the LLRs in its HBM) to rank `dst` point to
    point (NCCL over NVLink between GPUs; gloo on CPU in the tests), and rank `dst` writes each
    block into the full grid in its own memory. Returns the full grid on `dst`, None elsewhere.
    Not part of detection: bench.py times it separately (`placement` in the JSON line)."""
    import torch
    import torch.distributed as dist
    world = len(blocks)
    if not (dist.is_available() and dist.is_initialized()) or world == 1:
        return local
    rank = dist.get_rank()
    if rank != dst:
        dist.send(local.contiguous(), dst)
        return None
    full = torch.empty(tuple(full_shape), dtype=local.dtype, device=local.device)
    for r in range(world):
        if r == dst:
            part = local
        else:
            part = torch.empty(block_llr_shape(blocks[r], full_shape, sym_per_slot), dtype=local.dtype,
                               device=local.device)
            dist.recv(part, src=r)
        place_block(full, part, blocks[r], sym_per_slot)
    return full


def shard_seed(base_seed: int, rank: int) -> int:
    """Seed of an independently drawn per-rank workload (replica runs only; the strong-scaling
    path slices one seeded job with block_partition instead)."""
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


def gather_objects(obj, world: int, dst: int = 0):
    """Result placement for verification: gather one picklable object per rank to rank dst
    (list on dst, None elsewhere). Never inside a timed region."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or world == 1:
        return [obj]
    objs = [None] * world if dist.get_rank() == dst else None
    dist.gather_object(obj, objs, dst=dst)
    return objs


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
