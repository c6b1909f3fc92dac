"""Frame sharding across ranks (one process per GPU).

Frames are independent units (reference hybrid.py:3-7), so the hot path
shards by frame index with no collective on the data path: rank r of W owns
global frames ``[first + r*per_rank, first + (r+1)*per_rank)`` of every
Eb/N0 point, and generates (or receives) only those.  Because the frame RNG
is keyed by the global index (channel.frame_rng / pc_gen_frames), the union
of the shards is exactly the single-process workload.  The only
communication is one small all-reduce per point: the error / routing
counters (sum) and the timing (max), both off the timed data path.
"""

from __future__ import annotations

COUNTER_FIELDS = ("frames", "bit_errors", "frame_errors", "frames_to_scl", "bp_iterations")


def shard_range(rank: int, world: int, per_rank: int, first: int = 0) -> tuple[int, int]:
    """Global frame indices [lo, hi) owned by ``rank``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    lo = first + rank * per_rank
    return lo, lo + per_rank


def split_total(total: int, world: int) -> list[tuple[int, int]]:
    """Contiguous near-equal split of ``total`` frames over ``world`` ranks."""
    base, extra = divmod(total, world)
    out, lo = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((lo, lo + n))
        lo += n
    return out


def merge_counters(counters: dict, group=None, device=None) -> dict:
    """Sum per-rank counters over the process group (identity when not distributed)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([int(counters.get(k, 0)) for k in COUNTER_FIELDS], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return dict(zip(COUNTER_FIELDS, (int(v) for v in t.tolist())))


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (used for the barrier-bracketed step time)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
