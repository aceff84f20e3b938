"""Sharding across GPUs: independent codewords / stripe groups,
no collective on the data path.

Rank r of N owns the contiguous global codeword range [r * per_rank,
(r + 1) * per_rank) (weak scaling: per-rank work fixed) and generates its
inputs from (seed, global codeword index), so the union over ranks is exactly
the single-process workload of N * per_rank codewords.  The only collectives
are the barrier around the timed region and the max over ranks of the step
time (the slowest rank defines the job).
"""

from __future__ import annotations

import os


def env_rank() -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard_range(rank: int, world: int, per_rank: int) -> tuple[int, int]:
    """Global codeword range [lo, hi) owned by `rank` (weak scaling)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    return rank * per_rank, (rank + 1) * per_rank


def split_range(rank: int, world: int, total: int) -> tuple[int, int]:
    """Contiguous split of a fixed total (strong scaling), remainder spread."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity if 1 rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]
