"""Batch sharding across ranks for independent systems.

Systems are independent, so the batched path shards with no collective on the data path: rank r
of W owns systems [r*B, (r+1)*B) (weak scaling, B systems per rank) and generates them from their
GLOBAL indices, so every system's inputs -- and, the kernels being deterministic, its outputs --
do not depend on W. The only collective is one all_gather of a few per-rank statistics after the
timed region; throughput is all systems over the slowest rank's time.
"""
from __future__ import annotations

import torch

STAT_FIELDS = ("seconds", "kernel_ms", "max_rel_residual", "failed_systems", "e2e_seconds")


def shard_range(rank: int, world: int, per_rank: int) -> tuple[int, int]:
    """First global system index and count owned by ``rank`` (weak scaling)."""
    if not (0 <= rank < world) or per_rank < 1:
        raise ValueError("bad shard")
    return rank * per_rank, per_rank


def gather_stats(stats: torch.Tensor, world: int) -> torch.Tensor:
    """All-gather a 1-D float64 tensor of per-rank statistics -> [world, len] (identity for world 1)."""
    if world == 1:
        return stats.reshape(1, -1)
    import torch.distributed as dist

    out = [torch.empty_like(stats) for _ in range(world)]
    dist.all_gather(out, stats)
    return torch.stack(out)


def aggregate(all_stats: torch.Tensor, per_rank: int, steps: int) -> dict:
    """Whole-job numbers from the gathered [world, len(STAT_FIELDS)] table."""
    world = all_stats.shape[0]
    t_max = float(all_stats[:, 0].max())
    return {
        "world": world,
        "seconds_max": t_max,
        "systems": world * per_rank * steps,
        "systems_per_s": world * per_rank * steps / t_max,
        "kernel_ms_max": float(all_stats[:, 1].max()),
        "max_rel_residual": float(all_stats[:, 2].max()),
        "failed_systems": int(all_stats[:, 3].sum()),
        "e2e_seconds_max": float(all_stats[:, 4].max()),
    }
