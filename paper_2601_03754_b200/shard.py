"""Batch sharding across ranks for independent systems.

Systems are independent, so the batched path shards with no collective on the data path. Two
partitions of the global system index space:

* strong (the default, BASELINE.json configs[4]: 8192 systems in total "sharded across 1/2/4/8
  B200"): rank r of G owns the contiguous slice [r*B/G, (r+1)*B/G) of the B systems (the first
  B mod G ranks take one extra system when G does not divide B);
* weak: every rank owns its own B systems, rank r the slice [r*B, (r+1)*B).

Every rank generates its systems from their GLOBAL indices, so each system's inputs -- and, the
kernels being deterministic, its outputs -- do not depend on G. The only collective is one
all_gather of a few per-rank statistics after the timed region; throughput is all systems over
the slowest rank's time.
"""
from __future__ import annotations

import torch

STAT_FIELDS = ("seconds", "kernel_ms", "max_rel_residual", "failed_systems", "e2e_seconds", "systems")


def shard_range(rank: int, world: int, total: int, scaling: str = "strong") -> tuple[int, int]:
    """(first global system index, count) owned by ``rank``.

    strong: ``total`` systems split into contiguous slices; weak: ``total`` systems per rank."""
    if not (0 <= rank < world) or total < 1:
        raise ValueError("bad shard")
    if scaling == "weak":
        return rank * total, total
    if scaling != "strong":
        raise ValueError(f"scaling must be 'strong' or 'weak', not {scaling!r}")
    if total < world:
        raise ValueError(f"{total} systems cannot be split over {world} ranks")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def gather_stats(stats: torch.Tensor, world: int) -> torch.Tensor:
    """All-gather a 1-D float64 tensor of per-rank statistics -> [world, len] (identity for world 1)."""
    if world == 1:
        return stats.reshape(1, -1)
    import torch.distributed as dist

    out = [torch.empty_like(stats) for _ in range(world)]
    dist.all_gather(out, stats)
    return torch.stack(out)


def aggregate(all_stats: torch.Tensor, steps: int) -> dict:
    """Whole-job numbers from the gathered [world, len(STAT_FIELDS)] table: every rank's systems
    over the slowest rank's time (max over ranks)."""
    world = all_stats.shape[0]
    col = {k: all_stats[:, i] for i, k in enumerate(STAT_FIELDS)}
    t_max = float(col["seconds"].max())
    systems = int(col["systems"].sum())
    e2e_max = float(col["e2e_seconds"].max())
    return {
        "world": world,
        "seconds_max": t_max,
        "systems_per_step": systems,
        "systems": systems * steps,
        "systems_per_s": systems * steps / t_max,
        "kernel_ms_max": float(col["kernel_ms"].max()),
        "max_rel_residual": float(col["max_rel_residual"].max()),
        "failed_systems": int(col["failed_systems"].sum()),
        "e2e_seconds_max": e2e_max,
    }
