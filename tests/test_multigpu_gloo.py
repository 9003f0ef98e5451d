"""The N>1 host path of the batched benchmark on CPU with torch.distributed + gloo, world size 2:
sharding by global system index (inputs identical to a single-rank run), the post-timing
all_gather of per-rank statistics, and the whole-job aggregation."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import btdgen
from paper_2601_03754_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, per_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, cnt = shard.shard_range(rank, world, per_rank)
    p = btdgen.kalman(cnt, 9, 4, seed=5, first_system=first)
    # per-rank statistics: fake timing that differs by rank, a checksum of the shard's inputs
    stats = torch.tensor([1.0 + rank, 0.5 * (rank + 1), 1e-7 * (rank + 1), float(rank), 2.0],
                         dtype=torch.float64)
    allst = shard.gather_stats(stats, world)
    chk = torch.tensor([float(p.D.sum()), float(p.E.sum()), float(p.b.sum())], dtype=torch.float64)
    allchk = [torch.empty_like(chk) for _ in range(world)]
    dist.all_gather(allchk, chk)
    if rank == 0:
        q.put((allst.numpy().tolist(), [c.numpy().tolist() for c in allchk]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_aggregation():
    world, per_rank = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    allst, allchk = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allst = torch.tensor(allst, dtype=torch.float64)
    agg = shard.aggregate(allst, per_rank, steps=4)
    assert agg["world"] == 2 and agg["seconds_max"] == 2.0
    assert agg["systems"] == 2 * 3 * 4 and agg["systems_per_s"] == pytest.approx(24 / 2.0)
    assert agg["failed_systems"] == 1 and agg["max_rel_residual"] == pytest.approx(2e-7)
    # each rank generated exactly its slice of the single-rank batch
    full = btdgen.kalman(world * per_rank, 9, 4, seed=5)
    for r in range(world):
        sl = slice(r * per_rank, (r + 1) * per_rank)
        ref = [float(full.D[sl].sum()), float(full.E[sl].sum()), float(full.b[sl].sum())]
        assert allchk[r] == pytest.approx(ref, rel=1e-12)


def test_shard_range():
    assert shard.shard_range(0, 4, 8192) == (0, 8192)
    assert shard.shard_range(3, 4, 8192) == (3 * 8192, 8192)
    with pytest.raises(ValueError):
        shard.shard_range(4, 4, 10)
    one = shard.gather_stats(torch.zeros(5, dtype=torch.float64), 1)
    assert one.shape == (1, 5)
