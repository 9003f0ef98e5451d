"""The N>1 host path of the batched benchmark on CPU with torch.distributed + gloo, world size 2.

It drives bench.py's own per-rank code (``bench.run_rank``: shard -> generate from global system
indices -> warm-up -> barrier -> timed steps -> barrier -> fp64 residual check -> statistics), the
post-timing all_gather (``shard.gather_stats``) and the whole-job aggregation and JSON line
(``shard.aggregate``, ``bench.build_line``), with the CUDA factor+solve replaced by a host stub
(the oracle's block-sparse ND Cholesky, test infrastructure only) -- SURVEY.md §8(e)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import btdgen
from paper_2601_03754_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_step_factory(prob, dev, stream):
    """Host stand-in for btd.factor_solve over the rank's batch (oracle O3 per system)."""
    from oracle import ndchol

    B, N, n, _ = prob.D.shape
    nC = sum((N >> (l - 1)) - 1 for l in range(1, N.bit_length() + 1))
    out = (torch.empty_like(prob.D), torch.empty(B, nC, n, n, dtype=prob.D.dtype), torch.empty_like(prob.b),
           torch.zeros(B, dtype=torch.int32))
    f = prob.f64()

    def step():
        for j in range(B):
            Do, Co, xo = ndchol.factor_solve(f.D[j].numpy(), f.E[j].numpy(), f.b[j].numpy())
            out[0][j] = torch.from_numpy(np.ascontiguousarray(Do))
            out[1][j] = torch.from_numpy(np.ascontiguousarray(Co))
            out[2][j] = torch.from_numpy(np.ascontiguousarray(xo))

    return step, out, None


def _worker(rank, world, port, argv, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    args = bench.parse_args(argv)
    res = bench.run_rank(args, rank, world, torch.device("cpu"), step_factory=_oracle_step_factory,
                         barrier=dist.barrier)
    allst = shard.gather_stats(res["stats"], world)
    # each rank's inputs, to check them against the single-rank batch
    p = btdgen.kalman(res["count"], bench.N_BLK, bench.N_SZ, seed=5, first_system=res["first"])
    chk = torch.tensor([float(p.D.sum()), float(p.E.sum()), float(p.b.sum()), res["first"], res["count"]],
                       dtype=torch.float64)
    allchk = [torch.empty_like(chk) for _ in range(world)]
    dist.all_gather(allchk, chk)
    if rank == 0:
        agg = shard.aggregate(allst, args.steps)
        line = bench.build_line(args, agg, res, {"hbm": 6550.0, "src": "test"})
        q.put((allst.numpy().tolist(), [c.numpy().tolist() for c in allchk], agg, line))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling,total", [("strong", 5), ("weak", 2)])
def test_two_rank_gloo_bench_path(scaling, total):
    world, steps = 2, 2
    argv = ["--gpus", "2", "--steps", str(steps), "--warmup", "3", "--scaling", scaling, "--batch", str(total),
            "--no-e2e", "--no-cpu-baseline", "--no-latency"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, argv, q)) for r in range(world)]
    for p in procs:
        p.start()
    allst, allchk, agg, line = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allst = torch.tensor(allst, dtype=torch.float64)
    per_rank = [int(r[shard.STAT_FIELDS.index("systems")]) for r in allst]
    want = [3, 2] if scaling == "strong" else [total, total]
    assert per_rank == want
    # whole-job aggregation: all systems over the slowest rank's time
    t = allst[:, 0]
    assert agg["world"] == 2 and agg["seconds_max"] == pytest.approx(float(t.max()))
    assert agg["systems"] == sum(want) * steps
    assert agg["systems_per_s"] == pytest.approx(sum(want) * steps / float(t.max()))
    assert agg["failed_systems"] == 0 and agg["max_rel_residual"] < 1e-5  # fp32 inputs, fp64 stub
    assert line["value"] == pytest.approx(agg["systems_per_s"]) and line["n_gpus"] == 2
    assert line["scaling"] == scaling and line["config"]["global_batch"] == sum(want)
    # each rank generated exactly its contiguous slice of the single-rank batch
    firsts = [int(c[3]) for c in allchk]
    assert firsts == ([0, 3] if scaling == "strong" else [0, total])
    full = btdgen.kalman(sum(want), bench.N_BLK, bench.N_SZ, seed=5)
    for r in range(world):
        sl = slice(firsts[r], firsts[r] + want[r])
        ref = [float(full.D[sl].sum()), float(full.E[sl].sum()), float(full.b[sl].sum())]
        assert allchk[r][:3] == pytest.approx(ref, rel=1e-12)


def test_shard_range():
    # strong (default): contiguous slices covering [0, B) exactly, sizes differing by at most one
    for B, G in [(8192, 1), (8192, 2), (8192, 8), (10, 4), (7, 7)]:
        sl = [shard.shard_range(r, G, B) for r in range(G)]
        assert sl[0][0] == 0 and sum(c for _, c in sl) == B
        assert all(sl[r][0] + sl[r][1] == sl[r + 1][0] for r in range(G - 1))
        assert max(c for _, c in sl) - min(c for _, c in sl) <= 1
    assert shard.shard_range(3, 8, 8192) == (3 * 1024, 1024)
    # weak: B per rank
    assert shard.shard_range(3, 4, 8192, "weak") == (3 * 8192, 8192)
    with pytest.raises(ValueError):
        shard.shard_range(4, 4, 10)
    with pytest.raises(ValueError):
        shard.shard_range(0, 4, 3)
    one = shard.gather_stats(torch.zeros(6, dtype=torch.float64), 1)
    assert one.shape == (1, 6)


def test_critical_path_floor_from_chain_latency(monkeypatch, tmp_path):
    """bench._critical_path: t_chain(n) from the microbenchmark's JSON lines and the floor
    L(N) x (t_chain + t_sync) against the measured latency (SURVEY.md §8(d) regime 1)."""
    import subprocess
    import types

    lines = ['{"n": 16, "dtype": "f64", "trsm_vectors": 32, "potrf_cyc": 3930, "trsm_cyc": 1965, '
             '"syrk_cyc": 0, "bwd_cyc": 0, "err": "no error"}',
             '{"n": 32, "dtype": "f64", "trsm_vectors": 64, "potrf_cyc": 0, "trsm_cyc": 0, "syrk_cyc": 0, '
             '"bwd_cyc": 0, "err": "too many resources"}',
             '{"gridsync_cyc": 1965, "grid": 148, "sm_khz": 1965000}']
    monkeypatch.setattr(bench.os.path, "exists", lambda p: True)
    monkeypatch.setattr(subprocess, "run", lambda *a, **k: types.SimpleNamespace(stdout="\n".join(lines)))
    lat = {"c2_fp64_n16": {"64": {"graph_warm": 30.0}}, "c3_fp64_n32": {"1024": {"graph_warm": 400.0}}}
    out = bench._critical_path(torch.device("cpu"), lat)
    assert out["gridsync_us"] == 1.0 and out["chain"]["f64_n16"]["chain_us"] == 3.0
    assert "f64_n32" not in out["chain"]                   # failed rows are dropped
    f = out["floors"]["c2_fp64_n16/N64"]                     # L(64) = 7 levels x (3 + 1) us
    assert f["floor_us"] == 28.0 and abs(f["frac"] - 28.0 / 30.0) < 1e-4
    assert "c3_fp64_n32/N1024" not in out["floors"]
