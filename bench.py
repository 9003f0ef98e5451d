#!/usr/bin/env python
"""Benchmark: batched factor+solve of SPD block-tridiagonal systems on B200 (BASELINE.json config c5).

One "step" = one pass of the whole hot path (load, Schur downdates, potrf,
trsm, fill gemm, forward and backward sweeps) over one batch of 8192 independent systems with
n = 12, N = 128, fp32, m = 1 per GPU (weak scaling: each rank owns its own 8192 systems, no
collective on the data path). Inputs are seeded synthetic ``kalman`` systems
(btdgen) generated on the device before timing.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Rank 0 prints one JSON line. ``--impl reference`` times the CPU oracle (O1, oracle/seqchol.c)
on the host cores instead (no reference implementation exists for this paper).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

B_PER_GPU, N_BLK, N_SZ, M_RHS = 8192, 128, 12, 1
DTYPE = torch.float32
W_BYTES = 4
METRIC = "batched factor+solve throughput (fp32, n=12, N=128, 8192 systems per GPU)"
UNIT = "systems/s"


def algorithmic_bytes_per_system(N=N_BLK, n=N_SZ, m=M_RHS, w=W_BYTES) -> dict:
    """Compulsory HBM traffic of one factor+solve in the C-ABI layout:
    read D, E, b once; write Dhat (full n x n blocks, zeros above the diagonal), every coupling
    block of C and x once."""
    L = N.bit_length()
    nC = sum((N >> (l - 1)) - 1 for l in range(1, L + 1))
    rd = ((2 * N - 1) * n * n + N * n * m) * w
    wr = (N * n * n + nC * n * n + N * n * m) * w
    return dict(read=rd, write=wr, total=rd + wr, nC=nC)


def algorithmic_flops_per_system(N=N_BLK, n=N_SZ, m=M_RHS) -> float:
    """Table 1 conventions: potrf n^3/3, trsm n^3, syrk n^3, gemm 2n^3 per
    block op; solve: trsm n^2 m, gemm 2 n^2 m."""
    L = N.bit_length()
    f = 0.0
    for l in range(1, L + 1):
        s = 1 << (l - 1)
        for c in range(s, N + 1, 2 * s):
            hasL, hasR = c > s, c + s <= N
            f += n ** 3 / 3 + (hasL + hasR) * (n ** 3 + n ** 3) + (hasL and hasR) * 2 * n ** 3
            f += 2 * (n * n * m) + (hasL + hasR) * 2 * (2 * n * n * m)
    return f


def _peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return dict(hbm=float(pk["hbm_gbs"]), src="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(hbm=6650.0, src="fallback (B200_PROFILING.md)")


def _ncu_traffic() -> float | None:
    """Per-launch dram bytes of the dominant kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_fused_c5.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("config") == [B_PER_GPU, N_BLK, N_SZ, M_RHS, "fp32"]:
            return float(d["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons via NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.01):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_oracle_rate(sample_systems: int, steps: int = 1, threads: int | None = None) -> dict:
    """O1 (Alg. 1 + block substitution, plain C, fp64 accumulation; fp32 inputs upcast) on the
    host cores over `sample_systems` systems of the same workload; returns systems/s."""
    import btdgen
    from oracle import o1

    prob = btdgen.kalman(sample_systems, N_BLK, N_SZ, seed=5).cast(DTYPE).f64()
    D, E, b = prob.D.numpy(), prob.E.numpy(), prob.b.numpy()
    threads = threads or os.cpu_count() or 1
    o1.seq_batch(D[:min(64, sample_systems)], E[:min(64, sample_systems)], b[:min(64, sample_systems)], threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        _, info = o1.seq_batch(D, E, b, threads)
        times.append(time.perf_counter() - t0)
        assert not info.any()
    t = statistics.median(times)
    return dict(value=sample_systems / t, unit=UNIT, cores=threads, kind="oracle",
                sample=f"{sample_systems} kalman systems (n=12, N=128, fp32 inputs upcast to fp64), "
                       f"O1 sequential block Cholesky + solve, {threads} host threads, median of {steps}",
                seconds_per_step=t)


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    sample = args.ref_sample
    r = cpu_oracle_rate(sample, steps=args.steps)
    v = r["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["seconds_per_step"] * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (btdgen kalman, seeded)",
            "config": {"workload": "c5 batched MPC-for-RL: fp32 n=12 N=128 m=1, sampled systems on host",
                       "batch_sample": sample, "N": N_BLK, "n": N_SZ, "m": M_RHS},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _latency_sweep(dev) -> dict:
    """Single-system factor+solve latency (µs) vs N for n=32 (config c3's sweep), c1 and c2;
    CUDA-graph replay, warm L2, median of 50."""
    import btdgen
    import paper_2601_03754_b200 as btd

    out = {}
    cases = [("c1_fp64_n2", 2, torch.float64, [8]), ("c2_fp64_n16", 16, torch.float64, [64]),
             ("c3_fp64_n32", 32, torch.float64, [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]),
             ("c3_fp32_n32", 32, torch.float32, [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]),
             ("c4_fp64_n128", 128, torch.float64, [256])]
    # n-sweep at N = 512, fp64 (the paper's block-size experiment)
    nsweep = [("nsweep_fp64_N512_n%d" % n, n, torch.float64, [512]) for n in (4, 8, 12, 16, 24, 32, 48, 64, 96)]
    s = torch.cuda.Stream(dev)
    for name, n, dt, Ns in cases + nsweep:
        res = {}
        for N in Ns:
            p = btdgen.kalman(1, N, n, seed=N, device=dev).cast(dt)
            plan = btd.Plan(N, n, 1, 1, dt)
            outs = (torch.empty_like(p.D), torch.empty(1, plan.num_coupling_blocks, n, n, dtype=dt, device=dev),
                    torch.empty_like(p.b), torch.empty(1, dtype=torch.int32, device=dev))
            with torch.cuda.stream(s):
                for _ in range(3):
                    btd.factor_solve(p.D, p.E, p.b, plan=plan, out=outs)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    btd.factor_solve(p.D, p.E, p.b, plan=plan, out=outs)
                ts = []
                for _ in range(50 if n <= 32 else 5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    g.replay()
                    e1.record(s)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
            res[str(N)] = round(statistics.median(ts), 2)
            res[f"{N}_variant"] = plan.variant
        out[name] = res
    return out


def run_ours(args):
    import btdgen
    import paper_2601_03754_b200 as btd

    ws, rank, local = _dist()
    if args.gpus > 1 or ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    from paper_2601_03754_b200 import shard

    first, B = shard.shard_range(rank, max(ws, 1), args.batch)
    prob = btdgen.kalman(B, N_BLK, N_SZ, m=M_RHS, seed=5, first_system=first, device=dev).cast(DTYPE)
    D, E, b = prob.D, prob.E, prob.b
    plan = btd.Plan(N_BLK, N_SZ, B, M_RHS, DTYPE)
    Dhat = torch.empty_like(D)
    C = torch.empty(B, plan.num_coupling_blocks, N_SZ, N_SZ, dtype=DTYPE, device=dev)
    x = torch.empty_like(b)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(dev)
    out = (Dhat, C, x, info)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            btd.factor_solve(D, E, b, plan=plan, out=out, stream=stream)
    stream.synchronize()
    assert int(info.abs().sum()) == 0, "factorization failed in warm-up"

    # ---- timed region: K steps, barrier + synchronize on both sides, CUDA events on `stream`
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                ev[k][0].record(stream)
                btd.factor_solve(D, E, b, plan=plan, out=out, stream=stream)
                ev[k][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if ws > 1:
        torch.distributed.barrier()
    t_total = t_start.elapsed_time(t_end) / 1e3
    kern_ms = [a.elapsed_time(c) for a, c in ev]
    launches = args.steps * plan.launches("factor_solve")

    # ---- correctness spot check of the timed outputs (after timing): residual of every system in fp64
    r = btdgen.block_tridiag_matvec(D.double(), E.double(), x.double()) - b.double()
    rel = (r.flatten(1).norm(dim=1) / b.double().flatten(1).norm(dim=1)).max().item()
    nfail = int((info != 0).sum())

    # ---- end to end through the public host-buffer entry point (pinned host in, host out)
    e2e = None
    if not args.no_e2e:
        ws_h = btd.HostWorkspace(plan, device=dev)
        hD, hE, hb = D.cpu().pin_memory(), E.cpu().pin_memory(), b.cpu().pin_memory()
        with torch.cuda.stream(stream):
            btd.factor_solve_host(hD, hE, hb, ws_h, chunks=args.e2e_chunks, stream=stream)
        stream.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(args.e2e_steps):
                btd.factor_solve_host(hD, hE, hb, ws_h, chunks=args.e2e_chunks, stream=stream)
        e1.record(stream)
        stream.synchronize()
        t_e2e = e0.elapsed_time(e1) / 1e3
        h2d = hD.numel() * 4 + hE.numel() * 4 + hb.numel() * 4
        d2h = (Dhat.numel() + C.numel() + x.numel()) * 4 + info.numel() * 4
        e2e = dict(t=t_e2e, steps=args.e2e_steps, h2d=h2d, d2h=d2h)
        del ws_h

    # ---- gather per-rank numbers (after timing; NCCL all_gather of a few floats)
    stats = torch.tensor([t_total, statistics.mean(kern_ms), rel, float(nfail), e2e["t"] if e2e else 0.0],
                         dtype=torch.float64, device=dev)
    allst = shard.gather_stats(stats, max(ws, 1)).cpu()
    if rank != 0:
        torch.distributed.destroy_process_group()
        return
    agg = shard.aggregate(allst, B, args.steps)
    t_max = agg["seconds_max"]
    kern_avg_ms = agg["kernel_ms_max"]
    n = agg["world"]
    value = agg["systems_per_s"]
    ab = algorithmic_bytes_per_system()
    pk = _peaks()
    achieved = ab["total"] * B / (kern_avg_ms / 1e3) / 1e9
    trafficpl = _ncu_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (btdgen kalman, seeded, on device)",
        "config": {"workload": "c5 batched MPC-for-RL: 8192 independent SPD block-tridiagonal systems per GPU, "
                               "fp32, n=12, N=128, m=1 (BASELINE.json configs[4])",
                   "batch_per_gpu": B, "global_batch": B * n, "N": N_BLK, "n": N_SZ, "m": M_RHS,
                   "parallelism": f"dp{n} (independent systems, no data-path collective)",
                   "l2": "inputs (1.25 GB/GPU) and outputs larger than L2 (126 MB): no flush needed",
                   "variant": plan.variant},
        "us_per_system": t_max / args.steps / B * 1e6,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm"], "unit": "GB/s",
                     "frac": achieved / pk["hbm"], "traffic": trafficpl,
                     "algorithmic_bytes_per_launch": ab["total"] * B, "peak_source": pk["src"],
                     "kernel": "btd_fused_r_kernel<float,12,4,32,true,true,1,true>",
                     "kernel_ms_avg": kern_avg_ms},
        "flops_per_system": algorithmic_flops_per_system(),
        "check": {"max_rel_residual_fp64": agg["max_rel_residual"], "failed_systems": agg["failed_systems"]},
        "clocks": clk.summary(),
    }
    if e2e:
        t_e2e_max = agg["e2e_seconds_max"]
        line["e2e"] = {"value": n * B * e2e["steps"] / t_e2e_max, "unit": UNIT, "h2d_bytes_per_step": e2e["h2d"],
                       "d2h_bytes_per_step": e2e["d2h"], "steps": e2e["steps"], "chunks": args.e2e_chunks,
                       "api": "btd_factor_solve_host (pinned host buffers, copies inside the timed region)"}
    if not args.no_cpu_baseline:
        cb = cpu_oracle_rate(args.cpu_sample, steps=1)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if args.latency:
        line["latency_us"] = _latency_sweep(dev)
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=B_PER_GPU)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunks", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=8192)
    ap.add_argument("--ref-sample", type=int, default=1024)
    ap.add_argument("--latency", action="store_true", default=True)
    ap.add_argument("--no-latency", dest="latency", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
