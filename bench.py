#!/usr/bin/env python
"""Benchmark: batched factor+solve of SPD block-tridiagonal systems on B200 (BASELINE.json config c5).

One "step" = one pass of the whole hot path (load, Schur downdates, potrf,
trsm, fill gemm, forward and backward sweeps) over one batch of independent systems with
n = 12, N = 128, fp32, m = 1. The batch is 8192 systems IN TOTAL, split into contiguous slices
[r*B/G, (r+1)*B/G) over G ranks (strong scaling, BASELINE.json configs[4] / SURVEY.md §8(e));
``--scaling weak`` gives every rank its own 8192 systems instead. No collective on the data path.
Inputs are seeded synthetic ``kalman`` systems (btdgen) generated on the device before timing.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scaling strong|weak]
  torchrun --nproc-per-node N bench.py --gpus N ...

``--gpus N`` (N > 1) without a torchrun environment re-launches itself under
``torch.distributed.run`` (one process per GPU, rendezvous on 127.0.0.1). Rank 0 prints one
JSON line. ``--impl reference`` times the CPU oracle (O1, oracle/seqchol.c) on the host cores
instead (no reference implementation exists for this paper).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

B_TOTAL, N_BLK, N_SZ, M_RHS = 8192, 128, 12, 1
DTYPE = torch.float32
W_BYTES = 4
UNIT = "systems/s"


def metric_name(scaling: str) -> str:
    per = "8192 systems in total" if scaling == "strong" else "8192 systems per GPU"
    return f"batched factor+solve throughput (fp32, n=12, N=128, {per})"


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
    """Roofline denominators. HBM: the measured copy bandwidth (MEASURED_PEAKS.json). FP32/FP64 ALU
    peaks (no tensor cores on these paths): derived from the unit counts and the max SM clock,
    148 SMs x 128 FP32 / 64 FP64 FMA lanes x 2 flop."""
    out = dict(hbm=6650.0, src="fallback (B200_PROFILING.md)", mhz=1965.0)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        out.update(hbm=float(pk["hbm_gbs"]), src="measured (MEASURED_PEAKS.json)",
                   mhz=float(pk.get("sm_max_mhz", 1965.0)))
    except Exception:
        pass
    out["fp32_tflops"] = 148 * 128 * 2 * out["mhz"] * 1e6 / 1e12
    out["fp64_tflops"] = 148 * 64 * 2 * out["mhz"] * 1e6 / 1e12
    return out


def _ncu_traffic(batch: int) -> float | None:
    """Per-launch dram bytes of the dominant kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_fused_c5.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("config") == [batch, N_BLK, N_SZ, M_RHS, "fp32"]:
            return float(d["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


def _ncu_kernel_name() -> str | None:
    """Name of the dominant kernel as recorded by the committed ncu capture (profiles/ncu_fused_c5.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_fused_c5.json")) as f:
            return json.load(f).get("kernel")
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons via NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int | None, period: float = 0.01):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.ok = False
        self.max_mhz = None
        if index is None:
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _respawn_under_torchrun(nproc: int):
    """`python bench.py --gpus N` outside torchrun: re-exec as N ranks (one per GPU) on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


# ------------------------------------------------------------------ CPU oracle timing (baseline legs)

def cpu_oracle_rate(sample_systems: int, steps: int = 20, warmup: int = 3, threads: int | None = None) -> dict:
    """O1 (Alg. 1 + block substitution, plain C, fp64 accumulation; fp32 inputs upcast) on the
    host cores over `sample_systems` systems of the same workload; median over `steps` timed
    passes after `warmup` untimed ones; returns systems/s."""
    import btdgen
    from oracle import o1

    prob = btdgen.kalman(sample_systems, N_BLK, N_SZ, seed=5).cast(DTYPE).f64()
    D, E, b = prob.D.numpy(), prob.E.numpy(), prob.b.numpy()
    threads = threads or os.cpu_count() or 1
    for _ in range(warmup):
        o1.seq_batch(D, E, b, threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        _, info = o1.seq_batch(D, E, b, threads)
        times.append(time.perf_counter() - t0)
        assert not info.any()
    t = statistics.median(times)
    return dict(value=sample_systems / t, unit=UNIT, cores=threads, kind="oracle",
                sample=f"{sample_systems} kalman systems (n=12, N=128, fp32 inputs upcast to fp64), "
                       f"O1 sequential block Cholesky + solve, {threads} host threads, median of {steps} "
                       f"after {warmup} warm-up passes",
                seconds_per_step=t, times=times)


def run_reference(args):
    """The base contract's reference arm for this tier: the CPU oracle O1, as it stands, on the
    host cores; each step a bounded sample (args.ref_sample systems) of the c5 workload."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    sample = args.ref_sample
    r = cpu_oracle_rate(sample, steps=args.steps, warmup=args.warmup)
    v = r["value"]
    line = {"impl": "reference", "metric": metric_name(args.scaling), "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["seconds_per_step"] * 1e3, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (btdgen kalman, seeded)",
            "config": {"workload": "c5 batched MPC-for-RL: fp32 n=12 N=128 m=1, sampled systems on host",
                       "batch_sample": sample, "N": N_BLK, "n": N_SZ, "m": M_RHS},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ single-system latency (§8(d) regime 1)

def _l2_flusher(dev):
    """A buffer of 2x the L2 size; writing it evicts the system's data from L2."""
    try:
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    except Exception:
        l2 = 126 << 20
    buf = torch.empty(max(2 * l2, 64 << 20) // 4, dtype=torch.float32, device=dev)
    return lambda: buf.fill_(1.0)


def _latency_case(dev, s, N, n, dt, reps, flush, variant="auto"):
    import btdgen
    import paper_2601_03754_b200 as btd

    p = btdgen.kalman(1, N, n, seed=N, device=dev).cast(dt)
    plan = btd.Plan(N, n, 1, 1, dt, variant)
    outs = (torch.empty_like(p.D), torch.empty(1, plan.num_coupling_blocks, n, n, dtype=dt, device=dev),
            torch.empty_like(p.b), torch.empty(1, dtype=torch.int32, device=dev))

    def call():
        btd.factor_solve(p.D, p.E, p.b, plan=plan, out=outs, stream=s)

    def timed(fn, pre=None):
        ts = []
        for _ in range(reps):
            if pre is not None:
                pre()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return round(statistics.median(ts), 2)

    with torch.cuda.stream(s):
        for _ in range(5):
            call()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call()
        r = {"variant": plan.variant,
             "graph_warm": timed(g.replay),
             "graph_l2_flushed": timed(g.replay, flush),
             "host_launch_warm": timed(call)}
    assert int(outs[3].abs().sum()) == 0
    return r


def _latency_sweep(dev) -> dict:
    """Single-system factor+solve latency (µs) for c1, c2, the c3 N-sweep (fp32 and fp64), c4 and
    the n-sweep at N = 512: CUDA-graph replay with warm L2, graph replay after an L2 flush, and
    host-launched calls (warm); median of 50 (5 for n > 32). Each case also carries its
    throughput floor max(flops / ALU peak, bytes / HBM peak) and that floor's fraction of the
    graph-replay time (SURVEY.md §8(d) "Per-regime roofline statement")."""
    pk = _peaks()
    out = {}
    cases = [("c1_fp64_n2", 2, torch.float64, [8]), ("c2_fp64_n16", 16, torch.float64, [64]),
             ("c3_fp64_n32", 32, torch.float64, [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]),
             ("c3_fp32_n32", 32, torch.float32, [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]),
             ("c4_fp64_n128", 128, torch.float64, [256]),
             # Alg. 5 (right-looking, atomic Schur updates) against the deferred schedule (§8(f) f2)
             ("c2_fp64_n16_atomic", 16, torch.float64, [64]),
             ("c3_fp64_n32_atomic", 32, torch.float64, [64, 256, 1024]),
             ("c3_fp32_n32_atomic", 32, torch.float32, [64, 256, 1024])]
    # n-sweep at N = 512, fp64 (the paper's block-size experiment)
    nsweep = [("nsweep_fp64_N512_n%d" % n, n, torch.float64, [512]) for n in (4, 8, 12, 16, 24, 32, 48, 64, 96)]
    s = torch.cuda.Stream(dev)
    flush = _l2_flusher(dev)
    for name, n, dt, Ns in cases + nsweep:
        res = {}
        w = 8 if dt == torch.float64 else 4
        for N in Ns:
            r = _latency_case(dev, s, N, n, dt, 50 if n <= 32 else 5, flush,
                              "atomic" if name.endswith("_atomic") else "auto")
            fl = algorithmic_flops_per_system(N, n, 1)
            by = algorithmic_bytes_per_system(N, n, 1, w)["total"]
            t_fp = fl / ((pk["fp64_tflops"] if w == 8 else pk["fp32_tflops"]) * 1e12) * 1e6
            t_hbm = by / (pk["hbm"] * 1e9) * 1e6
            r["floor_us"] = round(max(t_fp, t_hbm), 3)
            r["floor_bound"] = "alu" if t_fp >= t_hbm else "hbm"
            r["floor_frac"] = round(r["floor_us"] / r["graph_warm"], 5)
            res[str(N)] = r
        out[name] = res
    return out


def _critical_path(dev, latency: dict) -> dict | None:
    """Critical-path floor of the single-system regime: t_chain(n) = measured
    potrf -> trsm -> syrk latency of ONE column op in one CTA with its blocks in shared memory,
    plus one grid.sync, from tools/micro/chain_latency (built by __graft_entry__.build()); floor(N)
    = L(N) x (t_chain + t_sync). Reported next to the graph-replay latency of the same config."""
    import subprocess

    exe = os.path.join(ROOT, "tools", "micro", "chain_latency")
    if not os.path.exists(exe):
        return None
    try:
        txt = subprocess.run([exe], capture_output=True, text=True, timeout=120,
                             env=dict(os.environ, CUDA_VISIBLE_DEVICES=str(dev.index or 0))).stdout
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}
    rows = [json.loads(l) for l in txt.splitlines() if l.startswith("{")]
    sync = next((r for r in rows if "gridsync_cyc" in r), None)
    if sync is None:
        return {"raw": rows}
    mhz = sync["sm_khz"] / 1e3
    out = {"gridsync_us": round(sync["gridsync_cyc"] / mhz, 3), "sm_mhz": mhz, "chain": {}, "floors": {}}
    for r in rows:
        if "potrf_cyc" not in r or not r["potrf_cyc"] or r.get("err", "no error") != "no error":
            continue
        cyc = r["potrf_cyc"] + r["trsm_cyc"] + r["syrk_cyc"]
        out["chain"][f"{r['dtype']}_n{r['n']}"] = dict(potrf_us=round(r["potrf_cyc"] / mhz, 3),
                                                        trsm_us=round(r["trsm_cyc"] / mhz, 3),
                                                        syrk_us=round(r["syrk_cyc"] / mhz, 3),
                                                        chain_us=round(cyc / mhz, 3))
    for name, res in latency.items():
        dt = "f64" if "fp64" in name else "f32"
        n = int(name.split("_n")[1].split("_")[0])
        key = f"{dt}_n{n}"
        if key not in out["chain"]:
            continue
        for N, r in res.items():
            L = int(N).bit_length()
            fl = L * (out["chain"][key]["chain_us"] + out["gridsync_us"])
            out["floors"][f"{name}/N{N}"] = dict(floor_us=round(fl, 2), measured_us=r["graph_warm"],
                                                 frac=round(fl / r["graph_warm"], 4))
    return out


def _ext_bench(dev) -> dict:
    """The §8(f) rows on the device: CUDA events on the launching stream, 3 warm-up calls, mean of
    `reps` calls (host-launched, outputs allocated by the binding). Systems/s or ms per call."""
    import btdgen
    import paper_2601_03754_b200 as btd
    from paper_2601_03754_b200 import ext, partition

    s = torch.cuda.Stream(dev)
    out = {}

    def timeit(fn, reps):
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                fn()
            e1.record(s)
            e1.synchronize()
        return e0.elapsed_time(e1) / reps

    def rres(D, E, x, b):
        r = btdgen.block_tridiag_matvec(D.double(), E.double(), x.double()) - b.double()
        return float((r.flatten(1).norm(dim=1) / b.double().flatten(1).norm(dim=1)).max())

    # f1: the forward sweep interlaced with the factorization ("about 12%") against a
    # separate factor then solve, on c5 and on one c3 system (fp64, n=32, N=1024)
    B = B_TOTAL
    f1 = {}
    for name, prob, plan in (
            ("c5_fp32_n12_N128_B8192", btdgen.kalman(B, N_BLK, N_SZ, seed=5, device=dev).cast(torch.float32),
             btd.Plan(N_BLK, N_SZ, B, 1, torch.float32)),
            ("c3_fp64_n32_N1024", btdgen.kalman(1, 1024, 32, seed=5, device=dev),
             btd.Plan(1024, 32, 1, 1, torch.float64))):
        o = btd.factor_solve(prob.D, prob.E, prob.b, plan=plan)
        t_fs = timeit(lambda: btd.factor_solve(prob.D, prob.E, prob.b, plan=plan, out=o, stream=s), 10)
        t_sep = timeit(lambda: (btd.factor(prob.D, prob.E, plan=plan, out=(o[0], o[1], o[3]), stream=s),
                                btd.solve(o[0], o[1], prob.b, plan=plan, out=o[2], stream=s)), 10)
        f1[name] = dict(interlaced_ms=round(t_fs, 4), separate_ms=round(t_sep, 4),
                        saving=round(1 - t_fs / t_sep, 4), variant=plan.variant)
        del o, prob
    out["f1_interlace"] = f1
    # f4a: the c5 workload with binary64 inputs: binary64 direct vs binary32 factor + refinement
    p = btdgen.kalman(B, N_BLK, N_SZ, seed=5, device=dev)
    plan32 = btd.Plan(N_BLK, N_SZ, B, 1, torch.float32)
    plan64 = btd.Plan(N_BLK, N_SZ, B, 1, torch.float64)
    work = torch.empty(ext.mixed_workspace_bytes(plan32), dtype=torch.uint8, device=dev)
    mixed = {"workload": f"{B} kalman systems, n={N_SZ}, N={N_BLK}, binary64 inputs"}
    o64 = btd.factor_solve(p.D, p.E, p.b, plan=plan64)
    ms = timeit(lambda: btd.factor_solve(p.D, p.E, p.b, plan=plan64, out=o64, stream=s), 5)
    mixed["fp64_direct"] = dict(ms=round(ms, 4), systems_per_s=B / ms * 1e3, variant=plan64.variant,
                                max_rel_residual=rres(p.D, p.E, o64[2], p.b))
    for it in (0, 1, 2, 3):
        ms = timeit(lambda: ext.mixed_factor_solve(p.D, p.E, p.b, iters=it, plan=plan32, work=work, stream=s), 5)
        x = ext.mixed_factor_solve(p.D, p.E, p.b, iters=it, plan=plan32, work=work)[2]
        mixed[f"iters{it}"] = dict(ms=round(ms, 4), systems_per_s=B / ms * 1e3,
                                   max_rel_residual=rres(p.D, p.E, x, p.b), launches=5 + 2 * it)
    out["f4a_mixed"] = mixed
    del p, o64, work
    # f4b: arrowhead, the c5 block-tridiagonal part with an 8-wide border (fp32)
    pa = btdgen.arrow(B, N_BLK, N_SZ, 8, seed=5, device=dev).cast(torch.float32)
    pla = btd.Plan(N_BLK, N_SZ, B, 9, torch.float32)
    ms = timeit(lambda: ext.arrow_factor_solve(pa.D, pa.E, pa.G, pa.Z, pa.b, pa.ba, plan=pla, stream=s), 5)
    out["f4b_arrow"] = dict(workload=f"{B} systems fp32 n={N_SZ} N={N_BLK} border na=8", ms=round(ms, 4),
                            systems_per_s=B / ms * 1e3, variant=pla.variant, launches=5)
    del pa
    # f4c: block banded, bandwidth 3, n = 4 (super-blocks of 12), fp32
    pb = btdgen.banded(B, N_BLK, 4, 3, seed=5, device=dev).cast(torch.float32)
    plb = btd.Plan(-(-N_BLK // 3), 12, B, 1, torch.float32)
    ms = timeit(lambda: ext.banded_factor_solve(pb.D, pb.A, pb.b, plan=plb, stream=s), 5)
    out["f4c_banded"] = dict(workload=f"{B} systems fp32 n=4 N={N_BLK} w=3", ms=round(ms, 4),
                             systems_per_s=B / ms * 1e3, variant=plb.variant, launches=3)
    del pb
    # f3: one long system (fp64, n = 32, N = 4095) split into p chunks. ONE GPU here: the chunks run
    # one after another, so this measures the per-chunk work, not a multi-GPU latency.
    pp = btdgen.kalman(1, 4095, 32, seed=5, device=dev)
    part = {"workload": "single system fp64 n=32 N=4095, chunks sequential on one GPU"}
    for nparts in (1, 2, 4, 8):
        ms = timeit(lambda: partition.solve(pp.D[0], pp.E[0], pp.b[0], nparts), 3)
        x, _ = partition.solve(pp.D[0], pp.E[0], pp.b[0], nparts)
        part[f"p{nparts}"] = dict(ms=round(ms, 4), max_rel_residual=rres(pp.D, pp.E, x[None], pp.b))
    out["f3_partition"] = part
    return out


# ------------------------------------------------------------------ the batched benchmark, one rank

def _pcie_bandwidth(dev, mb: int = 512) -> dict | None:
    """Pinned host <-> device copy bandwidth (GB/s), each direction alone: best of 5 copies of
    `mb` MB, CUDA events. The ceiling of the e2e number (all step bytes cross PCIe)."""
    try:
        h = torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True)
        d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
        s = torch.cuda.Stream(dev)
        out = {}
        for name, dst, src in (("h2d_gbs", d, h), ("d2h_gbs", h, d)):
            best = 0.0
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    e0.record(s)
                    dst.copy_(src, non_blocking=True)
                    e1.record(s)
                e1.synchronize()
                best = max(best, (mb << 20) / (e0.elapsed_time(e1) / 1e3) / 1e9)
            out[name] = best
        # both directions at once (separate streams and buffers): the bidirectional rate
        h2 = torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True)  # empty_like drops pinning
        d2 = torch.empty_like(d)
        s2 = torch.cuda.Stream(dev)
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            s2.wait_event(e0)
            with torch.cuda.stream(s):
                d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
            s.wait_stream(s2)
            e1.record(s)
            e1.synchronize()
            best = max(best, 2 * (mb << 20) / (e0.elapsed_time(e1) / 1e3) / 1e9)
        out["bidir_gbs"] = best
        out["how"] = (f"pinned {mb} MB copies, each direction alone and both at once on two streams, best of 5, "
                      f"CUDA events")
        return out
    except Exception:
        return None


class _CudaClock:
    """Device time with CUDA events on the launching stream."""

    def __init__(self, stream):
        self.s = stream

    def mark(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record(self.s)
        return e

    @staticmethod
    def ms(a, b) -> float:
        return a.elapsed_time(b)

    def sync(self):
        self.s.synchronize()


class _HostClock:
    """Wall time; used only by the CPU (gloo) test of the rank/aggregation path."""

    def mark(self):
        return time.perf_counter()

    @staticmethod
    def ms(a, b) -> float:
        return (b - a) * 1e3

    def sync(self):
        pass


def _gpu_step_factory(prob, dev, stream):
    """The product path: one btd_factor_solve launch over the rank's batch on `stream`."""
    import paper_2601_03754_b200 as btd

    B = prob.D.shape[0]
    plan = btd.Plan(N_BLK, N_SZ, B, M_RHS, DTYPE)
    out = (torch.empty_like(prob.D),
           torch.empty(B, plan.num_coupling_blocks, N_SZ, N_SZ, dtype=DTYPE, device=dev),
           torch.empty_like(prob.b), torch.empty(B, dtype=torch.int32, device=dev))

    def step():
        btd.factor_solve(prob.D, prob.E, prob.b, plan=plan, out=out, stream=stream)

    return step, out, plan


def run_rank(args, rank: int, world: int, dev: torch.device, step_factory=None, barrier=None) -> dict:
    """One rank of the batched benchmark: shard -> generate its systems from their global indices ->
    W warm-up steps -> barrier -> K timed steps (device clock on the launching stream) -> barrier
    -> fp64 residual check of every system -> per-rank statistics (shard.STAT_FIELDS).
    ``step_factory(prob, dev, stream) -> (step, (Dhat, C, x, info), plan)``; the default is the
    CUDA path. The CPU gloo test passes a host stub to drive the same shard/gather/aggregate code."""
    import btdgen
    from paper_2601_03754_b200 import shard

    first, B = shard.shard_range(rank, world, args.batch, args.scaling)
    prob = btdgen.kalman(B, N_BLK, N_SZ, m=M_RHS, seed=5, first_system=first, device=dev).cast(DTYPE)
    on_gpu = dev.type == "cuda"
    stream = torch.cuda.Stream(dev) if on_gpu else None
    step, out, plan = (step_factory or _gpu_step_factory)(prob, dev, stream)
    Dhat, C, x, info = out
    clock = _CudaClock(stream) if on_gpu else _HostClock()
    barrier = barrier or (lambda: None)

    for _ in range(args.warmup):
        step()
    clock.sync()
    assert int(info.abs().sum()) == 0, "factorization failed in warm-up"

    # ---- timed region: K steps, barrier + synchronize on both sides, device events on `stream`
    barrier()
    if on_gpu:
        torch.cuda.synchronize(dev)
    marks = []
    with ClockSampler(dev.index if on_gpu else None) as clk:
        t0 = clock.mark()
        for _ in range(args.steps):
            a = clock.mark()
            step()
            marks.append((a, clock.mark()))
        t1 = clock.mark()
        if on_gpu:
            torch.cuda.synchronize(dev)
    barrier()
    t_total = clock.ms(t0, t1) / 1e3
    kern_ms = [clock.ms(a, b) for a, b in marks]

    # ---- correctness check of the timed outputs (after timing): residual of every system in fp64
    r = btdgen.block_tridiag_matvec(prob.D.double(), prob.E.double(), x.double()) - prob.b.double()
    rel = (r.flatten(1).norm(dim=1) / prob.b.double().flatten(1).norm(dim=1)).max().item()
    nfail = int((info != 0).sum())

    # ---- end to end through the public host-buffer entry point (pinned host in, host out)
    e2e = None
    if on_gpu and not args.no_e2e:
        import paper_2601_03754_b200 as btd

        ws_h = btd.HostWorkspace(plan, device=dev)
        hD, hE, hb = prob.D.cpu().pin_memory(), prob.E.cpu().pin_memory(), prob.b.cpu().pin_memory()
        btd.factor_solve_host(hD, hE, hb, ws_h, chunks=args.e2e_chunks, stream=stream)
        stream.synchronize()
        barrier()
        e0 = clock.mark()
        for _ in range(args.e2e_steps):
            btd.factor_solve_host(hD, hE, hb, ws_h, chunks=args.e2e_chunks, stream=stream)
        e1 = clock.mark()
        stream.synchronize()
        h2d = (hD.numel() + hE.numel() + hb.numel()) * W_BYTES
        d2h = (Dhat.numel() + C.numel() + x.numel()) * W_BYTES + info.numel() * 4
        e2e = dict(t=clock.ms(e0, e1) / 1e3, steps=args.e2e_steps, h2d=h2d, d2h=d2h, pcie=_pcie_bandwidth(dev))
        del ws_h

    stats = torch.tensor([t_total, statistics.mean(kern_ms), rel, float(nfail), e2e["t"] if e2e else 0.0,
                          float(B)], dtype=torch.float64)
    return dict(stats=stats, e2e=e2e, clocks=clk.summary(), plan=plan, first=first, count=B)


def build_line(args, agg: dict, local: dict, pk: dict | None = None) -> dict:
    """Rank 0's JSON line from the aggregated statistics (shard.aggregate) and rank 0's extras."""
    pk = pk or _peaks()
    n = agg["world"]
    per_step = agg["systems_per_step"]
    per_rank_max = max(int(local["count"]), 1)
    ab = algorithmic_bytes_per_system()
    kern_avg_ms = agg["kernel_ms_max"]
    achieved = ab["total"] * local["count"] / (kern_avg_ms / 1e3) / 1e9 if kern_avg_ms > 0 else None
    plan = local.get("plan")
    line = {
        "metric": metric_name(args.scaling), "value": agg["systems_per_s"], "unit": UNIT, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": agg["seconds_max"] / args.steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (btdgen kalman, seeded, on device)",
        "config": {"workload": "c5 batched MPC-for-RL: independent SPD block-tridiagonal systems, fp32, n=12, "
                               "N=128, m=1 (BASELINE.json configs[4])",
                   "global_batch": per_step, "batch_per_gpu": per_rank_max if per_step % n == 0 else
                   f"{per_step // n}-{-(-per_step // n)}", "N": N_BLK, "n": N_SZ, "m": M_RHS,
                   "partition": "contiguous global-index slices [r*B/G,(r+1)*B/G)" if args.scaling == "strong"
                   else "B systems per rank, rank r owns [r*B,(r+1)*B)",
                   "parallelism": f"dp{n} (independent systems, no data-path collective)",
                   "l2": "inputs (1.25 GB at 8192 systems) and outputs exceed L2 (126 MB): no flush needed",
                   "variant": getattr(plan, "variant", None)},
        "us_per_system": agg["seconds_max"] / args.steps / per_step * 1e6 * n,
        "gpu_launches": args.steps * (plan.launches("factor_solve") if hasattr(plan, "launches") else 1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm"], "unit": "GB/s",
                     "frac": achieved / pk["hbm"] if achieved else None,
                     "traffic": _ncu_traffic(local["count"]),
                     "algorithmic_bytes_per_launch": ab["total"] * local["count"], "peak_source": pk["src"],
                     "kernel": _ncu_kernel_name(),
                     "kernel_ms_avg": kern_avg_ms},
        "flops_per_system": algorithmic_flops_per_system(),
        "check": {"max_rel_residual_fp64": agg["max_rel_residual"], "failed_systems": agg["failed_systems"]},
        "clocks": local["clocks"],
    }
    e2e = local.get("e2e")
    if e2e:
        line["e2e"] = {"value": per_step * e2e["steps"] / agg["e2e_seconds_max"], "unit": UNIT,
                       "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"], "steps": e2e["steps"],
                       "chunks": args.e2e_chunks,
                       "api": "btd_factor_solve_host (pinned host buffers, copies inside the timed region)"}
        pc = e2e.get("pcie")
        if pc:
            # the copies of one step overlap each other and the kernels: the slower direction, or both
            # directions together, bound it
            floor_s = max(e2e["h2d"] / (pc["h2d_gbs"] * 1e9), e2e["d2h"] / (pc["d2h_gbs"] * 1e9),
                          (e2e["h2d"] + e2e["d2h"]) / (pc.get("bidir_gbs", float("inf")) * 1e9))
            line["e2e"]["roofline"] = {"bound": "pcie", "h2d_gbs": pc["h2d_gbs"], "d2h_gbs": pc["d2h_gbs"],
                                       "bidir_gbs": pc.get("bidir_gbs"),
                                       "ceiling": per_step / floor_s,
                                       "frac": line["e2e"]["value"] / (per_step / floor_s),
                                       "how": pc["how"]}
    return line


def run_ours(args):
    from paper_2601_03754_b200 import shard

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        barrier = dist.barrier
    else:
        barrier = None
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    res = run_rank(args, rank, ws, dev, barrier=barrier)
    # ---- gather per-rank numbers (after timing; one NCCL all_gather of a few floats)
    allst = shard.gather_stats(res["stats"].to(dev), ws).cpu()
    if rank != 0:
        torch.distributed.destroy_process_group()
        return
    agg = shard.aggregate(allst, args.steps)
    line = build_line(args, agg, res)
    if not args.no_cpu_baseline and ws == 1:
        cb = cpu_oracle_rate(args.cpu_sample)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if args.latency and ws == 1:
        line["latency_us"] = _latency_sweep(dev)
        line["critical_path"] = _critical_path(dev, line["latency_us"])
    if args.ext and ws == 1:
        line["extensions"] = _ext_bench(dev)
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--batch", type=int, default=B_TOTAL,
                    help="systems in total (strong) or per rank (weak)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunks", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=8192)
    ap.add_argument("--ref-sample", type=int, default=1024)
    ap.add_argument("--latency", action="store_true", default=True)
    ap.add_argument("--no-latency", dest="latency", action="store_false")
    ap.add_argument("--ext", action="store_true", default=True)
    ap.add_argument("--no-ext", dest="ext", action="store_false")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    return args


def main():
    args = parse_args()
    ws, _, _ = _dist()
    if args.gpus > 1 and ws == 1 and "TORCHELASTIC_RUN_ID" not in os.environ:
        _respawn_under_torchrun(args.gpus)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
