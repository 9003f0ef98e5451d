"""Run one factor+solve configuration repeatedly (for ncu captures and quick timing).

python tools/run_case.py --N 128 --n 12 --batch 8192 --dtype f32 --reps 3 [--variant auto] [--time]
Inputs: btdgen ``dd`` on the device (cheap to generate; no torch kernels worth profiling)."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import btdgen  # noqa: E402
import paper_2601_03754_b200 as btd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=128)
ap.add_argument("--n", type=int, default=12)
ap.add_argument("--batch", type=int, default=8192)
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--variant", default="auto")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--time", action="store_true")
ap.add_argument("--graph", action="store_true")
a = ap.parse_args()
dt = torch.float32 if a.dtype == "f32" else torch.float64
dev = torch.device("cuda")
p = btdgen.dd(a.batch, a.N, a.n, m=a.m, seed=1, device=dev).cast(dt)
plan = btd.Plan(a.N, a.n, a.batch, a.m, dt, a.variant)
out = (torch.empty_like(p.D), torch.empty(a.batch, plan.num_coupling_blocks, a.n, a.n, dtype=dt, device=dev),
       torch.empty_like(p.b), torch.empty(a.batch, dtype=torch.int32, device=dev))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(2):
        btd.factor_solve(p.D, p.E, p.b, plan=plan, out=out, stream=s)
    s.synchronize()
    fn = lambda: btd.factor_solve(p.D, p.E, p.b, plan=plan, out=out, stream=s)  # noqa: E731
    if a.graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        fn = g.replay
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
assert int(out[3].abs().sum()) == 0
if a.time:
    med = statistics.median(ts)
    print(f"N={a.N} n={a.n} batch={a.batch} {a.dtype} variant={plan.variant} launches={plan.launches()} "
          f"median {med*1e3:.1f} us  ({a.batch / (med / 1e3):.4g} systems/s)")
