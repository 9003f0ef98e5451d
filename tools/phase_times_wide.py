"""Per-phase cycles of CTA 0 of the WIDE kernel (timing build): BTD_LIB=...libbtd_timing.so python tools/phase_times_wide.py N n f32|f64"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import btdgen  # noqa: E402
import paper_2601_03754_b200 as btd  # noqa: E402

N, n = int(sys.argv[1]), int(sys.argv[2])
dt = torch.float32 if sys.argv[3] == "f32" else torch.float64
variant = sys.argv[4] if len(sys.argv) > 4 else "wide"
fn = btd.lib().btd_debug_timing_wide
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 32)()
p = btdgen.dd(1, N, n, seed=1, device="cuda").cast(dt)
btd.factor_solve(p.D, p.E, p.b, variant=variant)
torch.cuda.synchronize()
fn(buf, 1)
btd.factor_solve(p.D, p.E, p.b, variant=variant)
torch.cuda.synchronize()
fn(buf, 0)
names = (["loads", "deferred", "potrf", "trsm", "l11+fill+stores", "gridsync(fwd)", "bwd task", "gridsync(bwd)"]
         if variant == "wide" else
         ["P1 tasks", "P1 sync", "P2 tasks", "P2 sync", "P3 tasks", "P3 sync", "bwd tasks", "bwd sync"])
tot = sum(buf[i] for i in range(8))
for i, nm in enumerate(names):
    print(f"{nm:18s} {buf[i]:10d} cycles {buf[i] / max(tot, 1) * 100:5.1f}%")
print("total", tot, "cycles (CTA 0)")
if variant == "persist":
    for i, nm in [(8, "  P1 diag blocks"), (9, "  P1 panel trsm"), (10, "  P1 trailing upd")]:
        print(f"{nm:18s} {buf[i]:10d} cycles")
