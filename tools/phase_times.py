"""Per-phase cycle counts of CTA 0 of the fused-R kernel (needs the -DBTD_TIMING build):
python -m paper_2601_03754_b200.build --timing && BTD_LIB=paper_2601_03754_b200/libbtd_timing.so python tools/phase_times.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import btdgen  # noqa: E402
import paper_2601_03754_b200 as btd  # noqa: E402

L = btd.lib()
fn = L.btd_debug_timing_float
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 32)()
p = btdgen.dd(int(os.environ.get("BTD_BATCH", "8192")), 128, 12, seed=1, device="cuda").cast(torch.float32)
btd.factor_solve(p.D, p.E, p.b)
torch.cuda.synchronize()
fn(buf, 1)
btd.factor_solve(p.D, p.E, p.b)
torch.cuda.synchronize()
fn(buf, 0)
names = (["load", "phaseX(l>10)", "phaseY+bar", "backward level", "store x"] + [""] + [f"phaseX l={l}" for l in range(1, 11)]
         + ["", "", "", "", "l>=3: loads+potrf/trsm", "l>=3: stores+cache", "l>=3: fwd solve", "l>=3: SR push",
            "l>=3: F/SL", "bwd l>=3", "bwd l=2", "bwd l=1", "", "", "", ""])
tot = sum(buf[i] for i in range(16)) + sum(buf[i] for i in range(25, 28))
for i, nm in enumerate(names[:16]):
    if nm and buf[i]:
        print(f"{nm:16s} {buf[i]:10d} cycles {buf[i] / tot * 100:5.1f}%")
print("total", tot, "cycles for 1 system (CTA 0)")
for i in range(16, 32):
    if names[i] and buf[i]:
        print(f"  {names[i]:24s} {buf[i]:10d} cycles (sub-phase)")
