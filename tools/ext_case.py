"""Run each §8(f) extension once at the bench.py sizes (after one warm-up call), for ncu launch
lists: python tools/ext_case.py [mixed|arrow|banded|partition]..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import btdgen  # noqa: E402
import paper_2601_03754_b200 as btd  # noqa: E402
from paper_2601_03754_b200 import ext, partition  # noqa: E402

dev = torch.device("cuda:0")
which = sys.argv[1:] or ["mixed", "arrow", "banded", "partition"]
B, N, n = 8192, 128, 12
for w in which:
    if w == "mixed":
        p = btdgen.kalman(B, N, n, seed=5, device=dev)
        for _ in range(2):
            ext.mixed_factor_solve(p.D, p.E, p.b, iters=2)
    elif w == "arrow":
        p = btdgen.arrow(B, N, n, 8, seed=5, device=dev).cast(torch.float32)
        for _ in range(2):
            ext.arrow_factor_solve(p.D, p.E, p.G, p.Z, p.b, p.ba)
    elif w == "banded":
        p = btdgen.banded(B, N, 4, 3, seed=5, device=dev).cast(torch.float32)
        for _ in range(2):
            ext.banded_factor_solve(p.D, p.A, p.b)
    elif w == "partition":
        p = btdgen.kalman(1, 4095, 32, seed=5, device=dev)
        for parts in (1, 2, 4, 8):
            partition.solve(p.D[0], p.E[0], p.b[0], parts)
    torch.cuda.synchronize()
print("ok")
