"""Small factor / solve / factor+solve calls of every variant for compute-sanitizer runs
(tools/sanitize.sh): racecheck, synccheck and memcheck of the owner-computes schedule."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import btdgen  # noqa: E402
import paper_2601_03754_b200 as btd  # noqa: E402

dev = torch.device("cuda")
cases = [  # (variant, batch, N, n, dtype)
    ("fused", 3, 37, 12, torch.float32),   # FUSED-R2 (c5 kernel)
    ("fused", 2, 37, 9, torch.float32),    # FUSED-R (padded)
    ("fused", 2, 19, 16, torch.float64),   # FUSED-S
    ("level", 2, 19, 6, torch.float64),
    ("persist", 2, 19, 8, torch.float64),  # PERSIST-TEAM
    ("persist", 1, 9, 40, torch.float64),  # PERSIST2
    ("wide", 1, 33, 16, torch.float64),
    ("atomic", 1, 33, 16, torch.float64),
]
for variant, B, N, n, dt in cases:
    p = btdgen.kalman(B, N, n, seed=N + n, device=dev).cast(dt)
    Dh, C, x, info = btd.factor_solve(p.D, p.E, p.b, variant=variant)
    Dh2, C2, info2 = btd.factor(p.D, p.E, variant=variant)
    x2 = btd.solve(Dh2, C2, p.b, variant=variant)
    torch.cuda.synchronize()
    assert int(info.abs().sum()) == 0 and int(info2.abs().sum()) == 0
    print(variant, B, N, n, dt, "ok", flush=True)
