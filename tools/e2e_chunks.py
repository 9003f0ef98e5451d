"""e2e (btd_factor_solve_host) time per step vs the number of pipeline slices, c5 workload."""
import sys, torch
sys.path.insert(0, '.')
import btdgen
import paper_2601_03754_b200 as btd
dev = torch.device('cuda:0')
B, N, n = 8192, 128, 12
p = btdgen.kalman(B, N, n, seed=5, device=dev).cast(torch.float32)
plan = btd.Plan(N, n, B, 1, torch.float32)
ws = btd.HostWorkspace(plan, device=dev)
hD, hE, hb = p.D.cpu().pin_memory(), p.E.cpu().pin_memory(), p.b.cpu().pin_memory()
s = torch.cuda.Stream(dev)
for ch in (4, 8, 16, 32, 64, 128):
    btd.factor_solve_host(hD, hE, hb, ws, chunks=ch, stream=s); s.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s)
    for _ in range(3):
        btd.factor_solve_host(hD, hE, hb, ws, chunks=ch, stream=s)
    e1.record(s); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"chunks={ch}: {ms:.2f} ms/step  {B/ms*1e3/1e3:.1f} k systems/s", flush=True)
