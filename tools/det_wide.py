import torch, btdgen
from paper_2601_03754_b200 import btd
prob = btdgen.kalman(12, 50, 12, seed=4).cast(torch.float32)
D, E, b = prob.D.cuda(), prob.E.cuda(), prob.b.cuda()
r1 = btd.factor_solve(D, E, b, variant="wide")
bad = 0
for it in range(200):
    r2 = btd.factor_solve(D, E, b, variant="wide")
    for name, a, c in zip(("Dhat","C","x","info"), r1, r2):
        if not torch.equal(a, c):
            bad += 1
            d = (a.double() - c.double()).abs()
            idx = (d > 0).nonzero()
            print(it, name, "maxdiff", d.max().item(), "count", idx.shape[0], idx[:6].tolist())
    if bad > 10: break
sub = btd.factor_solve(D[5:9].contiguous(), E[5:9].contiguous(), b[5:9].contiguous(), variant="wide")
for name, a, c in zip(("Dhat","C","x","info"), r1, sub):
    print("sub", name, torch.equal(a[5:9], c), (a[5:9].double()-c.double()).abs().max().item())
print("bad", bad)
