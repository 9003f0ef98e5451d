import sys, torch, btdgen
from paper_2601_03754_b200 import btd
prob = btdgen.kalman(12, 50, 12, seed=4).cast(torch.float32)
D, E, b = prob.D.cuda(), prob.E.cuda(), prob.b.cuda()
r1 = btd.factor_solve(D, E, b, variant="wide")
torch.cuda.synchronize()
print("done")
