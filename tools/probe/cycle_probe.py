import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1302_3876_b200 as P
from paper_1302_3876_b200 import workloads as W
dev = torch.device("cuda", 0)
cyc = W.Config2Cycler(); ns, nens = cyc.ns, cyc.nens
rng = W.make_rng(0xC2)
ys = torch.from_numpy(np.stack([cyc.truth[:, None] + 0.1 * rng.standard_normal((ns, nens)) for _ in range(10)])).to(dev)
x0 = torch.from_numpy(cyc.x).to(dev); r = np.full(ns, 0.01)
model = P.Lorenz96(P.Lorenz96Config(nstate=ns))
for _ in range(2):
    res = P.cycle_l96(model, x0, ys, P.SelectionOperator.identity(), r, 5)
torch.cuda.synchronize()
print("ok")
