import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle as orc
from paper_2210_14907_b200 import inputs, nbm
cfg = inputs.config("c5", width=128)
n = 3000
s = nbm.Solver(cfg, 0, max_points=n)
pb, ar = orc.from_config(cfg)
th = orc.init_params(ar, 1)
pts = orc.sample(0, 6, 0, 0, n, cfg["H"])
s.theta.copy_(torch.from_numpy(th).cuda())
u = s.eval(torch.from_numpy(pts).cuda()).double().cpu().numpy()
want = orc.evaluate(pb, ar, th, pts, mode=orc.MODE_BF16)
want64 = orc.evaluate(pb, ar, th, pts)
err = np.abs(u-want)
i = np.argsort(-err)[:10]
print("max err", err.max(), "at", i, u[i], want[i], want64[i])
_, cls = orc.classify(pb, pts, cfg["h"])
sides = np.array([orc.side(pb, p) for p in pts])
print("sides of worst", sides[i], "count side1", sides.sum())
print("err by side", err[sides==0].max(), err[sides==1].max())
