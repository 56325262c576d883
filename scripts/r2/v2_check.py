"""K3w v2 sanity: bf16 W = 256 loss/grad vs the fp64 oracle and vs the v1 schedule (tooling)."""
import os, sys, time
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import numpy as np, torch
import oracle as orc
from paper_2210_14907_b200 import inputs, nbm

def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()

for nh, n, nb in [(2, 4096, 512), (3, 1000, 77), (4, 8192, 1024), (4, 37, 129), (4, 0, 200), (4, 300, 0)]:
    cfg = inputs.config("c4")
    cfg["sizes"] = [3] + [256] * nh + [1]
    pb, ar = orc.from_config(cfg)
    s = nbm.Solver(cfg, 0, max_points=max(n, nb, 1))
    pts = orc.sample(0, 5, 0, 0, n, cfg["H"]); b = orc.sample(1, 5, 0, 0, nb, cfg["H"])
    th = orc.init_params(ar, 0)
    t0 = time.time()
    loss, grad = s.loss_grad(dev(pts) if n else None, dev(b) if nb else None, theta=dev(th))
    torch.cuda.synchronize()
    st = s.status()
    gl, gg = float(loss.item()), grad.double().cpu().numpy()
    L, _, g, _ = orc.loss_grad(pb, ar, th, pts, b, cfg["h"])
    print(f"nh={nh} n={n} nb={nb} status={st} loss {gl:.6e} oracle {L:.6e} rel {abs(gl-L)/L:.2e} "
          f"grad rel {np.linalg.norm(gg-g)/np.linalg.norm(g):.2e} ({time.time()-t0:.1f}s)", flush=True)
    if n:
        s.theta.copy_(dev(th))
        u = s.eval(dev(pts[:min(n, 3000)])).double().cpu().numpy()
        want = orc.evaluate(pb, ar, th, pts[:min(n, 3000)])
        print("   eval max rel", np.abs(u - want).max() / np.abs(want).max(), flush=True)
    s.close()
