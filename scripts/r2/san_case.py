"""One small call of every kernel family through the C ABI, for compute-sanitizer (tooling):
c2 fp32 (K3f), c5-w128 bf16 (K3t), c3 bf16 SiLU (K3t streamed), c4 bf16 (K3w pairs), c5-w256 fp32 (K3fw),
the stable forms, eval, Adam, multi-resolution."""
import os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import torch
from paper_2210_14907_b200 import inputs, nbm

cases = [("c2", {}), ("c5", dict(width=128)), ("c3", {}), ("c4", {}), ("c5", dict(width=256, prec=inputs.PREC_FP32)),
         ("c5", dict(width=64)), ("c2", dict(stable=True)), ("c5", dict(width=128, stable=True)), ("c4", dict(stable=True))]
for name, kw in cases:
    stable = kw.pop("stable", False)
    cfg = inputs.config(name, **kw)
    if stable:
        cfg["stencil"] = inputs.STENCIL_STABLE
    n, nb = 1 << 13, 1 << 10
    s = nbm.Solver(cfg, 0, max_points=n)
    s.init_params(0)
    p = torch.empty(n, 3, device="cuda"); b = torch.empty(nb, 3, device="cuda")
    s.sample(0, 0, 0, 0, n, p); s.sample(1, 0, 0, 0, nb, b)
    loss, _ = s.loss_grad(p, b)
    if not stable:
        s.loss_grad(p[:1000], b[:100], levels=2)
        s.eval(p[:777])
    s.adam_step()
    torch.cuda.synchronize()
    print(name, kw, "stable" if stable else "", "loss", float(loss.item()), "status", s.status(), flush=True)
    s.close()
