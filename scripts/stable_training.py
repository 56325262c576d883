"""Training at small h with the direct and the stable stencil forms: config 5's
problem (32 spheres, u- = e^x cos(y) z, u+ = sin(x+y+z), beta 1:100), two 3-64^4-1 tanh nets,
h = 2/1024, 2^18 interior + 2^15 boundary points per step, Adam lr 1e-3; the nodal-grid errors
(nbm_error_norms, M = 64) after each block of steps.  Usage: python scripts/stable_training.py [steps]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_14907_b200 import inputs, nbm  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
rows = []
for prec, stencil in ((inputs.PREC_BF16, 0), (inputs.PREC_BF16, 1), (inputs.PREC_FP32, 0), (inputs.PREC_FP32, 1)):
    cfg = inputs.config("c5", width=64, prec=prec)
    cfg.update(stencil=stencil, H=inputs.h_lattice(2.0 / 1024), N=1 << 18, Nb=1 << 15)
    cfg["h"] = cfg["H"] / inputs.LATTICE
    s = nbm.Solver(cfg, 0, max_points=cfg["N"])
    s.init_params(0)
    pts = torch.empty(cfg["N"], 3, device="cuda")
    bpts = torch.empty(cfg["Nb"], 3, device="cuda")
    step = s.capture_step(pts, bpts, lr=1e-3)
    hist = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = 0.0
    for blk in range(4):
        e0.record()
        for _ in range(steps // 4):
            step()
        e1.record()
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        rmse, linf = s.error_norms(64)
        hist.append({"steps": (blk + 1) * (steps // 4), "loss": float(s.loss.item()), "rmse": rmse, "linf": linf})
    r = {"prec": "bf16" if prec == inputs.PREC_BF16 else "fp32", "stencil": "stable" if stencil else "direct",
         "ms_per_step": ms / steps, "history": hist}
    rows.append(r)
    print(json.dumps(r), flush=True)
    s.close()
json.dump(rows, open("gpurun_out/stable_training.json", "w"), indent=1)
