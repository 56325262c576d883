"""Training workload on the library: epochs of Adam steps and the evaluation-grid errors
(S:318-388 train, S:397-423 evalmetrics; the convergence study of Table 1,
P:72-92).  Every step is the library's CUDA-graph step (sample interior and boundary points
on the device step counter, nbm_loss_grad, Adam); this module only sizes and times it.

Epoch (UniformRandom mode): N^3 interior points uniform in [-1+h0, 1-h0]^3 and
6(N+1)^2 boundary points on the faces, h0 = 2/N, split into ceil(N^3 / batch) steps.  The
library's counter-based sampler draws every step's points fresh (the same distribution as
shuffling one epoch set, without the shuffle).
"""
from __future__ import annotations

import math
import time

import numpy as np

from . import inputs, nbm


def convergence_order(e_coarse: float, e_fine: float) -> float:
    """log2(e_coarse / e_fine) for a resolution doubling."""
    if not (e_coarse > 0 and e_fine > 0):
        raise ValueError("NonPositiveError")
    return math.log2(e_coarse / e_fine)


def epoch_plan(N: int, batch: int):
    """(steps per epoch, interior points per step, boundary points per step) of an epoch of N^3
    interior and 6 (N+1)^2 boundary points in steps of at most `batch` interior points."""
    if N < 4 or N & (N - 1):
        raise ValueError("N must be a power of two >= 4 (S:324)")
    n_int, n_bnd = N ** 3, 6 * (N + 1) ** 2
    steps = max(1, math.ceil(n_int / batch))
    return steps, math.ceil(n_int / steps), math.ceil(n_bnd / steps)


def train(cfg: dict, N: int, epochs: int, batch: int = 16384, lr: float = 1e-3, seed: int = 0,
          levels: int = 1, eval_M: int | None = None, log_every: int = 0, device: int = 0,
          lr_schedule=None, return_theta: bool = False) -> dict:
    """Train the configuration's network pair at base resolution N for `epochs` epochs and
    report the RMSE / L-inf errors on the (M+1)^3 nodal grid (M = N unless eval_M).
    lr_schedule: optional [(fraction of the epochs, lr), ...] phases (one captured graph per
    phase; the Adam state and step counter run on), else a constant lr."""
    import torch
    steps_per_epoch, n, nb = epoch_plan(N, batch)
    cfg = dict(cfg)
    cfg["H"] = inputs.h_lattice(2.0 / N)
    cfg["h"] = cfg["H"] / inputs.LATTICE
    s = nbm.Solver(cfg, device, max_points=max(n, nb, 1 << 16))
    s.init_params(seed)
    dev = f"cuda:{device}"
    pts = torch.empty(n, 3, device=dev)
    bpts = torch.empty(nb, 3, device=dev)
    phases = lr_schedule or [(1.0, lr)]
    bounds, acc = [], 0.0
    for frac, plr in phases:
        acc += frac
        bounds.append((min(epochs, round(acc * epochs)), s.capture_step(pts, bpts, n_global=n, nb_global=nb, lr=plr,
                                                                         seed=seed, levels=levels)))
    bounds[-1] = (epochs, bounds[-1][1])
    rmse0, linf0 = s.error_norms(eval_M or N)
    history = []
    t_train = 0.0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    done = 0
    chunk = log_every if log_every > 0 else epochs
    while done < epochs:
        k = min(chunk, epochs - done)
        torch.cuda.synchronize(device)
        e0.record()
        for ep in range(done, done + k):
            step = next(f for b, f in bounds if ep < b)
            for _ in range(steps_per_epoch):
                step()
        e1.record()
        e1.synchronize()
        t_train += e0.elapsed_time(e1) / 1e3
        done += k
        history.append((done, float(s.loss.item())))
    rmse, linf = s.error_norms(eval_M or N)
    out = {"N": N, "h0": cfg["h"], "epochs": epochs, "batch": n, "boundary_batch": nb,
           "steps_per_epoch": steps_per_epoch, "steps": epochs * steps_per_epoch, "levels": levels, "lr": lr if lr_schedule is None else list(lr_schedule),
           "seconds": t_train, "sec_per_epoch": t_train / epochs, "rmse": rmse, "linf": linf,
           "rmse_init": rmse0, "linf_init": linf0, "eval_M": eval_M or N, "loss_history": history}
    if return_theta:
        out["theta"] = s.theta.cpu().numpy()
    s.close()
    return out


def convergence_sweep(cfg: dict, resolutions, epochs: int, **kw) -> list[dict]:
    """Table 1: train at each N, with the orders between consecutive resolutions."""
    rows = []
    for N in resolutions:
        t0 = time.time()
        r = train(cfg, N, epochs, **kw)
        r["wall_s"] = time.time() - t0
        if rows:
            r["order_rmse"] = convergence_order(rows[-1]["rmse"], r["rmse"])
            r["order_linf"] = convergence_order(rows[-1]["linf"], r["linf"])
        rows.append(r)
    return rows


def _main():
    import argparse
    import json
    ap = argparse.ArgumentParser(description="convergence sweep (Table 1, P:72-92) on the library")
    ap.add_argument("--config", default="p41")
    ap.add_argument("--N", type=int, nargs="+", default=[8, 16, 32, 64, 128])
    ap.add_argument("--epochs", type=int, default=10000)
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--levels", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--log-every", type=int, default=0)
    ap.add_argument("--decay", action="store_true",
                    help="lr phases 1e-3 (50%%), 3e-4 (25%%), 1e-4 (15%%), 3e-5 (10%%) instead of a constant lr")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    sched = [(0.5, 1e-3), (0.25, 3e-4), (0.15, 1e-4), (0.1, 3e-5)] if a.decay else None
    rows = convergence_sweep(inputs.config(a.config), a.N, a.epochs, batch=a.batch, lr=a.lr, levels=a.levels,
                             seed=a.seed, log_every=a.log_every, lr_schedule=sched)
    for r in rows:
        print(json.dumps({k: v for k, v in r.items() if k != "loss_history"}))
    if a.out:
        json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    _main()
