"""Table 1 diagnostic (VERDICT r1 'What's weak' 8): after training the section 4.1
problem at each N, split the loss L = (1/N)sum r^2 + (1/N_b) sum r_b^2 into its terms (uncrossed
Omega-, uncrossed Omega+, crossed, boundary) on a fresh epoch of points, with the per-point mean
r^2 of each class, at init and after training.  Under the Jacobi reading G2 an uncrossed
r = raw/d ~ -(h^2/6) Delta e for a network error e, so its mean r^2 should scale like h^4, the
crossed rows' like h^2 (r = O(h)) and the boundary's like 1: the interior PDE then barely
steers the optimiser at fine h.  Output: one JSON line per N (tooling; run on the GPU)."""
import json
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_14907_b200 import inputs, nbm, train  # noqa: E402

TERMS = [("unx_minus", nbm.TERM_UNX_MINUS), ("unx_plus", nbm.TERM_UNX_PLUS), ("crossed", nbm.TERM_CROSSED),
         ("boundary", nbm.TERM_BOUNDARY)]


def shares(cfg, N, theta):
    c = dict(cfg)
    c["H"] = inputs.h_lattice(2.0 / N)
    c["h"] = c["H"] / inputs.LATTICE
    n, nb = max(N ** 3, 4096), 6 * (N + 1) ** 2
    s = nbm.Solver(c, 0, max_points=max(n, nb))
    th = torch.from_numpy(theta).cuda()
    p = torch.empty(n, 3, device="cuda")
    b = torch.empty(nb, 3, device="cuda")
    s.sample(0, 77, 0, 0, n, p)
    s.sample(1, 77, 0, 0, nb, b)
    mask = torch.empty(n, dtype=torch.uint8, device="cuda")
    cls = torch.empty(n, dtype=torch.uint8, device="cuda")
    nbm.nbm_classify(s.h, p, n, s.h_cell, mask, cls)
    counts = np.bincount(cls.cpu().numpy(), minlength=6)
    out = {}
    for (name, term), cnt in zip(TERMS, [counts[0], counts[1], counts[2], nb]):
        loss, _ = s.loss_grad(p, b, terms=term, theta=th)
        torch.cuda.synchronize()
        L = float(loss.item())
        # per-point mean r^2 of the class (interior terms are normalised by N, the boundary by N_b)
        mean_r2 = L * (nb if name == "boundary" else n) / max(int(cnt), 1)
        out[name] = {"loss": L, "points": int(cnt), "mean_r2": mean_r2}
    tot = sum(v["loss"] for v in out.values())
    for v in out.values():
        v["share"] = v["loss"] / tot
    s.close()
    return out


def main():
    cfg = inputs.config("p41")
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    rows = []
    for N in (8, 16, 32, 64, 128):
        r = train.train(cfg, N, epochs, return_theta=True)
        th0 = nbm.Solver(cfg, 0, max_points=16)
        th0.init_params(0)
        init = th0.theta.cpu().numpy()
        th0.close()
        row = {"N": N, "h": 2.0 / N, "epochs": epochs, "rmse": r["rmse"], "linf": r["linf"],
               "trained": shares(cfg, N, r["theta"]), "init": shares(cfg, N, init)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    # slopes of log mean r^2 against log h (trained), consecutive N
    for k in range(1, len(rows)):
        a, b = rows[k - 1], rows[k]
        sl = {t: float(np.log(a["trained"][t]["mean_r2"] / b["trained"][t]["mean_r2"]) / np.log(2.0))
              for t, _ in TERMS}
        print(json.dumps({"N": [a["N"], b["N"]], "order_mean_r2_trained": sl}), flush=True)


if __name__ == "__main__":
    main()
