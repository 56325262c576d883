"""North-star self-check 5 on the GPU path (VERDICT r1 missing-7): with the hidden layers
frozen, r is affine in the output layer (w_out, b_out of each net), so the minimiser of L
over those parameters has a closed form -- a dense least-squares solve.  The oracle probes
the affine map column by column (unit steps, fp64), numpy QR solves it; the CUDA path's
gradient with respect to the solved parameters must then vanish relative to its gradient at
the starting point, and its loss must equal the LS residual.

A few output weights per net (plus b_out) are solved for, so the solve stays well conditioned
(cond(A) ~ 1e4-1e5 at 2000 + 200 rows; the full w_out is nearly collinear and its minimiser
is then dominated by rounding).  theta* is rounded to fp32 before either side sees it.

Bars: fp32 (K3f) gradient ratio <= 1e-5 (the fp32 emulation reaches 2e-7 .. 6e-7) and loss
within 1e-5 (north_star fp32 bar); bf16 (K3t, K3w) ratio <= max(2e-2, 4 x the oracle's bf16
emulation ratio) (7e-3 .. 2.5e-2: the bf16 hidden features move the minimiser by that much),
capped at 0.1 (tests/_bars.py), and loss within 2e-2."""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm

from _bars import floor_tol

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _out_idx(sizes, n_nets, keep):
    """Indices of the first `keep` output weights and the output bias of each net (G17)."""
    P1 = inputs.param_count(sizes, 1)
    w = sizes[-2]
    idx = []
    for net in range(n_nets):
        end = (net + 1) * P1
        idx += list(range(end - w - 1, end - w - 1 + keep)) + [end - 1]
    return np.array(idx)


@pytest.mark.parametrize("sizes,prec,keep,gtol,ltol", [
    ([3, 32, 32, 1], inputs.PREC_FP32, 8, 1e-5, 1e-5),         # K3f
    ([3, 64, 64, 1], inputs.PREC_BF16, 4, 2e-2, 2e-2),         # K3t
    ([3, 256, 256, 1], inputs.PREC_BF16, 4, 2e-2, 2e-2),       # K3w
])
def test_least_squares_minimiser_zeroes_gpu_gradient(orc, sizes, prec, keep, gtol, ltol):
    cfg = inputs.config("c2")
    cfg.update(sizes=sizes, prec=prec, H=inputs.h_lattice(1 / 16))
    pb, ar = orc.from_config(cfg)
    n, nb = 2000, 200
    pts = orc.sample(0, 3, 0, 0, n, cfg["H"])
    b = orc.sample(1, 3, 0, 0, nb, cfg["H"])
    h = cfg["H"] / 2**24
    th0 = inputs.random_theta(sizes, 2, 5).astype(np.float64)
    idx = _out_idx(sizes, 2, keep)
    r0, rb0 = orc.residuals(pb, ar, th0, pts, b, h)
    base = np.concatenate([r0 / np.sqrt(n), rb0 / np.sqrt(nb)])
    cols = []
    for i in idx:
        t = th0.copy()
        t[i] += 1.0
        r1, rb1 = orc.residuals(pb, ar, t, pts, b, h)
        cols.append(np.concatenate([r1 / np.sqrt(n), rb1 / np.sqrt(nb)]) - base)
    A = np.stack(cols, 1)
    Q, R = np.linalg.qr(A)
    dx = -np.linalg.solve(R, Q.T @ base)
    Lstar = float(np.sum((A @ dx + base) ** 2))
    ts = th0.copy()
    ts[idx] += dx
    ts = ts.astype(np.float32).astype(np.float64)
    L0 = float(np.sum(base ** 2))
    assert Lstar < 0.3 * L0          # the solve moved the loss (a non-trivial check)
    _, _, g0o, _ = orc.loss_grad(pb, ar, th0, pts, b, h)
    if prec == inputs.PREC_BF16:
        _, _, gse, _ = orc.loss_grad(pb, ar, ts, pts, b, h, mode=orc.MODE_BF16)
        gtol = floor_tol(gtol, np.linalg.norm(gse[idx]) / np.linalg.norm(g0o[idx]))
        assert gtol is not None

    s = nbm.Solver(cfg, 0, max_points=n)
    dp, db = _dev(pts), _dev(b)
    l0, g0 = s.loss_grad(dp, db, theta=_dev(th0.astype(np.float32)))
    l0, g0 = float(l0.item()), g0.double().cpu().numpy().copy()   # the solver reuses its buffers
    ls, gs = s.loss_grad(dp, db, theta=_dev(ts.astype(np.float32)))
    ls, gs = float(ls.item()), gs.double().cpu().numpy().copy()
    ratio = np.linalg.norm(gs[idx]) / np.linalg.norm(g0[idx])
    assert ratio <= gtol, ratio
    assert abs(ls - Lstar) <= ltol * Lstar, (ls, Lstar)
    assert abs(l0 - L0) <= ltol * L0
    s.close()
