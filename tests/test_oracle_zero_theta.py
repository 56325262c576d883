"""Configs 3 and 4 pinned by closed forms at theta = 0 (the oracle against the definition, not itself).

Config 3 (star interface P:60 / G13, Gaussian charges G13, beta- = 2, beta+ = 80,
alpha = sigma = g = 0) has no exact solution, so its loss has no closed form in general.  At
theta = 0 it does (tests/_zero_theta.py): u = 0 (SiLU(0) = 0, zero output weights and bias), so on
a point whose 7 stencil positions lie on one side s, r = -f(p) / d with d = 6 beta_s / h^2, and
the boundary residuals u - g vanish.  A wrong side rule, beta swap, d or source scaling moves
the loss; every gradient entry is zero up to rounding (u is flat in the hidden weights through
w_o = 0, and the uncrossed row sums c_0 + sum_j c_j vanish for the output bias)."""
import numpy as np
import pytest

from paper_2210_14907_b200 import inputs

import _zero_theta


def test_config3_loss_at_zero_theta_closed_form(orc):
    cfg, pts, b, h, r, inside, f = _zero_theta.case_c3([3, 4, 4, 1], inputs.PREC_FP32)
    assert inside.sum() > 500 and (~inside).sum() > 100
    assert np.abs(r).max() > 1e-3 * np.abs(r).mean() > 0
    pb, ar = orc.from_config(cfg)
    L, lt, g, _ = orc.loss_grad(pb, ar, np.zeros(ar.P, np.float32), pts, b, h)
    assert L == pytest.approx((r * r).mean(), rel=1e-12)
    assert lt[3] == 0.0          # boundary: u = g = 0
    # zero up to the rounding of the cotangents (2/N) r c_j / d summed over a row
    assert np.abs(g).max() <= 1e-12 * 2 * np.abs(r).mean()
    # mutation: beta swapped between the phases moves the loss by far more than the tolerance
    rs = -f * h * h / (6.0 * np.where(inside, cfg["beta"][1], cfg["beta"][0]))
    assert abs((rs * rs).mean() - L) > 1e-3 * L


def test_config4_terms_at_zero_theta_closed_form(orc):
    """Config 4's problem at theta = 0 (tests/_zero_theta.py): outside the union r = -sin(x+y+z)
    h^2 / 2, inside exactly 0, boundary r_b = -sin(x+y+z); the outer output bias alone carries
    a gradient, 2 mean(r_b)."""
    cfg, pts, b, h, r, rb, inside = _zero_theta.case_c4([3, 4, 4, 1], inputs.PREC_FP32)
    pb, ar = orc.from_config(cfg)
    th = np.zeros(ar.P, np.float32)
    L, lt, g, gt = orc.loss_grad(pb, ar, th, pts, b, h, per_term=True)
    assert lt[0] == 0.0 and np.all(gt[0] == 0.0)                      # inside: f- = 0
    assert lt[1] == pytest.approx((r * r).sum() / len(pts), rel=1e-12)
    assert lt[2] == 0.0                                               # no crossed point kept
    assert lt[3] == pytest.approx((rb * rb).mean(), rel=1e-12)
    assert g[-1] == pytest.approx(2.0 * rb.mean(), rel=1e-12)
    assert np.abs(g[:-1]).max() <= 1e-12 * 2 * np.abs(r).mean()
