"""Config 4's problem on every kernel family against a closed form (tests/_zero_theta.py), not
the oracle: at theta = 0 every network value is 0, so over points whose stencils stay on one
side of the 32-sphere union the loss terms are (1/N) sum_outside (sin(x+y+z) h^2 / 2)^2, exactly 0
inside (f- = 0), and the mean of sin^2 over boundary points outside the union (P:40-41, S:256,
S:267, G2, G12, G14); the only non-zero gradient entry is the outer network's output bias,
-(2 / N_b) sum sin(x_b + y_b + z_b) (W_o = 0 blocks every other path; the uncrossed row sums
c_0 + sum_j c_j vanish).  Each term is checked on its own (the interior term is ~1e-12), in the
direct and the stable stencil form.  Kernels: K3w
(config 4's 3-256^4-1 bf16), K3h / K3t (W = 128 / 64 bf16), K3f / K3fw (fp32).  Bars: loss 2e-5
relative (fp32 sources), gradient 2e-5 of the output-bias entry."""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm

import _zero_theta

pytestmark = pytest.mark.gpu


D, S = inputs.STENCIL_DIRECT, inputs.STENCIL_STABLE


@pytest.mark.parametrize("sizes,prec,stencil", [
    ([3, 256, 256, 256, 256, 1], inputs.PREC_BF16, D),   # K3w (config 4)
    ([3, 128, 128, 128, 128, 1], inputs.PREC_BF16, D),   # K3h
    ([3, 64, 64, 64, 64, 1], inputs.PREC_BF16, D),       # K3t
    ([3, 64, 64, 64, 1], inputs.PREC_FP32, D),           # K3f
    ([3, 128, 128, 1], inputs.PREC_FP32, D),             # K3fw
    # the stable stencil form (G27): every propagated difference is 0 at theta = 0
    ([3, 256, 256, 256, 256, 1], inputs.PREC_BF16, S),   # K3w<STAB>
    ([3, 128, 128, 128, 128, 1], inputs.PREC_BF16, S),   # K3t<STAB> W = 128
    ([3, 64, 64, 64, 64, 1], inputs.PREC_BF16, S),       # K3t<STAB> W = 64
    ([3, 64, 64, 64, 1], inputs.PREC_FP32, S),           # K3f<STAB>
    ([3, 128, 128, 1], inputs.PREC_FP32, S),             # K3fw<STAB>
])
def test_config4_zero_theta_closed_form(sizes, prec, stencil):
    cfg, pts, b, h, r, rb, inside = _zero_theta.case_c4(sizes, prec)
    cfg["stencil"] = stencil
    assert inside.sum() > 50 and (~inside).sum() > 1000 and len(b) > 400
    s = nbm.Solver(cfg, 0, max_points=len(pts))
    theta = torch.zeros(s.P, dtype=torch.float32, device="cuda")
    dp, db = torch.from_numpy(pts).cuda(), torch.from_numpy(b).cuda()

    def run(terms):
        L, g = s.loss_grad(dp, db, theta=theta, terms=terms)
        return float(L.item()), g.double().cpu().numpy().copy()

    # outside the union (uncrossed): r = -sin(x+y+z) h^2 / 2; the gradient vanishes to rounding
    L, g = run(nbm.TERM_UNX_PLUS)
    want = (r * r).sum() / len(pts)
    assert abs(L - want) <= 2e-5 * want, (L, want)
    assert np.abs(g).max() <= 1e-5 * 2 * np.abs(r).mean()
    # inside (f- = 0): exactly zero
    L, g = run(nbm.TERM_UNX_MINUS)
    assert L == 0.0 and np.all(g == 0.0)
    # boundary: r_b = -g = -sin(x+y+z); only the outer network's output bias sees it
    L, g = run(nbm.TERM_BOUNDARY)
    want = (rb * rb).mean()
    assert abs(L - want) <= 2e-5 * want, (L, want)
    gbo = 2.0 * rb.mean()                     # d/d b_o of (1/N_b) sum (b_o - g)^2 at b_o = 0
    assert abs(g[-1] - gbo) <= 2e-5 * abs(gbo), (g[-1], gbo)
    assert np.abs(g[:-1]).max() <= 1e-6 * abs(gbo)
    assert s.status() == 0
    s.close()
