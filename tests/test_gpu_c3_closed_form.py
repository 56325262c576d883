"""Config 3 on the CUDA path against a closed form (tests/_zero_theta.py), not the oracle: at
theta = 0 every network value is 0, so the loss is mean (f(p) h^2 / (6 beta_s))^2 over points
whose stencils do not cross the star (G2, G13).  Config 3's own network
(3-128^4-1 SiLU, bf16: K3t) and a 3-64-64-1 SiLU one (SiLU runs on the bf16 kernels only).  The GPU forms f in fp32 (expf) and
the squares in fp64: relative bar 2e-5.  The gradient is zero up to rounding."""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm

import _zero_theta

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("sizes,prec", [([3, 128, 128, 128, 128, 1], inputs.PREC_BF16),
                                        ([3, 64, 64, 1], inputs.PREC_BF16)])
def test_config3_zero_theta_loss_closed_form(sizes, prec):
    cfg, pts, b, h, r, inside, _ = _zero_theta.case_c3(sizes, prec)
    cfg["H"] = inputs.h_lattice(h)
    assert cfg["H"] / 2**24 == h
    s = nbm.Solver(cfg, 0, max_points=len(pts))
    theta = torch.zeros(s.P, dtype=torch.float32, device="cuda")
    L, g = s.loss_grad(torch.from_numpy(pts).cuda(), torch.from_numpy(b).cuda(), theta=theta)
    L, g = float(L.item()), g.double().cpu().numpy().copy()
    want = (r * r).mean()
    assert abs(L - want) <= 2e-5 * want, (L, want)
    assert np.abs(g).max() <= 1e-5 * 2 * np.abs(r).mean()
    assert s.status() == 0
    s.close()
