"""GPU parity of the variable-coefficient assembly, sine networks and padded widths (SURVEY
8f NEXT-2; the paper's 4.1 benchmark P:68: sphere r = 0.5, u- = e^z, u+ = cos(x) sin(y),
mu- = y^2 ln(x+2) + 4, mu+ = e^{-z}, two 5 x 10 sine nets, 982 parameters), through the C ABI
against the fp64 oracle at the fp32 bars (test_gpu_parity.py's per-term rule)."""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm
from test_gpu_parity import TERMS, _dev, _parity

pytestmark = pytest.mark.gpu


def test_paper41_init_and_masks_bit_exact(orc):
    """Sine-net init (+-sqrt(6/fan_in)) and the stencil masks of the 4.1 sphere."""
    cfg = inputs.config("p41")
    s = nbm.Solver(cfg, 0, max_points=1 << 15)
    _, ar = orc.from_config(cfg)
    assert s.P == 982
    for seed in (0, 7):
        s.init_params(seed)
        assert np.array_equal(s.theta.cpu().numpy(), orc.init_params(ar, seed))
    pb, _ = orc.from_config(cfg)
    n = 1 << 15
    pts = orc.sample(0, 4, 0, 0, n, cfg["H"])
    mask = torch.empty(n, dtype=torch.uint8, device="cuda")
    cls = torch.empty(n, dtype=torch.uint8, device="cuda")
    nbm.nbm_classify(s.h, _dev(pts), n, s.h_cell, mask, cls)
    om, oc = orc.classify(pb, pts, cfg["h"])
    assert np.array_equal(mask.cpu().numpy(), om) and np.array_equal(cls.cpu().numpy(), oc)
    s.close()


@pytest.mark.parametrize("sizes,act", [([3, 10, 10, 10, 10, 10, 1], inputs.ACT_SINE),   # the paper's nets
                                       ([3, 32, 32, 32, 32, 32, 1], inputs.ACT_SINE),
                                       ([3, 64, 64, 64, 1], inputs.ACT_TANH),
                                       ([3, 20, 20, 20, 1], inputs.ACT_TANH)])
def test_paper41_parity(orc, sizes, act):
    """Loss and gradient per term on the 4.1 problem: per-point arm coefficients from mu at
    the face midpoints, crossed arms with mu at x_Gamma; sine units with
    cos(z) for act'; widths 10 and 20 run padded in the 16- and 32-wide kernels."""
    cfg = inputs.config("p41")
    cfg.update(sizes=sizes, act=act)
    lt = _parity(orc, cfg, 1 << 13, 1 << 10, seed=6, theta_seed=4)
    assert lt[2] > 0 and lt[3] > 0


@pytest.mark.parametrize("sizes", [[3, 48, 48, 48, 1], [3, 7, 7, 1]])
def test_padded_width_tanh_parity(orc, sizes):
    """Config 2 with hidden widths that are not a kernel width (48 -> 64, 7 -> 16)."""
    cfg = inputs.config("c2")
    cfg["sizes"] = sizes
    _parity(orc, cfg, 1 << 12, 1 << 9, seed=2, theta_seed=3)


def test_linear_mu_parity(orc):
    """Linear diffusion coefficients (NBM_MU_LINEAR) on config 2's pair and sphere, at h = 1/32
    where the uncrossed fp32 terms are resolved (at 1/128 they sit at the noise floor)."""
    cfg = inputs.config("c2")
    cfg.update(mu_kind=inputs.MU_LINEAR, mu_lin=np.array([[2.0, 0.3, -0.2, 0.1], [9.0, -1.0, 0.5, 2.0]], np.float32))
    cfg["H"] = inputs.h_lattice(1 / 32)
    cfg["h"] = cfg["H"] / inputs.LATTICE
    _parity(orc, cfg, 1 << 12, 1 << 9, seed=5, theta_seed=2)


def test_paper41_eval(orc):
    cfg = inputs.config("p41")
    n = 3000
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    th = inputs.random_theta(cfg["sizes"], 2, 8)
    pts = np.concatenate([orc.sample(0, 4, 0, 0, n - 100, cfg["H"]), orc.sample(1, 4, 0, 0, 100, cfg["H"])])
    s.theta.copy_(_dev(th))
    u = s.eval(_dev(pts)).double().cpu().numpy()
    assert np.allclose(u, orc.evaluate(pb, ar, th, pts), rtol=1e-5, atol=1e-6)
    s.close()


def test_variable_mu_rejected_on_split_plane_path(orc):
    cfg = inputs.config("p41")
    cfg.update(sizes=[3, 64, 64, 1], act=inputs.ACT_TANH, prec=inputs.PREC_FP32X)
    with pytest.raises(nbm.NbmError) as e:
        nbm.Solver(cfg, 0, max_points=16)
    assert e.value.code == 1


@pytest.mark.parametrize("w,nh,prec,hh", [(128, 3, inputs.PREC_BF16, 0.25), (64, 4, inputs.PREC_BF16, 0.25),
                                          (256, 3, inputs.PREC_BF16, 0.25), (128, 3, inputs.PREC_FP32, 1 / 16),
                                          (256, 2, inputs.PREC_FP32, 1 / 16)])
def test_variable_mu_tensor_core_and_wide_paths(orc, w, nh, prec, hh):
    """The section 4.1 coefficients mu-(x) = y^2 ln(x+2) + 4, mu+(x) = e^-z on K3t (bf16 W =
    64, 128), K3w (bf16 W = 256) and K3fw (fp32 W = 128, 256): per-point arm coefficients c_j/d
    (S:256 face midpoints, reading G24) in the residual epilogue.  Tanh networks with steep first
    layers at a coarse h so every term is resolved at the kernel's precision; each term and each
    parameter block against fp64 at the bar (bf16 2e-2 / fp32 1e-5, 1e-4), up to 4 x the
    oracle's own emulation floor (capped at 0.1)."""
    from _bars import check_blocks, floor_tol, rel
    cfg = inputs.config("p41")
    cfg.update(sizes=[3] + [w] * nh + [1], act=inputs.ACT_TANH, prec=prec, H=inputs.h_lattice(hh))
    cfg["h"] = cfg["H"] / inputs.LATTICE
    pb, ar = orc.from_config(cfg)
    n, nb = 2048, 256
    pts = orc.sample(0, 3, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 3, 0, 0, nb, cfg["H"])
    th = inputs.random_theta(cfg["sizes"], 2, 21)
    P1 = inputs.param_count(cfg["sizes"], 1)
    for net in range(2):
        th[net * P1:net * P1 + 3 * w] *= 16.0
    mode = orc.MODE_BF16 if prec == inputs.PREC_BF16 else orc.MODE_F32
    bl, bg = (2e-2, 2e-2) if prec == inputs.PREC_BF16 else (1e-5, 1e-4)
    L, lt, g, gt = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True)
    Le, lte, ge, gte = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True, mode=mode)
    s = nbm.Solver(cfg, 0, max_points=n)
    dth, dp, db = _dev(th), _dev(pts), _dev(bpts)
    loss, grad = s.loss_grad(dp, db, theta=dth)
    torch.cuda.synchronize()
    gl, gg = float(loss.item()), grad.double().cpu().numpy()
    assert abs(gl - L) <= floor_tol(bl, abs(Le - L) / L) * L and rel(gg, g) <= floor_tol(bg, rel(ge, g))
    assert check_blocks(gg, g, ge, cfg["sizes"], 2, bg) >= 2 * nh
    for k, term in enumerate(TERMS):
        assert lt[k] > 0, k
        tl, tg = s.loss_grad(dp, db, terms=term, theta=dth)
        torch.cuda.synchronize()
        tl, tg = float(tl.item()), tg.double().cpu().numpy()
        ltol, gtol = floor_tol(bl, abs(lte[k] - lt[k]) / lt[k]), floor_tol(bg, rel(gte[k], gt[k]))
        assert ltol is not None and gtol is not None, k
        assert abs(tl - lt[k]) <= ltol * lt[k], (k, tl, lt[k], ltol)
        assert rel(tg, gt[k]) <= gtol, (k, rel(tg, gt[k]), gtol)
    assert s.status() == 0
    s.close()
