"""GPU parity checks added in round 2: assertions that can fail where round 1's could not.

* theta snapping (G6) through the whole path: points whose +x arm meets a plane within
  1e-6 of either end, per term against the oracle (fp32 and the bf16 tensor-core kernels).
* sticky device errors: NBM_E_DEGENERATE and NBM_E_NONFINITE on every kernel
  family.
* bf16 per-term parity at a coarse cell width (h = 1/4) with a steep network (first-layer
  weights x16): there every term's bf16 noise floor (the oracle's MODE_BF16 deviation from
  fp64) is below ~1.5e-2, so the north_star's 2e-2 bar binds on the uncrossed stencil
  epilogues of K3t (tanh and SiLU) and K3w, which at the configs' own h (2/1023, 1/512) sit
  10^4 x below bf16 resolution.
* per-block gradients: every W_l and b_l of both networks against fp64, next to the global
  L2 check (a wrong small block cannot hide under the global norm).
"""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm

from _bars import check_blocks, floor_tol, rel
from test_oracle_pins_r2 import EPS, H32, degenerate_grid_cfg

pytestmark = pytest.mark.gpu

TERMS = [nbm.TERM_UNX_MINUS, nbm.TERM_UNX_PLUS, nbm.TERM_CROSSED, nbm.TERM_BOUNDARY]
F32_LOSS, F32_GRAD, BF16 = 1e-5, 1e-4, 2e-2


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _run(s, th, p, b, terms=nbm.TERM_ALL):
    loss, grad = s.loss_grad(p, b, terms=terms, theta=th)
    torch.cuda.synchronize()
    return float(loss.item()), grad.double().cpu().numpy().copy()


H4 = 0.25


def _snap_points(n_each=40):
    """lattice points in three families w.r.t. the plane x = c, c = 0.1875 + EPS, at h = 1/4:
    the +x arm of x = 0.1875 (Omega-) meets it at theta = EPS/h (snapped), the -x arm of
    x = 0.4375 (Omega+) at 1 - EPS/h (snapped), the +x arm of x = 0.1875 - 2^-21 at
    (2^-21 + EPS)/h = 1.9e-6 (crossed)."""
    rng = np.random.default_rng(5)
    c = 0.1875 + EPS
    xs = [0.1875, 0.4375, 0.1875 - 2.0 ** -21]
    pts = []
    for x in xs:
        yz = rng.integers(-2 ** 22, 2 ** 22, size=(n_each, 2)) / 2.0 ** 23   # lattice, |.| <= 1/2
        pts.append(np.column_stack([np.full(n_each, x), yz]))
    return c, np.concatenate(pts).astype(np.float32)


@pytest.mark.parametrize("w,prec", [(64, inputs.PREC_FP32), (128, inputs.PREC_BF16), (256, inputs.PREC_BF16)])
def test_theta_snapping_gpu(orc, w, prec):
    """Snapped arms through the whole path (K2 classify -> crossed-row assembly -> fused MLP):
    at h = 1/4 with a steep network (first-layer weights x16) the snapped rows' residuals are
    resolved at the kernel's precision, so a snapped arm assembled as crossed (mu_hat, jump
    correction, far-side network) would fail the bar by orders of magnitude."""
    c, pts = _snap_points()
    cfg = inputs.config("c2")
    cfg.update(ls_kind=inputs.LS_PLANE, plane=((1.0, 0.0, 0.0), c), H=inputs.h_lattice(H4),
               sizes=[3, w, w, w, 1], prec=prec)
    cfg["h"] = cfg["H"] / inputs.LATTICE
    pb, ar = orc.from_config(cfg)
    rows = [orc.assemble(pb, p, H4) for p in pts]
    assert sum(r.n_snapped for r in rows) == 80 and sum(r.n_crossed_arms for r in rows) == 40
    _, cls = orc.classify(pb, pts, cfg["h"])
    assert (cls == 2).sum() == 120          # mixed masks: all three families take the crossed path
    th = _steep_theta(cfg["sizes"])
    mode = orc.MODE_F32 if prec == inputs.PREC_FP32 else orc.MODE_BF16
    bar_l, bar_g = (F32_LOSS, F32_GRAD) if prec == inputs.PREC_FP32 else (BF16, BF16)
    s = nbm.Solver(cfg, 0, max_points=len(pts))
    none = np.zeros((0, 3), np.float32)
    for sel in (slice(0, 120), slice(0, 80)):      # all three families; the snapped ones alone
        L, _, g, _ = orc.loss_grad(pb, ar, th, pts[sel], none, cfg["h"], n_glob=120)
        Le, _, ge, _ = orc.loss_grad(pb, ar, th, pts[sel], none, cfg["h"], n_glob=120, mode=mode)
        ltol, gtol = floor_tol(bar_l, abs(Le - L) / L), floor_tol(bar_g, rel(ge, g))
        assert ltol is not None and gtol is not None
        loss, grad = s.loss_grad(_dev(pts[sel]), None, n_global=120, theta=_dev(th))
        torch.cuda.synchronize()
        assert abs(float(loss.item()) - L) <= ltol * L, (sel, float(loss.item()), L, ltol)
        assert rel(grad.double().cpu().numpy(), g) <= gtol, (sel, gtol)
    assert s.status() == 0
    s.close()


@pytest.mark.parametrize("w,prec", [(64, inputs.PREC_FP32), (128, inputs.PREC_BF16), (256, inputs.PREC_BF16)])
def test_sticky_degenerate(orc, w, prec):
    cfg, p = degenerate_grid_cfg()
    cfg.update(sizes=[3, w, w, 1], prec=prec)
    s = nbm.Solver(cfg, 0, max_points=16)
    s.init_params(0)
    s.loss_grad(_dev(p), None)
    assert s.status() == 7                  # NBM_E_DEGENERATE
    assert s.status() == 0                  # cleared on read
    s.loss_grad(_dev(np.array([[0.75, 0.0, 0.0]], np.float32)), None)
    assert s.status() == 0
    s.close()


@pytest.mark.parametrize("w,prec", [(64, inputs.PREC_FP32), (128, inputs.PREC_FP32), (128, inputs.PREC_BF16),
                                    (256, inputs.PREC_BF16)])
def test_sticky_nonfinite(orc, w, prec):
    cfg = inputs.config("c2")
    cfg.update(sizes=[3, w, w, 1], prec=prec)
    s = nbm.Solver(cfg, 0, max_points=4096)
    s.init_params(0)
    pts = torch.empty(4096, 3, device="cuda")
    bpts = torch.empty(512, 3, device="cuda")
    s.sample(0, 0, 0, 0, 4096, pts)
    s.sample(1, 0, 0, 0, 512, bpts)
    s.loss_grad(pts, bpts)
    assert s.status() == 0
    th = s.theta.clone()
    th[5] = float("inf")                    # a layer-1 weight of net-
    s.loss_grad(pts, bpts, theta=th)
    assert s.status() == 8                  # NBM_E_NONFINITE
    assert s.status() == 0
    s.close()


def _steep_theta(sizes, scale=16.0):
    th = inputs.random_theta(sizes, 2, 21)
    P1 = inputs.param_count(sizes, 1)
    for net in range(2):
        th[net * P1:net * P1 + 3 * sizes[1]] *= scale
    return th


COARSE = [(64, 3, inputs.ACT_TANH), (128, 4, inputs.ACT_TANH), (128, 3, inputs.ACT_SILU),
          (256, 2, inputs.ACT_TANH), (256, 4, inputs.ACT_TANH)]


@pytest.mark.parametrize("w,nh,act", COARSE)
def test_bf16_coarse_h_per_term(orc, w, nh, act):
    """K3t (W = 64, 128; tanh and SiLU) and K3w (W = 256): each of the four terms and each
    parameter block at h = 1/4 on the sphere problem of config 2, where the bf16 floors are
    resolved; every asserted tolerance is <= 0.1 and most are the bar itself."""
    cfg = inputs.config("c2")
    cfg.update(sizes=[3] + [w] * nh + [1], act=act, prec=inputs.PREC_BF16, H=inputs.h_lattice(0.25))
    cfg["h"] = cfg["H"] / inputs.LATTICE
    pb, ar = orc.from_config(cfg)
    n, nb = 4096, 512
    pts = orc.sample(0, 5, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 5, 0, 0, nb, cfg["H"])
    th = _steep_theta(cfg["sizes"])
    L, lt, g, gt = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True)
    Le, lte, ge, gte = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True, mode=orc.MODE_BF16)
    s = nbm.Solver(cfg, 0, max_points=n)
    dth, dp, db = _dev(th), _dev(pts), _dev(bpts)
    gl, gg = _run(s, dth, dp, db)
    assert abs(gl - L) <= BF16 * L and rel(gg, g) <= BF16
    assert check_blocks(gg, g, ge, cfg["sizes"], 2, BF16) == 4 * (nh + 1)
    asserted = 0
    for k, term in enumerate(TERMS):
        assert lt[k] > 0, k
        tl, tg = _run(s, dth, dp, db, terms=term)
        ltol = floor_tol(BF16, abs(lte[k] - lt[k]) / lt[k])
        gtol = floor_tol(BF16, rel(gte[k], gt[k]))
        assert ltol is not None and gtol is not None, (k, lte[k], lt[k])   # resolved at this h
        assert abs(tl - lt[k]) <= ltol * lt[k], (k, tl, lt[k], ltol)
        assert rel(tg, gt[k]) <= gtol, (k, rel(tg, gt[k]), gtol)
        asserted += 1
    assert asserted == 4
    s.close()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_fp32_per_block_gradients(orc, name):
    """fp32 (K3f) per parameter block at the configs' own h: every W_l, b_l of every network
    within max(1e-4, 4 x the fp32 emulation's deviation of that block) of fp64."""
    cfg = inputs.config(name)
    n, nb = (cfg["N"], cfg["Nb"]) if name == "c1" else (1 << 14, 1 << 11)
    pb, ar = orc.from_config(cfg)
    pts = orc.sample(0, 2, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 2, 0, 0, nb, cfg["H"])
    th = inputs.random_theta(cfg["sizes"], cfg["n_nets"], 4)
    L, _, g, _ = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"])
    _, _, g32, _ = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], mode=orc.MODE_F32)
    s = nbm.Solver(cfg, 0, max_points=n)
    gl, gg = _run(s, _dev(th), _dev(pts), _dev(bpts))
    assert abs(gl - L) <= F32_LOSS * L and rel(gg, g) <= F32_GRAD
    nblk = len(cfg["sizes"]) - 1
    assert check_blocks(gg, g, g32, cfg["sizes"], cfg["n_nets"], F32_GRAD) == 2 * nblk * cfg["n_nets"]
    s.close()


def test_bf16_per_block_full_size_c4(orc):
    """config 4's network (2 x 3-256^4-1, bf16, K3w) per parameter block on 2^13 + 2^10 of its
    points at its own h: blocks within max(2e-2, 4 x the bf16 emulation's block deviation)."""
    cfg = inputs.config("c4")
    pb, ar = orc.from_config(cfg)
    n, nb = 1 << 13, 1 << 10
    pts = orc.sample(0, 8, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 8, 0, 0, nb, cfg["H"])
    th = orc.init_params(ar, 0)
    L, _, g, _ = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"])
    _, _, ge, _ = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], mode=orc.MODE_BF16)
    s = nbm.Solver(cfg, 0, max_points=n)
    gl, gg = _run(s, _dev(th), _dev(pts), _dev(bpts))
    assert abs(gl - L) <= BF16 * L and rel(gg, g) <= BF16
    assert check_blocks(gg, g, ge, cfg["sizes"], 2, BF16) == 20
    s.close()


@pytest.mark.parametrize("w,nh", [(64, 3), (128, 3)])
def test_stable_fp32_saturated_units(orc, w, nh):
    """The fp32 stable form (G27; K3f W = 64, K3fw W = 128) with saturated units and large
    differences: h = 1/4 and first-layer weights x16 put |d| = |W h e_d| far above the series
    cut 1/4 and t = tanh z near +-1, the regime where g takes the direct tanh(z + d) - t - s2 d
    branch.  Every term at the strict fp32 bars against fp64."""
    cfg = inputs.config("c2")
    cfg.update(sizes=[3] + [w] * nh + [1], prec=inputs.PREC_FP32, stencil=inputs.STENCIL_STABLE,
               H=inputs.h_lattice(0.25))
    cfg["h"] = cfg["H"] / inputs.LATTICE
    pb, ar = orc.from_config(cfg)
    n, nb = 2048, 256
    pts = orc.sample(0, 7, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 7, 0, 0, nb, cfg["H"])
    th = _steep_theta(cfg["sizes"])
    L, lt, g, gt = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True)
    s = nbm.Solver(cfg, 0, max_points=n)
    dth, dp, db = _dev(th), _dev(pts), _dev(bpts)
    gl, gg = _run(s, dth, dp, db)
    assert abs(gl - L) <= F32_LOSS * L and rel(gg, g) <= F32_GRAD
    for k, term in enumerate(TERMS):
        assert lt[k] > 0
        tl, tg = _run(s, dth, dp, db, terms=term)
        assert abs(tl - lt[k]) <= F32_LOSS * lt[k], (k, tl, lt[k])
        assert rel(tg, gt[k]) <= F32_GRAD, (k, rel(tg, gt[k]))
    s.close()
