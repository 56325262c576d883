"""Pins of the oracle's variable-coefficient assembly and of the paper's 4.1 benchmark
(sphere r = 0.5, u- = e^z, u+ = cos(x) sin(y), mu- = y^2 ln(x+2) + 4, mu+ = e^{-z},
two 5 x 10 sine nets, 982 parameters)."""
import numpy as np
import pytest

from paper_2210_14907_b200 import inputs
import test_oracle_assembly as A


def _lin_cfg(mu_lin, k=(0.0, 0.0)):
    cfg = A._poly_cfg(k=k)
    cfg.update(mu_kind=inputs.MU_LINEAR, mu_lin=np.asarray(mu_lin, np.float32))
    return cfg


@pytest.mark.parametrize("k", [0.0, 2.0])
def test_linear_mu_quadratic_exactness(orc, k):
    """S:256 face-midpoint flux: for quadratic u and linear mu the flux difference
    (mu(x+h/2) (u1 - u0) - mu(x-h/2) (u0 - u-1)) / h^2 equals (mu u')' exactly, so with
    f = k u - mu Lap u - grad mu . grad u the uncrossed row's raw is 0 to round-off."""
    rng = np.random.default_rng(3)
    for trial in range(12):
        q = rng.normal(size=10)
        poly = np.concatenate([q, q])
        m = np.array([3.0, *rng.uniform(-0.8, 0.8, 3)], np.float32)
        cfg = _lin_cfg([m, m], k=(k, k))
        pb, _ = orc.from_config(cfg, poly=poly)
        H = inputs.h_lattice(rng.choice([1 / 8, 1 / 32, 1 / 128]))
        for p in inputs.random_lattice_points(20, H, seed=trial):
            row = orc.assemble(pb, p, H / 2**24)
            raw, scale = A._raw(row, A._poly_u(poly))
            assert abs(raw) <= 2e-13 * scale
            # centre coefficient = k + sum of the face coefficients (row sums to k)
            assert abs(sum(row.coef[j] for j in range(7)) - float(np.float32(k))) <= 1e-12 * row.d


def test_variable_mu_constant_annihilation(orc):
    """With k = 0 the centre coefficient equals minus the sum of the arm coefficients (the
    face values enter both), for the 4.1 fields on both sides of the sphere."""
    cfg = inputs.config("p41")
    pb, _ = orc.from_config(cfg)
    for p in inputs.random_lattice_points(200, cfg["H"], seed=1):
        row = orc.assemble(pb, p, cfg["h"])
        if row.crossed:
            continue
        assert abs(row.coef[0] + sum(row.coef[j] for j in range(1, 7))) <= 1e-12 * row.d


def _fd(fn, x, e=1e-4):
    g = np.zeros(3)
    for d in range(3):
        yp, ym = np.array(x, float), np.array(x, float)
        yp[d] += e
        ym[d] -= e
        g[d] = (fn(yp) - fn(ym)) / (2 * e)
    return g


def _u41(s, x):
    return np.exp(x[2]) if s == 0 else np.cos(x[0]) * np.sin(x[1])


def _mu41(s, x):
    return x[1] ** 2 * np.log(x[0] + 2.0) + 4.0 if s == 0 else np.exp(-x[2])


def test_paper41_fields_source_and_jumps(orc):
    """P:68's fields written out independently: u, mu; f = -div(mu grad u) by central
    differences of the flux mu grad u; alpha = u+ - u-, sigma = mu+ d_n u+ - mu- d_n u-."""
    cfg = inputs.config("p41")
    pb, _ = orc.from_config(cfg)
    rng = np.random.default_rng(5)
    for x in rng.uniform(-0.9, 0.9, size=(30, 3)):
        for s in (0, 1):
            assert abs(orc.exact(pb, s, x)[0] - _u41(s, x)) <= 1e-14
            assert abs(orc.mu(pb, s, x)[0] - _mu41(s, x)) <= 1e-13
            flux = lambda y, d: _mu41(s, y) * _fd(lambda z: _u41(s, z), y, 1e-5)[d]
            div = sum(_fd(lambda y: flux(y, d), x, 1e-3)[d] for d in range(3))
            assert abs(orc.f(pb, s, x) - (-div)) <= 2e-5 * max(1.0, abs(div))
    for _ in range(30):
        v = rng.normal(size=3)
        x = 0.5 * v / np.linalg.norm(v)
        n = orc.normal(pb, x)
        assert abs(orc.alpha(pb, x) - (_u41(1, x) - _u41(0, x))) <= 1e-14
        dn = [_fd(lambda y: _u41(s, y), x, 1e-5) @ n for s in (0, 1)]
        assert abs(orc.sigma(pb, x, n) - (_mu41(1, x) * dn[1] - _mu41(0, x) * dn[0])) <= 1e-8


def test_paper41_boundary_example(orc):
    """sphere case, p_b = (1,0,0): g = cos(1) sin(0) = 0, so the residual is the plus
    network's value there."""
    pb, _ = orc.from_config(inputs.config("p41"))
    assert orc.side(pb, [1.0, 0.0, 0.0]) == 1
    assert orc.g(pb, [1.0, 0.0, 0.0]) == 0.0
    assert orc.g(pb, [1.0, 0.5, 0.2]) == pytest.approx(np.cos(1.0) * np.sin(0.5), abs=1e-15)


def test_paper41_truncation_orders(orc):
    """S:262 example 3 on the 4.1 problem: with the exact solution substituted, uncrossed raw
    shrinks at order 2 (ratio 4 +- 25 % per halving) from h = 2/8 to 2/64; crossed r stays
    bounded and does not grow."""
    cfg = inputs.config("p41")
    pb, _ = orc.from_config(cfg)
    unx, crs = [], []
    for h in (2 / 8, 2 / 16, 2 / 32, 2 / 64):
        H = inputs.h_lattice(h)
        raw, r, cls = orc.residual_exact(pb, inputs.random_lattice_points(10000, H, seed=5), H / 2**24)
        unx.append(np.abs(raw[cls < 2]).max())
        crs.append(np.abs(r[cls == 2]).max())
    orders = np.log2(np.array(unx[:-1]) / np.array(unx[1:]))
    assert np.all(np.abs(orders - 2.0) < np.log2(1.25))
    assert all(crs[i + 1] <= crs[i] * 1.25 for i in range(len(crs) - 1))


def test_paper41_parameters_and_sine_init(orc):
    """S:178 / P:68: two [3,10,10,10,10,10,1] nets = 982 parameters; sine-net init uniform
    +-sqrt(6/fan_in) with zero biases."""
    cfg = inputs.config("p41")
    _, ar = orc.from_config(cfg)
    assert ar.P == 982
    th = orc.init_params(ar, 0)
    off = 0
    for _ in range(2):
        for l in range(1, 7):
            fi, fo = cfg["sizes"][l - 1], cfg["sizes"][l]
            w = th[off:off + fi * fo]
            amp = np.float32(np.sqrt(np.float32(6.0) / np.float32(fi)))
            assert np.abs(w).max() <= amp and (fi * fo < 30 or np.abs(w).max() > 0.7 * amp)
            assert np.all(th[off + fi * fo: off + fi * fo + fo] == 0)
            off += fi * fo + fo


def test_paper41_loss_gradient_matches_central_differences(orc):
    """S:281 example 3: the full-loss gradient over all 982 parameters matches central
    finite differences (step 1e-6, rel < 1e-5) on a 10-point batch of crossed and uncrossed
    points with boundary points, variable mu and sine nets."""
    cfg = inputs.config("p41")
    pb, ar = orc.from_config(cfg)
    cand = inputs.random_lattice_points(4000, cfg["H"], 9)
    _, cls = orc.classify(pb, cand, cfg["h"])
    pts = np.concatenate([cand[cls == 2][:5], cand[cls < 2][:5]])
    b = orc.sample(1, 2, 0, 0, 4, cfg["H"])
    th = orc.init_params(ar, 3).astype(np.float64) + np.random.default_rng(1).normal(size=ar.P) * 0.1
    L, lt, g, _ = orc.loss_grad(pb, ar, th, pts, b, cfg["h"])
    assert lt[2] > 0 and (lt[0] + lt[1]) > 0 and lt[3] > 0
    fd = np.zeros(ar.P)
    for i in range(ar.P):
        tp, tm = th.copy(), th.copy()
        tp[i] += 1e-6
        tm[i] -= 1e-6
        fd[i] = (orc.loss_grad(pb, ar, tp, pts, b, cfg["h"])[0] - orc.loss_grad(pb, ar, tm, pts, b, cfg["h"])[0]) / 2e-6
    scale = np.abs(g).max()
    assert np.all(np.abs(g - fd) <= 1e-5 * np.maximum(np.abs(g), 1e-3 * scale))
