"""Closed forms at theta = 0 (tests/test_oracle_c3_closed_form.py, tests/test_gpu_c3_closed_form.py,
tests/test_gpu_c4_closed_form.py): u = 0 everywhere, so on a point whose 7 stencil positions share
one side s the residual is r = -f_s(p) / d with d = 6 beta_s / h^2 (G2), and a
boundary residual is -g(p_b).  Points, sides and residuals are computed here in numpy
from the geometry and data formulas -- P:60's star (trigonometric form) and the Gaussian charges
(G13) for config 3, the union of spheres and the manufactured pair (G12, G14) for config 4 --
independently of the oracle and of the CUDA path."""
import numpy as np

from paper_2210_14907_b200 import inputs


def _phi_star(x, r0, amp, m, n):
    r = np.linalg.norm(x, axis=-1)
    th = np.arccos(np.clip(x[..., 2] / r, -1.0, 1.0))
    ph = np.arctan2(x[..., 1], x[..., 0])
    return r - r0 - amp * np.sin(m * th) * np.cos(n * ph)


def case_c3(sizes, prec, h=1.0 / 64, n=3000, seed=3):
    """-> cfg, interior points (uncrossed, one side), boundary points, h, r (fp64), inside mask"""
    cfg = inputs.config("c3")
    # config 3's eight charges plus one outside the star, so both phases carry a source
    q = np.append(cfg["charges_q"], np.float32(0.6)).astype(np.float32)
    c = np.vstack([cfg["charges_c"], np.array([[0.8, -0.75, 0.7]], np.float32)]).astype(np.float32)
    cfg.update(sizes=sizes, prec=prec, charges_q=q, charges_c=c)
    r0, amp, m, nn = [float(np.float32(v)) for v in cfg["star"]]
    rng = np.random.default_rng(seed)
    raw = c[rng.integers(0, len(c), n)].astype(np.float64) + rng.normal(0.0, 0.03, (n, 3))
    pts = (np.round(raw * 2**24) / 2**24).astype(np.float32)   # the 2^-24 lattice: arms exact
    arms = np.concatenate([np.zeros((1, 3)), h * np.vstack([np.eye(3), -np.eye(3)])])
    X = pts.astype(np.float64)[:, None, :] + arms[None, :, :]
    ph = _phi_star(X, r0, amp, m, nn)
    keep = (np.all(ph > 1e-9, axis=1) | np.all(ph < -1e-9, axis=1)) & np.all(np.abs(X) < 1 - 1e-9, axis=(1, 2))
    pts, ph = pts[keep], ph[keep]
    inside = ph[:, 0] < 0
    beta = np.where(inside, cfg["beta"][0], cfg["beta"][1]).astype(np.float64)
    s = float(np.float32(cfg["charge_sigma"]))
    d2 = ((pts.astype(np.float64)[:, None, :] - c.astype(np.float64)[None, :, :]) ** 2).sum(-1)
    f = (q.astype(np.float64)[None, :] * np.exp(-d2 / (2 * s * s))).sum(1) / ((2 * np.pi) ** 1.5 * s**3)
    r = -f * h * h / (6.0 * beta)
    b = np.array([[1.0, 0.2, -0.3], [-0.4, -1.0, 0.5], [0.1, 0.6, 1.0]], np.float32)
    return cfg, pts, b, h, r, inside, f


def case_c4(sizes, prec, n=4000, nb=600, seed=4):
    """Config 4's problem (32-sphere union, beta- = 1, beta+ = 100, the pair u- = e^x cos(y) z,
    u+ = sin(x + y + z): f- = 0, f+ = 3 beta+ sin(x + y + z), g = u+) at its own h_q.
    -> cfg, interior points (uncrossed), boundary points (outside the union), h, r, r_b"""
    cfg = inputs.config("c4")
    cfg.update(sizes=sizes, prec=prec)
    h = cfg["H"] / 2**24
    cen = cfg["centers"].astype(np.float64)
    rad = cfg["radii"].astype(np.float64)
    phi = lambda x: np.min(np.linalg.norm(x[..., None, :] - cen, axis=-1) - rad, axis=-1)
    rng = np.random.default_rng(seed)
    lim = (1 << 24) - cfg["H"]
    pts = (rng.integers(-lim, lim + 1, (n, 3)) / 2**24).astype(np.float32)   # the lattice: arms exact
    arms = np.concatenate([np.zeros((1, 3)), h * np.vstack([np.eye(3), -np.eye(3)])])
    ph = phi(pts.astype(np.float64)[:, None, :] + arms[None, :, :])
    keep = np.all(ph > 1e-9, axis=1) | np.all(ph < -1e-9, axis=1)
    pts, ph = pts[keep], ph[keep]
    inside = ph[:, 0] < 0
    xs = pts.astype(np.float64).sum(1)
    # outside: r = -3 beta+ sin(x+y+z) h^2 / (6 beta+) = -sin(x+y+z) h^2 / 2; inside f- = 0
    r = np.where(inside, 0.0, -np.sin(xs) * h * h / 2.0)
    face = rng.integers(0, 6, nb)
    b = (rng.integers(-(1 << 24), (1 << 24) + 1, (nb, 3)) / 2**24).astype(np.float32)
    b[np.arange(nb), face // 2] = np.where(face % 2 == 0, 1.0, -1.0)
    b = b[phi(b.astype(np.float64)) > 1e-9]
    rb = -np.sin(b.astype(np.float64).sum(1))
    return cfg, pts, b, h, r, rb, inside
