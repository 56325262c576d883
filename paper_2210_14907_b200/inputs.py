"""Seeded synthetic workload definitions shared by the CUDA path's harness and
the oracle's tests.

This module holds NONE of the method's arithmetic: it only lists the five
BASELINE.json configurations as plain parameters and draws their random
problem data (sphere centres/radii for config 4, charges for config 3) and
random parameter vectors with numpy's seeded generator.  Both sides receive
the same fp32 arrays.  The recipe is stated in DESIGN.md ("Inputs").
"""
from __future__ import annotations

import numpy as np

LATTICE = 1 << 24  # coordinates and h are multiples of 2^-24 (G9)

LS_NONE, LS_SPHERES, LS_STAR, LS_PLANE, LS_GRID = 0, 1, 2, 3, 4
SRC_SINE3PI, SRC_PAIR, SRC_GAUSS, SRC_PAPER41 = 0, 1, 2, 4
MU_CONST, MU_PAPER41, MU_LINEAR = 0, 1, 2
ACT_TANH, ACT_SILU, ACT_SINE = 0, 1, 2
PREC_FP32, PREC_BF16, PREC_FP32X = 0, 1, 2
STENCIL_DIRECT, STENCIL_STABLE = 0, 1


def h_lattice(h: float) -> int:
    """H such that h_q = H * 2^-24 (G9)."""
    return int(round(h * LATTICE))


def _config4_spheres(seed: int = 0):
    # BASELINE config 4: 32 spheres, radius ~ U[0.05, 0.2], centres ~ U[-0.8, 0.8]^3
    rng = np.random.default_rng(np.random.SeedSequence([seed, 4]))
    centers = rng.uniform(-0.8, 0.8, size=(32, 3)).astype(np.float32)
    radii = rng.uniform(0.05, 0.2, size=32).astype(np.float32)
    return centers, radii


def _config3_charges(seed: int = 0):
    # BASELINE config 3: 8 charges, q ~ U[-1,1], centres inside phi < 0.  The star
    # r - 0.5 - 0.15 sin5t cos3p has r >= 0.35 on Gamma, so centres drawn uniformly
    # in the ball |c| < 0.3 lie inside without evaluating the level set.
    rng = np.random.default_rng(np.random.SeedSequence([seed, 3]))
    q = rng.uniform(-1.0, 1.0, size=8).astype(np.float32)
    cs = []
    while len(cs) < 8:
        c = rng.uniform(-0.3, 0.3, size=3)
        if float(np.dot(c, c)) < 0.09:
            cs.append(c)
    return q, np.asarray(cs, dtype=np.float32)


def sampled_levelset(cfg: dict, nc: int) -> np.ndarray:
    """Nodal values of the configuration's sphere-union level set on the (nc+1)^3 grid over
    [-1,1]^3, x fastest, fp32 (S:82 Sampled variant, S:145 file order).  This is input data:
    the paper's level set lives on "a separate coarse mesh" that the method only
    interpolates; here the mesh is filled from the analytic geometry of the configuration."""
    if cfg["ls_kind"] == LS_SPHERES:
        g = np.linspace(-1.0, 1.0, nc + 1)
        z, y, x = np.meshgrid(g, g, g, indexing="ij")           # x fastest in C order
        X = np.stack([x, y, z], axis=-1).astype(np.float64)
        c = np.asarray(cfg["centers"], np.float64)
        r = np.asarray(cfg["radii"], np.float64)
        d = np.sqrt(((X[..., None, :] - c) ** 2).sum(-1)) - r
        return d.min(-1).astype(np.float32).reshape(-1)
    if cfg["ls_kind"] == LS_PLANE:
        g = np.linspace(-1.0, 1.0, nc + 1)
        z, y, x = np.meshgrid(g, g, g, indexing="ij")
        (a, b, cc), c0 = cfg["plane"]
        return (a * x + b * y + cc * z - c0).astype(np.float32).reshape(-1)
    raise ValueError("sampled level sets are built from sphere-union or plane geometries")


def with_grid(cfg: dict, nc: int) -> dict:
    """The configuration with its level set replaced by the sampled one on an nc^3 grid."""
    out = dict(cfg)
    out["grid"] = sampled_levelset(cfg, nc)
    out["ls_kind"] = LS_GRID
    out["name"] = cfg["name"]
    out["grid_n"] = nc
    return out


def config(name: str, width: int | None = None, prec: int | None = None) -> dict:
    """Plain parameter dict of a BASELINE.json configuration ('c1'..'c5')."""
    base = dict(box=(-1.0, 1.0), k=(0.0, 0.0), lambda_b=1.0, ls_kind=LS_NONE,
                centers=np.zeros((0, 3), np.float32), radii=np.zeros(0, np.float32),
                star=(0.5, 0.15, 5, 3), plane=((1.0, 0.0, 0.0), 0.0),
                charges_q=np.zeros(0, np.float32), charges_c=np.zeros((0, 3), np.float32),
                charge_sigma=0.02, seed=0, grid=None)
    if name == "c1":
        base.update(ls_kind=LS_NONE, beta=(1.0, 1.0), source=SRC_SINE3PI,
                    sizes=[3, 32, 32, 1], act=ACT_TANH, prec=PREC_FP32, n_nets=1,
                    N=4096, Nb=512, H=h_lattice(1 / 32), adam_steps=10, lr=1e-3)
    elif name == "c2":
        base.update(ls_kind=LS_SPHERES, centers=np.zeros((1, 3), np.float32),
                    radii=np.array([0.5], np.float32), beta=(1.0, 10.0), source=SRC_PAIR,
                    sizes=[3, 64, 64, 64, 1], act=ACT_TANH, prec=PREC_FP32, n_nets=2,
                    N=1 << 18, Nb=1 << 15, H=h_lattice(1 / 128), lr=1e-3)
    elif name == "c3":
        q, c = _config3_charges()
        base.update(ls_kind=LS_STAR, beta=(2.0, 80.0), source=SRC_GAUSS,
                    charges_q=q, charges_c=c, sizes=[3, 128, 128, 128, 128, 1],
                    act=ACT_SILU, prec=PREC_BF16, n_nets=2,
                    N=1 << 20, Nb=1 << 17, H=h_lattice(1 / 512), lr=1e-3)
    elif name in ("c4", "c5"):
        c, r = _config4_spheres()
        w = 256 if width is None else width
        base.update(ls_kind=LS_SPHERES, centers=c, radii=r, beta=(1.0, 100.0),
                    source=SRC_PAIR, sizes=[3, w, w, w, w, 1], act=ACT_TANH,
                    prec=PREC_BF16 if prec is None else prec, n_nets=2,
                    N=1 << 22, Nb=1 << 19, H=h_lattice(2 / 1023), lr=1e-3)
    elif name == "p41":
        # the paper's 4.1 benchmark: sphere r = 0.5, u- = e^z, u+ = cos(x) sin(y),
        # mu- = y^2 ln(x+2) + 4, mu+ = e^{-z}; two 5 x 10 sine nets (982 parameters); the
        # Table 1 resolution N = 2^7 (h = 2/128) with mesh-free points
        base.update(ls_kind=LS_SPHERES, centers=np.zeros((1, 3), np.float32),
                    radii=np.array([0.5], np.float32), beta=(1.0, 1.0), source=SRC_PAPER41,
                    mu_kind=MU_PAPER41, sizes=[3, 10, 10, 10, 10, 10, 1], act=ACT_SINE,
                    prec=PREC_FP32, n_nets=2, N=1 << 18, Nb=1 << 15, H=h_lattice(2 / 128), lr=1e-3)
    else:
        raise ValueError(name)
    if prec is not None:
        base["prec"] = prec
    base["name"] = name
    base["h"] = base["H"] / LATTICE
    return base


def param_count(sizes, n_nets: int) -> int:
    p = sum(sizes[l] * sizes[l - 1] + sizes[l] for l in range(1, len(sizes)))
    return p * n_nets


def random_theta(sizes, n_nets: int, seed: int, bias_scale: float = 0.1) -> np.ndarray:
    """Seeded fp32 parameter vector (Glorot-scale weights, small random biases),
    laid out net-, net+, layer by layer [W_l row-major, b_l] (G17)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 17]))
    out = []
    for _ in range(n_nets):
        for l in range(1, len(sizes)):
            fi, fo = sizes[l - 1], sizes[l]
            a = np.sqrt(6.0 / (fi + fo))
            out.append(rng.uniform(-a, a, size=fi * fo))
            out.append(rng.uniform(-bias_scale, bias_scale, size=fo))
    return np.concatenate(out).astype(np.float32)


def random_lattice_points(n: int, H: int, seed: int) -> np.ndarray:
    """n seeded interior points on the 2^-24 lattice in [-1+h, 1-h]^3 (numpy draw)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 23]))
    m = LATTICE - H
    ints = rng.integers(-m, m, size=(n, 3), endpoint=True)
    return (ints.astype(np.float64) / LATTICE).astype(np.float32)
