"""Pins of the oracle's level sets, sides, crossings and normals,
and of the manufactured data families (P:40-41 jump problem, configs 1-4)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2210_14907_b200 import inputs

SPEC = json.load(open(os.path.join(GOLDEN, "spec_vectors.json")))


def _sphere_cfg(beta=(1.0, 10.0)):
    cfg = inputs.config("c2")
    cfg["beta"] = beta
    return cfg


def test_spec_sphere_vectors(orc):
    pb, _ = orc.from_config(_sphere_cfg())
    g = SPEC["geometry"]
    for v in g["phi"]:
        assert orc.phi(pb, v["x"]) == v["phi"]
    for v in g["side"]:
        assert orc.side(pb, v["x"]) == v["side"]
    for v in g["normal"]:
        assert np.allclose(orc.normal(pb, v["x"]), v["n"], atol=v["tol"])
    for v in g["crossing"]:
        c = orc.crossing(pb, v["a"], v["b"])
        if v["theta"] is None:
            assert c is None
        else:
            th, xg, n = c
            assert abs(th - v["theta"]) < 1e-12
            assert np.allclose(xg, v["location"], atol=1e-12)
            assert np.allclose(n, v["normal"], atol=1e-12)


def test_spec_plane_crossing_exact(orc):
    v = SPEC["geometry"]["plane_crossing"]
    cfg = inputs.config("c1")
    cfg.update(ls_kind=inputs.LS_PLANE, plane=(v["plane_n"], v["plane_c"]))
    pb, _ = orc.from_config(cfg)
    th, xg, n = orc.crossing(pb, v["a"], v["b"])
    assert th == float(np.float32(v["theta"]))
    assert np.array_equal(n, [1.0, 0.0, 0.0])


def test_constant_level_set_is_degenerate(orc):
    cfg = inputs.config("c1")
    cfg.update(ls_kind=inputs.LS_PLANE, plane=((0.0, 0.0, 0.0), 0.3))   # phi == -0.3
    pb, _ = orc.from_config(cfg)
    with pytest.raises(RuntimeError):
        orc.normal(pb, [0.1, 0.2, 0.3])


def _geoms():
    c4 = inputs.config("c4")
    c3 = inputs.config("c3")
    # two heavily overlapping spheres: exercises the union rule of G8
    ov = inputs.config("c2")
    ov.update(centers=np.array([[0.0, 0, 0], [0.3, 0.05, 0]], np.float32),
              radii=np.array([0.4, 0.35], np.float32))
    return {"sphere": _sphere_cfg(), "union32": c4, "star": c3, "overlap": ov}


@pytest.mark.parametrize("name", ["sphere", "union32", "star", "overlap"])
def test_crossing_symmetry_and_bisection(orc, name):
    """theta(a->b) + theta(b->a) = 1; closed form agrees with an
    independent bisection of the side function (G8)."""
    cfg = _geoms()[name]
    pb, _ = orc.from_config(cfg)
    rng = np.random.default_rng(11)
    found = 0
    tries = 0
    while found < 60 and tries < 200000:
        tries += 1
        a = rng.uniform(-0.9, 0.9, 3)
        b = a.copy()
        b[rng.integers(3)] += rng.choice([-1, 1]) * 0.05
        c1 = orc.crossing(pb, a, b)
        if c1 is None:
            continue
        found += 1
        c2 = orc.crossing(pb, b, a)
        assert abs(c1[0] + c2[0] - 1.0) < 1e-10
        tb = orc.crossing_bisect(pb, a, b)
        assert abs(c1[0] - tb) < 1e-10
        assert abs(np.linalg.norm(c1[2]) - 1.0) < 1e-12
        # the normal points from Omega- to Omega+ 
        x = c1[1]
        assert orc.side(pb, x + 1e-7 * c1[2]) == 1 and orc.side(pb, x - 1e-7 * c1[2]) == 0
    assert found == 60


def test_sphere_crossing_location_on_sphere(orc):
    pb, _ = orc.from_config(_sphere_cfg())
    rng = np.random.default_rng(3)
    n = 0
    while n < 100:
        a = rng.uniform(-0.7, 0.7, 3)
        b = a.copy()
        b[rng.integers(3)] += 0.1
        c = orc.crossing(pb, a, b)
        if c:
            n += 1
            assert abs(np.linalg.norm(c[1]) - 0.5) < 1e-12


def test_star_polynomial_matches_trigonometric_form(orc):
    """G13: the recurrence form equals r - r0 - amp sin(5 t) cos(3 p)."""
    cfg = inputs.config("c3")
    pb, _ = orc.from_config(cfg)
    r0, amp, m, n = [float(np.float32(v)) for v in cfg["star"]]
    rng = np.random.default_rng(0)
    for x in rng.uniform(-1, 1, size=(1000, 3)):
        r = np.linalg.norm(x)
        th = np.arccos(x[2] / r)
        ph = np.arctan2(x[1], x[0])
        want = r - r0 - amp * np.sin(m * th) * np.cos(n * ph)
        assert abs(orc.phi(pb, x) - want) < 1e-13
    assert orc.phi(pb, [0, 0, 0]) == -r0
    assert abs(orc.phi(pb, [0, 0, 0.7]) - (0.7 - r0)) < 1e-15


def test_union_is_min_of_sphere_distances(orc):
    cfg = inputs.config("c4")
    pb, _ = orc.from_config(cfg)
    c = cfg["centers"].astype(np.float64)
    r = cfg["radii"].astype(np.float64)
    rng = np.random.default_rng(1)
    for x in rng.uniform(-1, 1, size=(500, 3)):
        want = np.min(np.linalg.norm(x - c, axis=1) - r)
        assert abs(orc.phi(pb, x) - want) < 1e-15


# ---------------- manufactured data ----------------

def _fd_laplacian(fn, x, e=1e-3):
    x = np.asarray(x, float)
    lap = 0.0
    for d in range(3):
        v = []
        for k in (-2, -1, 0, 1, 2):
            y = x.copy()
            y[d] += k * e
            v.append(fn(y))
        lap += (-v[0] + 16 * v[1] - 30 * v[2] + 16 * v[3] - v[4]) / (12 * e * e)
    return lap


def _fd_grad(fn, x, e=1e-5):
    x = np.asarray(x, float)
    g = np.zeros(3)
    for d in range(3):
        yp, ym = x.copy(), x.copy()
        yp[d] += e
        ym[d] -= e
        g[d] = (fn(yp) - fn(ym)) / (2 * e)
    return g


@pytest.mark.parametrize("name,k", [("c1", 0.0), ("c2", 0.0), ("c2", 2.5), ("c1", 1.5)])
def test_source_is_k_u_minus_div_beta_grad_u(orc, name, k):
    """f_s = k_s u_s - beta_s Lap u_s, checked by 4th-order finite differences
    of the exact solution; the exact gradient is checked by central differences."""
    cfg = inputs.config(name)
    cfg["k"] = (k, 2 * k)
    pb, _ = orc.from_config(cfg)
    rng = np.random.default_rng(2)
    for x in rng.uniform(-0.9, 0.9, size=(40, 3)):
        for s in (0, 1):
            u = lambda y: orc.exact(pb, s, y)[0]
            lap = _fd_laplacian(u, x)
            kk = float(np.float32(cfg["k"][s]))
            bb = float(np.float32(cfg["beta"][s]))
            want = kk * u(x) - bb * lap
            assert abs(orc.f(pb, s, x) - want) < 1e-6 * max(1.0, abs(want))
            assert np.allclose(orc.exact(pb, s, x)[1], _fd_grad(u, x), atol=1e-8)


def test_jump_data_of_config2_pair(orc):
    """alpha = [u] = u+ - u-, sigma = beta+ d_n u+ - beta- d_n u- on the sphere (G12)."""
    pb, _ = orc.from_config(_sphere_cfg())
    rng = np.random.default_rng(4)
    for _ in range(50):
        v = rng.normal(size=3)
        x = 0.5 * v / np.linalg.norm(v)
        n = orc.normal(pb, x)
        up = np.sin(x.sum())
        um = np.exp(x[0]) * np.cos(x[1]) * x[2]
        assert abs(orc.alpha(pb, x) - (up - um)) < 1e-14
        dn_p = _fd_grad(lambda y: orc.exact(pb, 1, y)[0], x) @ n
        dn_m = _fd_grad(lambda y: orc.exact(pb, 0, y)[0], x) @ n
        assert abs(orc.sigma(pb, x, n) - (10.0 * dn_p - 1.0 * dn_m)) < 1e-8


def test_gaussian_charge_is_normalised(orc):
    """G13: the smoothed charge integrates to q (midpoint rule, spectrally accurate)."""
    cfg = inputs.config("c3")
    cfg.update(charges_q=np.array([1.0], np.float32), charges_c=np.zeros((1, 3), np.float32))
    pb, _ = orc.from_config(cfg)
    s = float(np.float32(0.02))
    hq = 0.25 * s
    ax = np.arange(-28, 29) * hq
    tot = 0.0
    for x in ax:
        for y in ax:
            for z in ax:
                tot += orc.f(pb, 0, [x, y, z])
    assert abs(tot * hq**3 - 1.0) < 1e-6


def test_boundary_data_is_side_exact_solution(orc):
    pb, _ = orc.from_config(_sphere_cfg())
    x = [1.0, 0.2, -0.3]
    assert orc.g(pb, x) == pytest.approx(np.sin(0.9), abs=1e-15)
    cfg3 = inputs.config("c3")
    pb3, _ = orc.from_config(cfg3)
    assert orc.g(pb3, x) == 0.0                                           # G13: u = 0 on faces


# ---- sampled level set ("a separate coarse mesh") ----

def _grid_cfg(nc, base=None):
    return inputs.with_grid(_sphere_cfg() if base is None else base, nc)


def test_grid_reproduces_nodes_and_linear_fields(orc):
    """Trilinear interpolation equals the nodal values at the nodes and reproduces a linear
    level set exactly (its fp32 nodes are exact here); the S:133 example "linear phi,
    a=(0,0,0), b=(1,0,0) -> theta = x0" holds for the linear-interpolant crossing."""
    cfg = _sphere_cfg()
    cfg.update(ls_kind=inputs.LS_PLANE, plane=((1.0, 0.0, 0.0), 0.125))
    g = _grid_cfg(32, cfg)
    pb, _ = orc.from_config(g)
    nodes = np.asarray(g["grid"]).reshape(33, 33, 33)
    for i, j, k in [(0, 0, 0), (32, 32, 32), (5, 17, 29), (31, 0, 12)]:
        x = [-1 + i / 16, -1 + j / 16, -1 + k / 16]
        assert orc.phi(pb, x) == float(nodes[k, j, i])
    pts = inputs.random_lattice_points(500, inputs.h_lattice(1 / 64), 3).astype(np.float64)
    for x in pts:
        assert abs(orc.phi(pb, x) - (x[0] - 0.125)) <= 1e-15
    th, xg, n = orc.crossing(pb, [0, 0, 0], [1, 0, 0])
    assert th == 0.125 and np.allclose(n, [1, 0, 0], atol=1e-12)


def test_grid_sphere_interpolation_error_is_second_order(orc):
    """S:82 example: the sampled sphere's |phi_sampled - phi| <= C hc^2 at random points
    (C measured; away from the centre where the Hessian of |x| blows up), and the error falls
    by ~4x per halving of hc (trilinear interpolation is second order)."""
    pb0, _ = orc.from_config(_sphere_cfg())
    rng = np.random.default_rng(7)
    x = rng.uniform(-0.95, 0.95, size=(1000, 3))
    x = x[np.linalg.norm(x, axis=1) > 0.25]
    errs = []
    for nc in (16, 32, 64):
        pb, _ = orc.from_config(_grid_cfg(nc))
        e = max(abs(orc.phi(pb, p) - orc.phi(pb0, p)) for p in x)
        hc = 2.0 / nc
        assert e <= 1.0 * hc * hc
        errs.append(e)
    assert 3.0 < errs[0] / errs[1] < 5.5 and 3.0 < errs[1] / errs[2] < 5.5


def test_grid_crossings_and_normals(orc):
    """theta(a->b) + theta(b->a) = 1, crossing locations within C hc^2 of |x| = 0.5
    (Sampled), normals of the sampled sphere ~ radial (step hc/2)."""
    nc = 64
    pb, _ = orc.from_config(_grid_cfg(nc))
    rng = np.random.default_rng(11)
    n_cross = 0
    for _ in range(3000):
        a = rng.uniform(-0.8, 0.8, 3)
        b = a + rng.normal(size=3) * 0.05
        c1 = orc.crossing(pb, a, b)
        if c1 is None:
            continue
        c2 = orc.crossing(pb, b, a)
        assert abs(c1[0] + c2[0] - 1.0) <= 1e-12
        # the linear-interpolant root is off the curved interface by <= |b-a|^2 max|phi''|/8
        # along the arm (phi'' <= 1/r = 2), plus the trilinear error
        assert abs(np.linalg.norm(c1[1]) - 0.5) <= 2.0 * (2.0 / nc) ** 2 + np.dot(b - a, b - a) / 4
        assert np.dot(c1[2], c1[1] / np.linalg.norm(c1[1])) > 0.99
        n_cross += 1
    assert n_cross > 20
    assert np.allclose(orc.normal(pb, [0.5, 0, 0]), [1, 0, 0], atol=1e-3)
    assert np.allclose(orc.normal(pb, [0, -0.5, 0]), [0, -1, 0], atol=1e-3)


def test_grid_jump_suite_exact(orc):
    """The S:294 jump suite on a sampled plane: with dyadic theta and h the plane's fp32 nodes
    are exact, the interpolant is the plane itself, and every crossed row reproduces the exact
    piecewise-linear solution (r ~ round-off), so assembly on the Sampled variant is pinned."""
    import test_oracle_assembly as A
    h = 1.0 / 16
    ex = A.SPEC["jump_suite"]
    worst, n = 0.0, 0
    for th in (0.25, 0.5, 0.75):
        for bm, bp, a, b in [(1.0, 3.0, 2.0, -1.0), (0.5, 1.0, -1.0, 2.0), (3.0, 0.5, 0.0, 2.0), (1.0, 1.0, 2.0, 0.0)]:
            for axis, orient, cs in [(0, 1, 0), (1, -1, 1), (2, 1, 1), (0, -1, 0)]:
                pb, poly, p = A._plane_case(orc, axis, orient, th, bm, bp, a, b, cs, h=h)
                nvec = [0.0, 0.0, 0.0]
                nvec[axis] = float(orient)
                x0 = float(np.float32(p[axis] + (orient if cs == 0 else -orient) * th * np.float32(h)))
                base = A._poly_cfg(beta=(bm, bp))
                base.update(ls_kind=inputs.LS_PLANE, plane=(nvec, float(orient) * x0))
                g = inputs.with_grid(base, 32)
                pbg, _ = orc.from_config(g, poly=poly)
                row = orc.assemble(pbg, p, h)
                assert row.side == cs and row.crossed and row.n_crossed_arms == 1
                raw, scale = A._raw(row, A._poly_u(poly))
                worst = max(worst, abs(raw / row.d))
                n += 1
    assert n == 48 and worst < ex["tol"]
