"""Pins of the error norms and convergence orders of the evaluation stage (SURVEY
8f NEXT-2; Table 1): the paper's printed orders, closed forms of the section 4.1
exact solution, brute force on a tiny grid."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2210_14907_b200 import inputs

T1 = json.load(open(os.path.join(GOLDEN, "table1.json")))


def test_orders_reproduce_table1(orc):
    """Every Order entry of Table 1 is log2 of the ratio of consecutive Solution entries."""
    for col in ("rmse", "linf"):
        e, o = T1[col], T1[col + "_order"]
        for i in range(1, len(e)):
            assert orc.convergence_order(e[i - 1], e[i]) == pytest.approx(o[i], abs=0.011), (col, i)


def test_order_properties(orc):
    assert orc.convergence_order(0.3, 0.3) == 0.0
    assert orc.convergence_order(0.2, 0.05) == pytest.approx(2.0)
    assert orc.convergence_order(0.05, 0.2) == -orc.convergence_order(0.2, 0.05)
    with pytest.raises(ValueError):
        orc.convergence_order(0.0, 1.0)


def _p41():
    return inputs.config("p41")


def test_zero_network_gives_the_exact_solution_norms(orc):
    """theta = 0 except the output bias c: u = c everywhere, so e = c - u*; u* from P:72
    (u- = e^z inside the sphere r = 0.5, u+ = cos x sin y outside; phi <= 0 is Omega-)."""
    cfg = _p41()
    pb, ar = orc.from_config(cfg)
    M = 12
    g = (-1.0 + 2.0 * np.arange(M + 1) / M).astype(np.float32).astype(np.float64)
    z, y, x = np.meshgrid(g, g, g, indexing="ij")               # x fastest
    inside = np.sqrt(x * x + y * y + z * z) - 0.5 <= 0.0
    ustar = np.where(inside, np.exp(z), np.cos(x) * np.sin(y))
    for c in (0.0, 0.75):
        th = np.zeros(ar.P)
        P1 = ar.P // 2
        th[P1 - 1] = c
        th[ar.P - 1] = c
        rmse, linf = orc.error_norms(pb, ar, th, M)
        e = c - ustar
        assert rmse == pytest.approx(np.sqrt(np.mean(e * e)), rel=1e-12)
        assert linf == pytest.approx(np.abs(e).max(), rel=1e-12)


def test_brute_force_tiny_grid(orc):
    cfg = _p41()
    pb, ar = orc.from_config(cfg)
    th = orc.init_params(ar, 3).astype(np.float64)
    M = 2
    errs = []
    for k in range(3):
        for j in range(3):
            for i in range(3):
                p = np.array([-1.0 + i, -1.0 + j, -1.0 + k])
                s = orc.side(pb, p)
                u, _ = orc.exact(pb, s, p)
                errs.append(orc.forward(ar, th, s, p) - u)
    errs = np.array(errs)
    rmse, linf = orc.error_norms(pb, ar, th, M)
    assert rmse == pytest.approx(np.sqrt(np.mean(errs ** 2)), rel=1e-14)
    assert linf == pytest.approx(np.abs(errs).max(), rel=1e-14)
    assert rmse <= linf


def test_no_exact_solution_rejected(orc):
    cfg = inputs.config("c3")
    pb, ar = orc.from_config(cfg)
    with pytest.raises(ValueError):
        orc.error_norms(pb, ar, np.zeros(ar.P), 4)
