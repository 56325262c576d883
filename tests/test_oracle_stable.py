"""Pins of the stable difference-propagation evaluation (oracle/stable_stencil.py, DESIGN.md
G27) against the plain definition of the uncrossed residual and its
gradient (oracle.c, fp64), extended-precision closed forms and the Taylor series of tanh."""
import numpy as np
import pytest

from oracle import stable_stencil as st
from paper_2210_14907_b200 import inputs

LD = np.longdouble


def _cfg(sizes, k=1.5):
    cfg = inputs.config("c1")
    cfg.update(sizes=sizes, n_nets=1, k=(k, k), beta=(1.0, 1.0))
    return cfg


def test_tanh_minus_id_series():
    """tanh(d) - d against 80-bit tanh, both branches and the cut."""
    d = np.concatenate([np.geomspace(1e-4, 0.2499, 40), np.geomspace(0.2501, 3.0, 20)])
    d = np.concatenate([d, -d])
    ref = np.tanh(d.astype(LD)) - d.astype(LD)
    got = st.tanh_minus_id(d)
    rel = np.abs((got - ref) / ref).astype(np.float64)
    assert rel[np.abs(d) < st.CUT].max() < 2e-5          # series truncation (d^9 term)
    assert rel.max() < 1e-10 / 1e-4 ** 2                  # direct branch: fp64 cancellation only


def test_g_is_tanh_addition_remainder():
    rng = np.random.default_rng(3)
    z = rng.uniform(-3, 3, 500)
    d = rng.uniform(-0.5, 0.5, 500) * 10.0 ** rng.uniform(-3, 0, 500)
    t = np.tanh(z)
    zl, dl = z.astype(LD), d.astype(LD)
    ref = np.tanh(zl + dl) - np.tanh(zl) - (1 - np.tanh(zl) ** 2) * dl
    got = st.g_fun(t, d)
    # g = O(d^2); extended-precision reference loses ~1e-19 / d^2 relative
    assert np.all(np.abs(got - ref.astype(np.float64)) <= 2e-5 * np.abs(ref.astype(np.float64)) + 1e-17)


def test_single_unit_closed_form_small_h():
    """[3, 1, 1] net: DU_d = v (tanh(z + w_d h) + tanh(z - w_d h) - 2 tanh z), 80-bit."""
    w, b0, v, c = np.array([0.3, -0.7, 1.1]), 0.2, -1.4, 0.05
    th = np.concatenate([w, [b0], [v], [c]])
    x = np.random.default_rng(4).uniform(-1, 1, (20, 3))
    h = 2.0 / 1023.0
    u, dU, DU, _ = st.forward(th, [3, 1, 1], x, h)
    z = (x.astype(LD) @ w.astype(LD)) + LD(b0)
    for dd in range(3):
        wh = LD(w[dd]) * LD(h)
        ref2 = LD(v) * (np.tanh(z + wh) + np.tanh(z - wh) - 2 * np.tanh(z))
        ref1 = LD(v) * (np.tanh(z + wh) - np.tanh(z))
        assert np.allclose(DU[:, dd], ref2.astype(np.float64), rtol=1e-9, atol=0)
        assert np.allclose(dU[:, dd], ref1.astype(np.float64), rtol=1e-12, atol=0)
    assert np.allclose(u, v * np.tanh(x @ w + b0) + c, rtol=1e-15)


def test_forward_matches_plain_differences(orc):
    """u, first and second differences of a [3,16,16,16,1] net equal the plain fp64 values
    from oracle.c's forward at the 7 stencil vertices (h = 1/32: plain cancellation small, series
    truncation below 1e-12)."""
    cfg = _cfg([3, 16, 16, 16, 1])
    _, ar = orc.from_config(cfg)
    th = inputs.random_theta(cfg["sizes"], 1, seed=5).astype(np.float64)
    x = np.random.default_rng(6).uniform(-0.8, 0.8, (30, 3))
    h = 1.0 / 32.0
    u, dU, DU, _ = st.forward(th, cfg["sizes"], x, h)
    for i, p in enumerate(x):
        uc = orc.forward(ar, th, 0, p)
        assert u[i] == pytest.approx(uc, abs=1e-13)
        for dd in range(3):
            e = np.eye(3)[dd] * h
            up, um = orc.forward(ar, th, 0, p + e), orc.forward(ar, th, 0, p - e)
            assert dU[i, dd] == pytest.approx(up - uc, abs=1e-13)
            assert DU[i, dd] == pytest.approx(up + um - 2 * uc, abs=1e-12)


@pytest.mark.parametrize("h", [1 / 16, 1 / 64])
def test_loss_grad_equals_plain_definition(orc, h):
    """The stable form's r, L and dL/dtheta equal oracle.c's uncrossed term --
    pins the hand-derived backward maps dP/dz ... dQ/dD used by the CUDA kernel."""
    cfg = _cfg([3, 16, 16, 16, 1])
    pb, ar = orc.from_config(cfg)
    th = inputs.random_theta(cfg["sizes"], 1, seed=7).astype(np.float32)
    # points on the 2^-24 lattice (G9) so that the arms x +- h e_d are exact in fp32 on both sides
    pts = np.random.default_rng(8).uniform(-0.9, 0.9, (64, 3))
    pts = (np.round(pts * 2.0 ** 24) / 2.0 ** 24).astype(np.float32)
    none = np.zeros((0, 3), np.float32)
    hf = float(np.float32(h))
    r_plain, _ = orc.residuals(pb, ar, th, pts, none, hf)
    L0, lt, g0, gt = orc.loss_grad(pb, ar, th, pts, none, hf, per_term=True)
    k, beta = float(np.float32(cfg["k"][0])), float(np.float32(cfg["beta"][0]))
    cc, ch = st.residual_coefficients(k, beta, hf)
    # rhs b/d recovered from the plain definition: r = u_c + c_hat sum_j u_j - b/d
    lin = np.zeros(len(pts))
    for i, p in enumerate(pts.astype(np.float64)):
        vals = [orc.forward(ar, th, 0, p)]
        for dd in range(3):
            for sgn in (1, -1):
                vals.append(orc.forward(ar, th, 0, p + sgn * hf * np.eye(3)[dd]))
        lin[i] = vals[0] + ch * sum(vals[1:])
    rhs = lin - r_plain
    L, r, g = st.loss_grad_unx(th.astype(np.float64), cfg["sizes"], pts, hf, k, beta, rhs)
    assert np.allclose(r, r_plain, rtol=0, atol=1e-9 * np.abs(r_plain).max())
    assert L == pytest.approx(lt[orc.T_UNX_MINUS], rel=1e-9)
    ref = gt[orc.T_UNX_MINUS]
    assert np.abs(g - ref).max() <= 1e-8 * np.abs(ref).max()


def test_bf16_noise_floor_resolved():
    """The point of the reading: with bf16 GEMM operands at h = 2/1023 (configs 4/5) the
    stable form's second differences keep ~1e-2 relative accuracy, the plain 7-value
    differences do not (G27)."""
    sizes = [3, 64, 64, 64, 1]
    th = inputs.random_theta(sizes, 1, seed=9).astype(np.float64)
    x = np.random.default_rng(10).uniform(-0.9, 0.9, (200, 3))
    h = 2.0 / 1023.0
    _, _, DU, _ = st.forward(th, sizes, x, h)
    _, _, DUb, _ = st.forward(th, sizes, x, h, rnd=st.bf16)
    err_stable = np.linalg.norm(DUb - DU) / np.linalg.norm(DU)
    # plain: round each of the 7 network values' hidden operands to bf16 (same rounding model)
    ub, _, _, _ = st.forward(th, sizes, x, 0.0, rnd=st.bf16)
    plain = np.zeros_like(DU)
    for dd in range(3):
        e = np.eye(3)[dd] * h
        up, _, _, _ = st.forward(th, sizes, x + e, 0.0, rnd=st.bf16)
        um, _, _, _ = st.forward(th, sizes, x - e, 0.0, rnd=st.bf16)
        plain[:, dd] = up + um - 2 * ub
    err_plain = np.linalg.norm(plain - DU) / np.linalg.norm(DU)
    assert err_stable < 2e-2
    assert err_plain > 1.0
