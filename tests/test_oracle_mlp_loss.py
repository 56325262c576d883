"""Pins of the oracle's surrogate, loss, gradient and Adam (S:156-226, S:264-290,
S:345-362).  North-star self-checks 4 (finite differences on a tiny
network) and 5 (linear-in-theta model vs a brute-force dense least squares)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2210_14907_b200 import inputs

SPEC = json.load(open(os.path.join(GOLDEN, "spec_vectors.json")))


def _cfg(sizes, act=0, n_nets=2, geom="sphere", beta=(1.0, 10.0)):
    cfg = inputs.config("c2")
    cfg.update(sizes=sizes, act=act, n_nets=n_nets, beta=beta)
    if geom == "none":
        cfg.update(ls_kind=inputs.LS_NONE, source=inputs.SRC_SINE3PI)
    return cfg


def test_param_counts(orc):
    for v in SPEC["surrogate"]["param_count"]:
        _, ar = orc.from_config(_cfg(v["sizes"], n_nets=v["n_nets"]))
        assert ar.P == v["P"], v["cite"]
        assert inputs.param_count(v["sizes"], v["n_nets"]) == v["P"]


def test_zero_weights_give_output_bias(orc):
    _, ar = orc.from_config(_cfg([3, 5, 5, 1], n_nets=1))
    th = np.zeros(ar.P)
    th[-1] = 0.37
    for x in np.random.default_rng(0).uniform(-1, 1, (10, 3)):
        assert orc.forward(ar, th, 0, x) == 0.37


@pytest.mark.parametrize("act,fn", [(0, np.tanh), (1, lambda z: z / (1 + np.exp(-z))), (2, np.sin)])
def test_single_unit_closed_form(orc, act, fn):
    """[3,1,1] net -> v act(w.p + b0) + c."""
    _, ar = orc.from_config(_cfg([3, 1, 1], act=act, n_nets=1))
    w, b0, v, c = np.array([0.3, -0.7, 1.1]), 0.2, -1.4, 0.05
    th = np.concatenate([w, [b0], [v], [c]])
    for x in np.random.default_rng(1).uniform(-1, 1, (10, 3)):
        assert orc.forward(ar, th, 0, x) == pytest.approx(v * fn(w @ x + b0) + c, abs=1e-15)


def test_backward_special_cases(orc):
    _, ar = orc.from_config(_cfg([3, 4, 1], n_nets=1))
    th = np.random.default_rng(2).normal(size=ar.P)
    x = np.array([0.1, 0.2, -0.3])
    assert np.all(orc.backward(ar, th, 0, x, 0.0) == 0.0)
    _, lin = orc.from_config(_cfg([3, 1], n_nets=1))
    g = orc.backward(lin, np.ones(4), 0, x, 1.0)
    assert np.array_equal(g, np.concatenate([x, [1.0]]))


@pytest.mark.parametrize("act", [0, 1, 2])
def test_backward_matches_central_differences(orc, act):
    """random net, random p, every component vs central FD (step 1e-6)."""
    _, ar = orc.from_config(_cfg([3, 6, 5, 4, 1], act=act, n_nets=2))
    rng = np.random.default_rng(3 + act)
    th = rng.normal(size=ar.P) * 0.7
    for net in (0, 1):
        x = rng.uniform(-1, 1, 3)
        cot = rng.normal()
        g = orc.backward(ar, th, net, x, cot)
        fd = np.zeros(ar.P)
        for i in range(ar.P):
            tp, tm = th.copy(), th.copy()
            tp[i] += 1e-6
            tm[i] -= 1e-6
            fd[i] = cot * (orc.forward(ar, tp, net, x) - orc.forward(ar, tm, net, x)) / 2e-6
        scale = np.abs(g).max()
        assert np.all(np.abs(g - fd) <= 1e-5 * np.maximum(np.abs(g), 1e-2 * scale))


def _mixed_batch(orc, cfg, n=10, nb=4, h=1 / 16, seed=0):
    """interior points near the sphere so the batch mixes crossed and uncrossed rows."""
    pb, ar = orc.from_config(cfg)
    H = inputs.h_lattice(h)
    cand = inputs.random_lattice_points(4000, H, seed)
    _, cls = orc.classify(pb, cand, H / 2**24)
    crossed = cand[cls == 2][: n // 2]
    rest = cand[cls < 2][: n - len(crossed)]
    pts = np.concatenate([crossed, rest])
    b = orc.sample(1, seed, 0, 0, nb, H)
    return pb, ar, pts, b, H / 2**24


@pytest.mark.parametrize("act", [0, 1])
def test_loss_gradient_matches_central_differences(orc, act):
    """North-star self-check 4 / S:281 / S:353 / S:513: full loss gradient vs central
    FD over all parameters of a tiny [3,4,4,1] pair on a mixed 10-point batch."""
    cfg = _cfg([3, 4, 4, 1], act=act)
    pb, ar, pts, b, h = _mixed_batch(orc, cfg)
    _, cls = orc.classify(pb, pts, h)
    assert (cls == 2).sum() >= 3 and (cls < 2).sum() >= 3
    th = np.random.default_rng(4).normal(size=ar.P) * 0.8
    L, lt, g, _ = orc.loss_grad(pb, ar, th, pts, b, h)
    assert L == pytest.approx(lt.sum()) and lt[2] > 0 and lt[3] > 0
    fd = np.zeros(ar.P)
    for i in range(ar.P):
        tp, tm = th.copy(), th.copy()
        tp[i] += 1e-6
        tm[i] -= 1e-6
        fd[i] = (orc.loss_grad(pb, ar, tp, pts, b, h)[0] - orc.loss_grad(pb, ar, tm, pts, b, h)[0]) / 2e-6
    scale = np.abs(g).max()
    assert np.all(np.abs(g - fd) <= 1e-5 * np.maximum(np.abs(g), 1e-3 * scale))


def test_residual_definition_and_cotangent_examples(orc):
    """r = 0 -> zero gradient; loss is (1/N) sum r^2 + (1/Nb) sum rb^2 (G1)."""
    cfg = _cfg([3, 5, 5, 1])
    pb, ar, pts, b, h = _mixed_batch(orc, cfg, n=12, nb=6)
    th = orc.init_params(ar, 0)
    r, rb = orc.residuals(pb, ar, th, pts, b, h)
    L, lt, _, _ = orc.loss_grad(pb, ar, th, pts, b, h)
    assert L == pytest.approx((r**2).mean() + (rb**2).mean(), rel=1e-13)
    assert lt[3] == pytest.approx((rb**2).mean(), rel=1e-13)
    # empty interior and lambda_b = 0 -> loss 0, grad 0
    cfg0 = dict(cfg, lambda_b=0.0)
    pb0, _ = orc.from_config(cfg0)
    L0, _, g0, _ = orc.loss_grad(pb0, ar, th, np.zeros((0, 3)), b, h)
    assert L0 == 0.0 and np.all(g0 == 0.0)


def test_boundary_residual_is_linear_in_output_bias(orc):
    """r_b has slope 1 in the output bias of the selected network."""
    cfg = _cfg([3, 5, 1])
    pb, ar = orc.from_config(cfg)
    th = orc.init_params(ar, 1).astype(np.float64)
    b = np.array([[1.0, 0.1, -0.2], [-0.3, 1.0, 0.4]], np.float32)
    _, rb0 = orc.residuals(pb, ar, th, np.zeros((0, 3)), b, 1 / 16)
    P1 = ar.P // 2
    th2 = th.copy()
    th2[P1 - 1] += 0.25     # net- output bias
    th2[-1] += 0.5          # net+ output bias
    _, rb1 = orc.residuals(pb, ar, th2, np.zeros((0, 3)), b, 1 / 16)
    assert np.allclose(rb1 - rb0, 0.5, atol=1e-14)                     # both outside the sphere


def test_terms_partition_and_shards(orc):
    """per-term losses/grads sum to the total; contiguous shards with the global
    normalisation sum to the full batch (G18)."""
    cfg = _cfg([3, 6, 6, 1])
    pb, ar = orc.from_config(cfg)
    H = inputs.h_lattice(1 / 32)
    pts = orc.sample(0, 1, 0, 0, 600, H)
    b = orc.sample(1, 1, 0, 0, 80, H)
    th = orc.init_params(ar, 2)
    h = H / 2**24
    L, lt, g, gt = orc.loss_grad(pb, ar, th, pts, b, h, per_term=True)
    assert np.allclose(gt.sum(0), g, rtol=1e-13, atol=1e-18)
    for k in range(4):
        Lk, ltk, gk, _ = orc.loss_grad(pb, ar, th, pts, b, h, terms=1 << k)
        assert Lk == pytest.approx(lt[k], rel=1e-13, abs=1e-30)
        assert np.allclose(gk, gt[k], rtol=1e-12, atol=1e-20)
    acc_L, acc_g = 0.0, np.zeros(ar.P)
    for r in range(4):
        lo, hi = r * 600 // 4, (r + 1) * 600 // 4
        blo, bhi = r * 80 // 4, (r + 1) * 80 // 4
        Ls, _, gs, _ = orc.loss_grad(pb, ar, th, pts[lo:hi], b[blo:bhi], h, n_glob=600, nb_glob=80)
        acc_L += Ls
        acc_g += gs
    assert acc_L == pytest.approx(L, rel=1e-14)
    assert np.allclose(acc_g, g, rtol=1e-12, atol=1e-14 * np.abs(g).max())
    # determinism
    g1 = orc.loss_grad(pb, ar, th, pts, b, h)[2]
    assert np.array_equal(orc.loss_grad(pb, ar, th, pts, b, h)[2], g1)


def test_linear_in_theta_least_squares(orc):
    """North-star self-check 5: freezing the hidden layers makes r affine in the output
    layer (random features).  The loss minimiser from a brute-force dense least-squares
    solve (numpy QR) must zero the oracle's gradient and reproduce the LS residual."""
    cfg = _cfg([3, 12, 12, 1])
    pb, ar = orc.from_config(cfg)
    H = inputs.h_lattice(1 / 16)
    pts = orc.sample(0, 3, 0, 0, 300, H)
    b = orc.sample(1, 3, 0, 0, 60, H)
    h = H / 2**24
    th0 = orc.init_params(ar, 5).astype(np.float64)
    P1 = ar.P // 2
    out_idx = np.r_[P1 - 13:P1, ar.P - 13:ar.P]       # w_out (12) + b_out of each net
    r0, rb0 = orc.residuals(pb, ar, th0, pts, b, h)
    base = np.concatenate([r0 / np.sqrt(len(pts)), rb0 / np.sqrt(len(b))])
    cols = []
    for i in out_idx:                                  # r is affine: probe unit directions
        t = th0.copy()
        t[i] += 1.0
        r1, rb1 = orc.residuals(pb, ar, t, pts, b, h)
        cols.append(np.concatenate([r1 / np.sqrt(len(pts)), rb1 / np.sqrt(len(b))]) - base)
    A = np.stack(cols, 1)
    Q, R = np.linalg.qr(A)
    dx = -np.linalg.solve(R, Q.T @ base)
    Lstar = float(np.sum((A @ dx + base) ** 2))
    ts = th0.copy()
    ts[out_idx] += dx
    L, _, g, _ = orc.loss_grad(pb, ar, ts, pts, b, h)
    _, _, g0, _ = orc.loss_grad(pb, ar, th0, pts, b, h)
    assert L == pytest.approx(Lstar, rel=1e-9)
    assert np.linalg.norm(g[out_idx]) <= 1e-9 * np.linalg.norm(g0[out_idx])
    # Adam on the output layer only decreases the loss toward L*
    th, m, v = th0.copy(), np.zeros(ar.P), np.zeros(ar.P)
    Ls = []
    for t in range(1, 301):
        L_t, _, gt, _ = orc.loss_grad(pb, ar, th, pts, b, h)
        Ls.append(L_t)
        gm = np.zeros(ar.P)
        gm[out_idx] = gt[out_idx]
        th, m, v = orc.adam(th, m, v, gm, t, lr=0.05 / np.sqrt(t))
    assert Ls[-1] < Ls[0] and Ls[-1] >= Lstar * (1 - 1e-9)
    assert (Ls[-1] - Lstar) < 0.2 * (Ls[0] - Lstar)


def test_adam_closed_forms(orc):
    tr = SPEC["training"]
    th, m, v = orc.adam([1.0], [0.0], [0.0], [0.0], 1)
    assert th[0] == 1.0
    e = tr["adam_first_step"]
    th, m, v = orc.adam([0.0], [0.0], [0.0], [e["g"]], 1, lr=e["lr"])
    assert th[0] == pytest.approx(e["delta"], rel=1e-12)
    e = tr["adam_two_steps"]
    th, m, v = orc.adam([0.0], [0.0], [0.0], [e["g"]], 1)
    th, m, v = orc.adam(th, m, v, [e["g"]], 2)
    assert m[0] == pytest.approx(e["m"], rel=1e-14) and v[0] == pytest.approx(e["v"], rel=1e-14)


def test_adam_fp32_mirror_close_to_fp64(orc):
    rng = np.random.default_rng(6)
    P = 1000
    th = rng.normal(size=P).astype(np.float32)
    m = (rng.normal(size=P) * 1e-3).astype(np.float32)
    v = (rng.uniform(size=P) * 1e-6).astype(np.float32)
    g = (rng.normal(size=P) * 1e-3).astype(np.float32)
    a = orc.adam(th, m, v, g, 7)
    b = orc.adam_f32(th, m, v, g, 7)
    assert np.allclose(b[0], a[0], rtol=0, atol=4e-7 * np.abs(a[0]).max())
    assert np.allclose(b[1], a[1], rtol=1e-6)
    assert np.allclose(b[2], a[2], rtol=1e-6)


def test_xavier_init(orc):
    """G11: Glorot-uniform bounds, zero biases, deterministic, distinct per seed."""
    sizes = [3, 64, 64, 64, 1]
    _, ar = orc.from_config(_cfg(sizes))
    t0 = orc.init_params(ar, 0)
    assert np.array_equal(t0, orc.init_params(ar, 0))
    assert not np.array_equal(t0, orc.init_params(ar, 1))
    off = 0
    for net in range(2):
        for l in range(1, len(sizes)):
            fi, fo = sizes[l - 1], sizes[l]
            W = t0[off:off + fi * fo]
            a = np.sqrt(6 / (fi + fo))
            assert np.all(np.abs(W) <= a * (1 + 1e-6)) and np.abs(W).max() > 0.9 * a
            assert abs(W.mean()) < 5 * a / np.sqrt(3 * W.size)
            assert np.all(t0[off + fi * fo: off + fi * fo + fo] == 0)
            off += fi * fo + fo
    assert off == ar.P


def test_precision_emulations_are_close_to_fp64(orc):
    """The fp32 / bf16 emulation modes (noise-floor yardsticks) stay near
    fp64 on the well-conditioned terms (boundary + crossed)."""
    cfg = inputs.config("c2")
    cfg.update(sizes=[3, 32, 32, 32, 1])
    pb, ar = orc.from_config(cfg)
    H = cfg["H"]
    pts = orc.sample(0, 0, 0, 0, 2000, H)
    b = orc.sample(1, 0, 0, 0, 250, H)
    th = orc.init_params(ar, 0)
    L64, lt64, g64, _ = orc.loss_grad(pb, ar, th, pts, b, cfg["h"], terms=0b1100)
    L32, _, g32, _ = orc.loss_grad(pb, ar, th, pts, b, cfg["h"], terms=0b1100, mode=orc.MODE_F32)
    Lbf, _, gbf, _ = orc.loss_grad(pb, ar, th, pts, b, cfg["h"], terms=0b1100, mode=orc.MODE_BF16)
    assert abs(L32 - L64) < 1e-6 * L64
    assert np.linalg.norm(g32 - g64) < 1e-5 * np.linalg.norm(g64)
    assert abs(Lbf - L64) < 2e-2 * L64
    assert np.linalg.norm(gbf - g64) < 2e-2 * np.linalg.norm(g64)


def test_multiresolution_loss_gradient_matches_central_differences(orc):
    """S:353 example 3 "on a 10-point batch with L=2" (and S:348's multi-level loss, SURVEY 8f
    NEXT-1): the multi-resolution loss gradient vs central FD over all parameters, with
    non-unit level weights; the level-1 rows (half the cell width) cross the interface on a
    different set of arms than level 0.  Also: L = 1 reduces to the single-level loss."""
    cfg = _cfg([3, 4, 4, 1], act=0)
    pb, ar, pts, b, h = _mixed_batch(orc, cfg)
    th = np.random.default_rng(5).normal(size=ar.P) * 0.8
    w = [1.0, 0.5]
    L, g = orc.loss_grad_ml(pb, ar, th, pts, b, h, 2, w)
    L1, _, g1, _ = orc.loss_grad(pb, ar, th, pts, b, h)
    Lm1, gm1 = orc.loss_grad_ml(pb, ar, th, pts, b, h, 1)
    assert Lm1 == pytest.approx(L1, rel=1e-14) and np.allclose(gm1, g1, rtol=1e-14, atol=0)
    _, c0 = orc.classify(pb, pts, h)
    _, c1 = orc.classify(pb, pts, h / 2)
    assert (c0 == 2).sum() != (c1 == 2).sum() or not np.array_equal(c0, c1)
    fd = np.zeros(ar.P)
    for i in range(ar.P):
        tp, tm = th.copy(), th.copy()
        tp[i] += 1e-6
        tm[i] -= 1e-6
        fd[i] = (orc.loss_grad_ml(pb, ar, tp, pts, b, h, 2, w)[0] - orc.loss_grad_ml(pb, ar, tm, pts, b, h, 2, w)[0]) / 2e-6
    scale = np.abs(g).max()
    assert np.all(np.abs(g - fd) <= 1e-5 * np.maximum(np.abs(g), 1e-3 * scale))
    assert L > L1   # the level-1 terms add non-negative contributions
