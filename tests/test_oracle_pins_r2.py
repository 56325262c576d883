"""Oracle pins added in round 2 (CPU, `-m "not gpu"`).

* theta snapping (reading G6): an arm whose crossing lies within 1e-6 of either end
  is assembled exactly like an arm that does not cross at all (near-side coefficient and
  network), so its row equals the row of the same point with the interface moved off the arm.
* DegenerateGradient: a sampled level set whose central-difference normal vanishes at
  a crossing raises it.
* bf16 emulation (MODE_BF16, G16): the C oracle's rounding points are pinned against
  an independent numpy statement of G16, and each rounding point is shown to matter (removing
  it from the numpy statement moves the result by more than the tolerance).
"""
import numpy as np
import pytest

from paper_2210_14907_b200 import inputs

H32 = 1.0 / 32
EPS = 2.0 ** -26          # fp32 ulp of [0.125, 0.25): the plane offset that puts theta = EPS/h


def _plane_cfg(c):
    cfg = inputs.config("c2")
    cfg.update(ls_kind=inputs.LS_PLANE, plane=((1.0, 0.0, 0.0), float(c)), H=inputs.h_lattice(H32))
    cfg["h"] = cfg["H"] / inputs.LATTICE
    return cfg


def _row_tuple(row):
    return ([row.coef[j] for j in range(7)], [row.tag[j] for j in range(7)], row.rhs, row.d, row.corr)


@pytest.mark.parametrize("near_end", [True, False])
def test_theta_snapping_equals_uncrossed_arm(orc, near_end):
    """theta < 1e-6 (near_end: the +x arm of a point in Omega-) or > 1 - 1e-6 (the -x
    arm of a point in Omega+) on the plane x = c: the row must equal the row of the same
    point with the plane moved off its arms (no crossing): coefficient -beta_s/h^2, the near
    side's network, no jump correction.  Both points are on the 2^-24 lattice."""
    c = 0.1875 + EPS                                    # fp32-exact plane offset
    px, arm, side = (0.1875, 1, 0) if near_end else (0.21875, 2, 1)
    p = np.array([px, 0.3125, -0.25], np.float32)
    pb, _ = orc.from_config(_plane_cfg(c))
    row = orc.assemble(pb, p, H32)
    th = (c - px) / H32 if near_end else (px - c) / H32
    assert (th < 1e-6) if near_end else (th > 1 - 1e-6)
    assert row.side == side and ((row.mask >> arm) & 1) == 1 - side   # the arm's end is across
    assert row.n_snapped == 1 and row.n_crossed_arms == 0
    # reference: the same point with no crossing on any arm (plane well away from the stencil)
    pb_far, _ = orc.from_config(_plane_cfg(0.75 if near_end else -0.75))
    ref = orc.assemble(pb_far, p, H32)
    assert ref.n_snapped == 0 and ref.n_crossed_arms == 0 and ref.side == side
    coef, tag, rhs, d, corr = _row_tuple(row)
    rcoef, rtag, rrhs, rd, rcorr = _row_tuple(ref)
    assert coef == rcoef and tag == rtag and corr == 0.0 and rhs == rrhs and d == rd
    beta = (1.0, 10.0)[side]
    assert tag[arm] == side and coef[arm] == -beta / H32 ** 2   # near-side beta and network


def test_theta_just_above_snap_is_crossed(orc):
    """Control for the snapping pin: at theta = 3 EPS / h = 1.43e-6 the arm is a crossed arm
    (far-side network, mu_hat from the harmonic blend, a jump correction)."""
    c = 0.1875 + 3 * EPS
    p = np.array([0.1875, 0.3125, -0.25], np.float32)
    pb, _ = orc.from_config(_plane_cfg(c))
    row = orc.assemble(pb, p, H32)
    assert row.n_snapped == 0 and row.n_crossed_arms == 1 and row.tag[1] == 1
    assert row.corr != 0.0 and row.coef[1] != -1.0 / H32 ** 2


def degenerate_grid_cfg():
    """An 8^3 sampled level set varying in x only, nodal values (-11, 1, -3) at x = -0.25, 0,
    0.25 (and -11 / -3 beyond): the linear crossing between x = 0 and 0.25 sits at x = 1/16
    where the central difference of the interpolant with step hc/2 = 1/8 is
    phi(3/16) - phi(-1/16) = -2 - (-2) = 0, so the normal is degenerate."""
    nc = 8
    g = np.linspace(-1.0, 1.0, nc + 1)
    px = np.where(g < -0.125, -11.0, np.where(g < 0.125, 1.0, -3.0))
    grid = np.broadcast_to(px[None, None, :], (nc + 1, nc + 1, nc + 1)).astype(np.float32).reshape(-1)
    cfg = inputs.config("c2")
    cfg.update(ls_kind=inputs.LS_GRID, grid=grid, grid_n=nc, H=inputs.h_lattice(H32))
    cfg["h"] = cfg["H"] / inputs.LATTICE
    # the crossed point: x = 1/16 - h/2 (theta = 1/2 on its +x arm)
    p = np.array([[0.0625 - H32 / 2, 0.5, -0.375]], np.float32)
    return cfg, p


def test_degenerate_gradient_raises(orc):
    cfg, p = degenerate_grid_cfg()
    pb, ar = orc.from_config(cfg)
    assert orc.phi(pb, p[0].astype(np.float64)) > 0
    assert orc.phi(pb, (p[0] + [H32, 0, 0]).astype(np.float64)) < 0
    with pytest.raises(RuntimeError, match="Degenerate"):
        orc.assemble(pb, p[0], H32)
    th = orc.init_params(ar, 0)
    with pytest.raises(RuntimeError):
        orc.loss_grad(pb, ar, th, p, np.zeros((0, 3), np.float32), cfg["h"])
    # a point of the same problem whose arms do not cross is assembled normally
    orc.assemble(pb, np.array([0.75, 0.0, 0.0], np.float32), H32)


# ---------------------------------------------------------------- bf16 emulation (G16)
def _bf16(a):
    """round-to-nearest-even to bfloat16, returned as float32"""
    u = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def _f32(a):
    return np.asarray(a, np.float64).astype(np.float32)


def _layers(theta, sizes, net):
    off = net * inputs.param_count(sizes, 1)
    out = []
    for l in range(1, len(sizes)):
        fi, fo = sizes[l - 1], sizes[l]
        W = theta[off:off + fi * fo].reshape(fo, fi).astype(np.float64)
        b = theta[off + fi * fo:off + fi * fo + fo].astype(np.float64)
        out.append((W, b, off))
        off += fi * fo + fo
    return out


def emulate_bf16(theta, sizes, act, net, x, cot, skip=()):
    """G16 written out from DESIGN.md: hidden x hidden GEMM operands (weights, activations,
    back-propagated deltas) RNE-rounded to bf16 with fp32 accumulation; layer 1 and the
    output layer in fp32; tanh' of hidden layers 1..NH-1 from the bf16 operand copy (layer NH
    exact); SiLU' of hidden layers 2..NH-1 stored in bf16; the bias gradients of hidden layers
    1..NH-1 and dW_1 are reductions of the bf16 delta (tensor-core tails), layer-1 inputs
    entering dW_1 as the two-term bf16 split x = bf16(x) + bf16(x - bf16(x)).
    `skip` removes named rounding points (mutation checks).  Returns (u, grad)."""
    L = len(sizes)
    lay = _layers(theta, sizes, net)
    bf = (lambda a, k: _f32(a) if k in skip else _bf16(a))
    h = [_f32(x)]
    z = [None]
    for l in range(1, L):
        W, b, _ = lay[l - 1]
        gemm = 2 <= l <= L - 2
        hin = h[-1].astype(np.float64)
        if gemm:
            W = bf(W, "w").astype(np.float64)
            hin = bf(hin, "h_fwd").astype(np.float64)
        zz = _f32(W @ hin + b)
        z.append(zz)
        if l < L - 1:
            zd = zz.astype(np.float64)
            a = np.tanh(zd) if act == inputs.ACT_TANH else zd / (1 + np.exp(-zd))
            h.append(_f32(a))
        else:
            h.append(zz)
    u = float(h[-1][0])
    grad = np.zeros(len(theta))
    d = np.array([cot], np.float32)
    for l in range(L - 1, 0, -1):
        W, b, off = lay[l - 1]
        fi, fo = sizes[l - 1], sizes[l]
        gemm = 2 <= l <= L - 2
        tail = l <= L - 3
        dv = d.astype(np.float64)
        if gemm or (tail and l == 1):
            dv = bf(dv, "d_dw").astype(np.float64)
        hv = h[l - 1].astype(np.float64)
        if gemm:
            hv = bf(hv, "h_dw").astype(np.float64)
        if tail and l == 1:
            hi = _bf16(hv)   # mutation "split": one bf16 term instead of two
            hv = hi.astype(np.float64) + (0.0 if "split" in skip else _bf16(hv - hi).astype(np.float64))
        grad[off:off + fi * fo] = np.outer(dv, hv).reshape(-1)
        grad[off + fi * fo:off + fi * fo + fo] = bf(d, "d_db") if tail else d
        if l == 1:
            break
        Wt = W
        dd = d.astype(np.float64)
        if gemm:
            Wt = bf(W, "w").astype(np.float64)
            dd = bf(dd, "d_dh").astype(np.float64)
        acc = _f32(Wt.T @ dd).astype(np.float64)
        zl = z[l - 1].astype(np.float64)
        hl = h[l - 1].astype(np.float64)
        if act == inputs.ACT_TANH:
            hh = bf(hl, "tanh_d").astype(np.float64) if l - 1 <= L - 3 else hl
            ad = 1.0 - hh * hh
        else:
            sg = 1.0 / (1.0 + np.exp(-zl))
            ad = sg * (1.0 + zl * (1.0 - sg))
            if 2 <= l - 1 <= L - 3:
                ad = bf(ad, "silu_d").astype(np.float64)
        d = _f32(acc * _f32(ad))
    return u, grad


POINTS = [np.array(v, np.float32) for v in ([0.3, -0.7, 0.55], [-0.81, 0.12, 0.9], [0.05, 0.5, -0.33],
                                             [0.6, 0.6, -0.6], [-0.2, -0.9, 0.1])]


def _setup(orc, act):
    cfg = inputs.config("c5", width=32)
    cfg.update(sizes=[3, 32, 32, 32, 32, 1], act=act)
    _, ar = orc.from_config(cfg)
    th = inputs.random_theta(cfg["sizes"], 2, 11, bias_scale=0.3)
    return cfg, ar, th


@pytest.mark.parametrize("act", [inputs.ACT_TANH, inputs.ACT_SILU])
def test_bf16_emulation_matches_g16(orc, act):
    """The C oracle's MODE_BF16 forward and per-evaluation backward equal the numpy G16
    statement up to fp32 accumulation order (1e-5 relative), on both networks."""
    cfg, ar, th = _setup(orc, act)
    for net in (0, 1):
        for x in POINTS:
            cot = 0.37
            u_c = orc.forward(ar, th, net, x.astype(np.float64), mode=orc.MODE_BF16)
            g_c = orc.backward(ar, th, net, x.astype(np.float64), cot, mode=orc.MODE_BF16)
            u_n, g_n = emulate_bf16(th, cfg["sizes"], act, net, x, cot)
            assert abs(u_c - u_n) <= 1e-5 * max(abs(u_c), 1e-3)
            assert np.linalg.norm(g_c - g_n) <= 1e-5 * np.linalg.norm(g_c)


@pytest.mark.parametrize("act,point", [(inputs.ACT_TANH, p) for p in ("w", "h_fwd", "d_dh", "d_dw", "h_dw",
                                                                        "d_db", "tanh_d", "split")] +
                         [(inputs.ACT_SILU, "silu_d")])
def test_bf16_emulation_rounding_points_matter(orc, act, point):
    """Mutation check: dropping any one G16 rounding point from the numpy statement moves the
    forward value or the gradient by far more than the 1e-5 agreement above, so each point
    of the C emulation is pinned individually."""
    cfg, ar, th = _setup(orc, act)
    worst = 0.0
    for net in (0, 1):
        for x in POINTS:
            u_c = orc.forward(ar, th, net, x.astype(np.float64), mode=orc.MODE_BF16)
            g_c = orc.backward(ar, th, net, x.astype(np.float64), 0.37, mode=orc.MODE_BF16)
            u_m, g_m = emulate_bf16(th, cfg["sizes"], act, net, x, 0.37, skip=(point,))
            worst = max(worst, abs(u_c - u_m) / max(abs(u_c), 1e-3),
                        np.linalg.norm(g_c - g_m) / np.linalg.norm(g_c))
    assert worst > 1e-4, (point, worst)
