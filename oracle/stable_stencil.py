"""Difference propagation through a tanh MLP: the numerically stable evaluation of the
uncrossed 7-point stencil (reading G27).  TEST INFRASTRUCTURE
ONLY (tests/ may import it; the product path never does).

The uncrossed residual of a point (in the M^-1-scaled form the CUDA path
and oracle.c use) is

    r = u(x) + c_hat * sum_j u(x + h a_j) - b / d,   c_hat = -(beta / h^2) / d,
    d = k + 6 beta / h^2,

and sum_j u(x + h a_j) = 6 u(x) + sum_d Du_d with the second differences
Du_d = u(x + h e_d) + u(x - h e_d) - 2 u(x), so

    r = c_c u(x) + c_hat * sum_d Du_d - b / d,   c_c = k / d   (= 1 + 6 c_hat).

This is the same number as the plain definition; only the evaluation order differs.  Instead
of 7 network values whose differences cancel to O(h^2), each hidden layer carries, per point
and axis d, the centre activation a, the first difference P_d = a(x + h e_d) - a(x) and the
second difference Q_d = a(x + h e_d) + a(x - h e_d) - 2 a(x).  With z, p_d, D_d the
pre-activation centre / first / second differences (linear layers: z = W a + b, p = W P,
D = W Q; no bias on differences), t = tanh z:

    tanh(z + d) - tanh(z) = (1 - t^2) d + g(d),
    g(d) = (1 - t^2) [(tanh d - d) - t tanh(d) d] / (1 + t tanh d),      (tanh addition)
    P = (1 - t^2) p + g(p),     Q = (1 - t^2) D + g(p) + g(D - p),

with tanh d - d from its odd Taylor series for |d| < 1/4 (no cancellation anywhere).  The
gradient is the chain rule through these maps (M = Q - P = tanh(z + D - p) - tanh z):

    dP/dz = -P (2t + P),  dP/dp = 1 - (t + P)^2,
    dQ/dz = -(2 t Q + P^2 + M^2),  dQ/dp = (M - P)(2t + M + P),  dQ/dD = 1 - (t + M)^2.

Pinned in tests/test_oracle_stable.py against the plain definition (oracle.c, fp64): equal
residuals and gradients.  `rnd` emulates a rounding for the noise-floor measurements of
DESIGN.md G27, at the CUDA path's rounding points: the operands of the hidden x hidden GEMMs
(activation rows, difference rows, gradient rows, W_2..W_NH); layer 1 and the output layer
stay unrounded (fp32 on the CUDA cores there).
"""
from __future__ import annotations

import numpy as np

# odd Taylor coefficients of tanh(d) - d = d^3 (c3 + d^2 (c5 + d^2 c7)) + O(d^9)
_TS = (-1.0 / 3.0, 2.0 / 15.0, -17.0 / 315.0)
CUT = 0.25


def tanh_minus_id(d: np.ndarray) -> np.ndarray:
    """tanh(d) - d: the series below CUT (truncation < 2e-5 relative), directly above."""
    d = np.asarray(d, np.float64)
    d2 = d * d
    s = _TS[2]
    for c in _TS[1::-1]:
        s = c + d2 * s
    return np.where(np.abs(d) < CUT, d * d2 * s, np.tanh(d) - d)


def g_fun(t, d):
    """g(d) = tanh(z + d) - tanh(z) - (1 - t^2) d, t = tanh z (tanh addition theorem)."""
    s = tanh_minus_id(d)
    td = d + s
    return (1.0 - t * t) * (s - t * td * d) / (1.0 + t * td)


def _layers(theta_net, sizes):
    off, out = 0, []
    for l in range(1, len(sizes)):
        fi, fo = sizes[l - 1], sizes[l]
        W = np.asarray(theta_net[off:off + fi * fo], np.float64).reshape(fo, fi)
        off += fi * fo
        b = np.asarray(theta_net[off:off + fo], np.float64)
        off += fo
        out.append((W, b))
    return out


def forward(theta_net, sizes, x, h, rnd=None):
    """Centre value and differences of one tanh network at points x [n, 3]:
    returns (u [n], dU [n, 3] = u(x + h e_d) - u(x), DU [n, 3] = second differences), cache."""
    R = rnd if rnd is not None else (lambda v: v)
    L = _layers(theta_net, sizes)
    x = np.asarray(x, np.float64)
    n = len(x)
    a = x
    P = np.broadcast_to(h * np.eye(3), (n, 3, 3)).copy()   # [n, axis d, feature]
    Q = np.zeros((n, 3, 3))
    cache = []
    for li, (W, b) in enumerate(L[:-1]):
        Rl = R if li > 0 else (lambda v: v)
        Wr = Rl(W)
        z = Rl(a) @ Wr.T + b
        p = Rl(P) @ Wr.T
        D = Rl(Q) @ Wr.T
        t = np.tanh(z)
        tt = t[:, None, :]
        gp, gm = g_fun(tt, p), g_fun(tt, D - p)
        Pn = (1.0 - tt * tt) * p + gp
        Qn = (1.0 - tt * tt) * D + gp + gm
        cache.append((a, P, Q, t, Pn, Qn))
        a, P, Q = t, Pn, Qn
    Wo, bo = L[-1]
    u = a @ Wo[0] + bo[0]
    dU = P @ Wo[0]
    DU = Q @ Wo[0]
    cache.append((a, P, Q))
    return u, dU, DU, cache


def backward(theta_net, sizes, cache, g_u, g_DU, rnd=None):
    """Gradient w.r.t. this network's parameters [W_l row-major, b_l per layer] of
    sum_i g_u[i] u_i + sum_{i,d} g_DU[i, d] DU_{i,d} (the first differences do not enter r)."""
    R = rnd if rnd is not None else (lambda v: v)
    L = _layers(theta_net, sizes)
    grads = []
    a, P, Q = cache[-1]
    Wo, bo = L[-1]
    g_u = np.asarray(g_u, np.float64)
    g_DU = np.asarray(g_DU, np.float64)
    grads.append((g_u @ a + np.einsum("nd,ndk->k", g_DU, Q)[None, :], np.array([g_u.sum()])))
    ga = g_u[:, None] * Wo[0][None, :]
    gP = np.zeros(P.shape)
    gQ = g_DU[:, :, None] * Wo[0][None, None, :]
    for li in range(len(L) - 2, -1, -1):
        W, b = L[li]
        a_in, P_in, Q_in, t, Pn, Qn = cache[li]
        if li < len(L) - 2:   # the CUDA path reads the rounded operand copies below the last layer
            t, Pn, Qn = R(t), R(Pn), R(Qn)
        tt = t[:, None, :]
        M = Qn - Pn
        gz = ga * (1.0 - t * t) - (gP * Pn * (2 * tt + Pn) + gQ * (2 * tt * Qn + Pn * Pn + M * M)).sum(axis=1)
        gp = gP * (1.0 - (tt + Pn) ** 2) + gQ * (M - Pn) * (2 * tt + M + Pn)
        gD = gQ * (1.0 - (tt + M) ** 2)
        gz, gp, gD = R(gz), R(gp), R(gD)
        Ri = R if li > 0 else (lambda v: v)
        gW = gz.T @ Ri(a_in) + np.einsum("ndo,ndi->oi", gp, Ri(P_in)) + np.einsum("ndo,ndi->oi", gD, Ri(Q_in))
        grads.append((gW, gz.sum(axis=0)))
        Wr = R(W)
        ga, gP, gQ = gz @ Wr, gp @ Wr, gD @ Wr
    out = []
    for gW, gb in reversed(grads):
        out += [gW.reshape(-1), gb.reshape(-1)]
    return np.concatenate(out)


def residual_coefficients(k: float, beta: float, h: float):
    """(c_c, c_hat) of the stable form, in fp64: d = k + 6 beta / h^2."""
    d = k + 6.0 * beta / (h * h)
    return k / d, -(beta / (h * h)) / d


def loss_grad_unx(theta_net, sizes, x, h, k, beta, rhs, n_glob=None, rnd=None):
    """Uncrossed-point loss (1/N) sum r^2 and its gradient through the stable form; rhs = b/d."""
    n_glob = len(x) if n_glob is None else n_glob
    cc, ch = residual_coefficients(k, beta, h)
    u, _, DU, cache = forward(theta_net, sizes, x, h, rnd)
    r = cc * u + ch * DU.sum(axis=1) - rhs
    L = float((r * r).sum() / n_glob)
    gr = 2.0 * r / n_glob
    g = backward(theta_net, sizes, cache, gr * cc, np.repeat((gr * ch)[:, None], 3, axis=1), rnd)
    return L, r, g


def bf16(v):
    """Round to bf16 (RNE) and back to fp64."""
    f = np.asarray(v, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)
