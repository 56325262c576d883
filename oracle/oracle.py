"""ctypes wrapper of the C oracle (oracle.c).  TEST INFRASTRUCTURE ONLY.

Exposes numpy-level functions; every computation happens in oracle.c, in
fp64 unless an emulation mode (F32/BF16) is requested for noise-floor
measurements.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
HDR = os.path.join(HERE, "oracle.h")
LIB = os.path.join(HERE, "liboracle.so")

MODE_F64, MODE_F32, MODE_BF16 = 0, 1, 2
T_UNX_MINUS, T_UNX_PLUS, T_CROSSED, T_BOUNDARY = 0, 1, 2, 3
T_ALL = 0xF


def build(force: bool = False) -> str:
    stale = (not os.path.exists(LIB) or
             os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)))
    if force or stale:
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", LIB + ".tmp", SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class Problem(C.Structure):
    _fields_ = [("ls_kind", C.c_int), ("n_spheres", C.c_int),
                ("centers", C.POINTER(C.c_double)), ("radii", C.POINTER(C.c_double)),
                ("star_r0", C.c_double), ("star_amp", C.c_double),
                ("star_m", C.c_int), ("star_n", C.c_int),
                ("plane_n", C.c_double * 3), ("plane_c", C.c_double),
                ("beta", C.c_double * 2), ("k", C.c_double * 2),
                ("source", C.c_int), ("n_charges", C.c_int),
                ("q", C.POINTER(C.c_double)), ("charge_centers", C.POINTER(C.c_double)),
                ("charge_sigma", C.c_double), ("poly", C.POINTER(C.c_double)),
                ("lambda_b", C.c_double), ("grid_n", C.c_int), ("grid_phi", C.POINTER(C.c_double)),
                ("mu_kind", C.c_int), ("mu_lin", C.POINTER(C.c_double))]


class Arch(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("sizes", C.POINTER(C.c_int)),
                ("act", C.c_int), ("n_nets", C.c_int)]


class Row(C.Structure):
    _fields_ = [("pos", (C.c_float * 3) * 7), ("tag", C.c_int * 7), ("coef", C.c_double * 7),
                ("f", C.c_double), ("corr", C.c_double), ("rhs", C.c_double), ("d", C.c_double),
                ("side", C.c_int), ("mask", C.c_int), ("crossed", C.c_int),
                ("n_crossed_arms", C.c_int), ("n_snapped", C.c_int), ("theta", C.c_double * 7)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        P = C.POINTER
        L.orc_philox.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.orc_sample.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                 P(C.c_float)]
        L.orc_phi.restype = C.c_double
        L.orc_phi.argtypes = [P(Problem), P(C.c_double)]
        L.orc_side.argtypes = [P(Problem), P(C.c_double)]
        L.orc_crossing.argtypes = [P(Problem), P(C.c_double), P(C.c_double), P(C.c_double),
                                   P(C.c_double), P(C.c_double)]
        L.orc_crossing_bisect.argtypes = [P(Problem), P(C.c_double), P(C.c_double), P(C.c_double)]
        L.orc_normal.argtypes = [P(Problem), P(C.c_double), P(C.c_double)]
        L.orc_exact.argtypes = [P(Problem), C.c_int, P(C.c_double), P(C.c_double), P(C.c_double)]
        for fn in ("orc_f",):
            getattr(L, fn).restype = C.c_double
            getattr(L, fn).argtypes = [P(Problem), C.c_int, P(C.c_double)]
        L.orc_mu.restype = C.c_double
        L.orc_mu.argtypes = [P(Problem), C.c_int, P(C.c_double), P(C.c_double)]
        L.orc_alpha.restype = C.c_double
        L.orc_alpha.argtypes = [P(Problem), P(C.c_double)]
        L.orc_sigma.restype = C.c_double
        L.orc_sigma.argtypes = [P(Problem), P(C.c_double), P(C.c_double)]
        L.orc_g.restype = C.c_double
        L.orc_g.argtypes = [P(Problem), P(C.c_double)]
        L.orc_assemble.argtypes = [P(Problem), P(C.c_float), C.c_float, C.c_int, P(Row)]
        L.orc_classify.argtypes = [P(Problem), P(C.c_float), C.c_int64, C.c_float,
                                   P(C.c_uint8), P(C.c_uint8)]
        L.orc_param_count.restype = C.c_int64
        L.orc_error_norms.argtypes = [P(Problem), P(Arch), P(C.c_double), C.c_int, C.c_int, P(C.c_double)]
        L.orc_param_count.argtypes = [P(Arch)]
        L.orc_init_params.argtypes = [P(Arch), C.c_uint64, P(C.c_float)]
        L.orc_forward.restype = C.c_double
        L.orc_forward.argtypes = [P(Arch), P(C.c_double), C.c_int, P(C.c_double), C.c_int]
        L.orc_backward.argtypes = [P(Arch), P(C.c_double), C.c_int, P(C.c_double), C.c_double,
                                   C.c_int, P(C.c_double)]
        L.orc_loss_grad.argtypes = [P(Problem), P(Arch), P(C.c_double), P(C.c_float), C.c_int64,
                                    P(C.c_float), C.c_int64, C.c_float, C.c_int64, C.c_int64,
                                    C.c_int, C.c_uint, P(C.c_double), P(C.c_double),
                                    P(C.c_double), C.c_int]
        L.orc_residuals.argtypes = [P(Problem), P(Arch), P(C.c_double), P(C.c_float), C.c_int64,
                                    P(C.c_float), C.c_int64, C.c_float, C.c_int,
                                    P(C.c_double), P(C.c_double)]
        L.orc_residual_exact.argtypes = [P(Problem), P(C.c_float), C.c_int64, C.c_float,
                                         P(C.c_double), P(C.c_double), P(C.c_uint8)]
        L.orc_eval.argtypes = [P(Problem), P(Arch), P(C.c_double), P(C.c_float), C.c_int64,
                               C.c_int, P(C.c_double)]
        L.orc_adam.argtypes = [C.c_int64, P(C.c_double), P(C.c_double), P(C.c_double),
                               P(C.c_double), C.c_int64, C.c_double, C.c_double, C.c_double,
                               C.c_double]
        L.orc_adam_f32.argtypes = [C.c_int64, P(C.c_float), P(C.c_float), P(C.c_float),
                                   P(C.c_float), C.c_int64, C.c_float, C.c_float, C.c_float,
                                   C.c_float]
        L.orc_num_threads.restype = C.c_int
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _theta(a):
    """theta as fp64: an fp32 vector is promoted exactly; an fp64 vector (finite-
    difference pins) is passed through unchanged."""
    return np.ascontiguousarray(np.asarray(a).astype(np.float64))


class OracleProblem:
    """Holds an orc_problem plus the arrays it points to (kept alive)."""

    def __init__(self, cfg: dict, poly=None):
        f32 = lambda v: float(np.float32(v))  # the CUDA path receives fp32 values
        self._keep = []
        p = Problem()
        p.ls_kind = cfg["ls_kind"]
        cen = _f64(np.asarray(cfg["centers"], np.float32).reshape(-1, 3))
        rad = _f64(np.asarray(cfg["radii"], np.float32).reshape(-1))
        self._keep += [cen, rad]
        p.n_spheres = len(rad)
        p.centers = _ptr(cen, C.c_double)
        p.radii = _ptr(rad, C.c_double)
        r0, amp, m, n = cfg["star"]
        p.star_r0, p.star_amp, p.star_m, p.star_n = f32(r0), f32(amp), int(m), int(n)
        pn, pc = cfg["plane"]
        for i in range(3):
            p.plane_n[i] = f32(pn[i])
        p.plane_c = f32(pc)
        p.beta[0], p.beta[1] = f32(cfg["beta"][0]), f32(cfg["beta"][1])
        p.k[0], p.k[1] = f32(cfg["k"][0]), f32(cfg["k"][1])
        p.source = cfg["source"]
        q = _f64(np.asarray(cfg["charges_q"], np.float32).reshape(-1))
        qc = _f64(np.asarray(cfg["charges_c"], np.float32).reshape(-1, 3))
        self._keep += [q, qc]
        p.n_charges = len(q)
        p.q = _ptr(q, C.c_double)
        p.charge_centers = _ptr(qc, C.c_double)
        p.charge_sigma = f32(cfg["charge_sigma"])
        if poly is not None:
            pa = _f64(np.asarray(poly).reshape(2, 10))
            self._keep.append(pa)
            p.poly = _ptr(pa, C.c_double)
        p.lambda_b = f32(cfg["lambda_b"])
        p.mu_kind = int(cfg.get("mu_kind", 0))
        if cfg.get("mu_lin") is not None:
            ml = _f64(np.asarray(cfg["mu_lin"], np.float32).reshape(2, 4))
            self._keep.append(ml)
            p.mu_lin = _ptr(ml, C.c_double)
        if cfg.get("grid") is not None:   # sampled level set: fp32 nodal values (as the CUDA path gets)
            gphi = _f64(np.asarray(cfg["grid"], np.float32).reshape(-1))
            self._keep.append(gphi)
            p.grid_n = int(round(len(gphi) ** (1.0 / 3.0))) - 1
            assert (p.grid_n + 1) ** 3 == len(gphi)
            p.grid_phi = _ptr(gphi, C.c_double)
        self.s = p
        self.ref = C.byref(p)


class OracleArch:
    def __init__(self, sizes, act: int, n_nets: int):
        self.sizes = np.ascontiguousarray(np.asarray(sizes, np.int32))
        a = Arch()
        a.n_layers = len(sizes)
        a.sizes = _ptr(self.sizes, C.c_int)
        a.act = act
        a.n_nets = n_nets
        self.s = a
        self.ref = C.byref(a)

    @property
    def P(self) -> int:
        return int(lib().orc_param_count(self.ref))


def from_config(cfg: dict, poly=None):
    return OracleProblem(cfg, poly), OracleArch(cfg["sizes"], cfg["act"], cfg["n_nets"])


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(ctr, np.uint32))
    k = np.ascontiguousarray(np.asarray(key, np.uint32))
    out = np.zeros(4, np.uint32)
    lib().orc_philox(_ptr(c, C.c_uint32), _ptr(k, C.c_uint32), _ptr(out, C.c_uint32))
    return out


def sample(kind: int, seed: int, step: int, first: int, n: int, H: int) -> np.ndarray:
    pts = np.zeros((n, 3), np.float32)
    lib().orc_sample(kind, seed, step, first, n, H, _ptr(pts, C.c_float))
    return pts


def phi(pb: OracleProblem, x) -> float:
    return lib().orc_phi(pb.ref, _ptr(_f64(x), C.c_double))


def side(pb: OracleProblem, x) -> int:
    return lib().orc_side(pb.ref, _ptr(_f64(x), C.c_double))


def crossing(pb: OracleProblem, a, b):
    th = np.zeros(1)
    xg = np.zeros(3)
    nr = np.zeros(3)
    rc = lib().orc_crossing(pb.ref, _ptr(_f64(a), C.c_double), _ptr(_f64(b), C.c_double),
                            _ptr(th, C.c_double), _ptr(xg, C.c_double), _ptr(nr, C.c_double))
    if rc < 0:
        raise RuntimeError("degenerate gradient")
    return (float(th[0]), xg, nr) if rc == 1 else None


def crossing_bisect(pb: OracleProblem, a, b):
    th = np.zeros(1)
    rc = lib().orc_crossing_bisect(pb.ref, _ptr(_f64(a), C.c_double), _ptr(_f64(b), C.c_double),
                                   _ptr(th, C.c_double))
    return float(th[0]) if rc == 1 else None


def normal(pb: OracleProblem, x):
    nr = np.zeros(3)
    rc = lib().orc_normal(pb.ref, _ptr(_f64(x), C.c_double), _ptr(nr, C.c_double))
    if rc < 0:
        raise RuntimeError("degenerate gradient")
    return nr


def exact(pb, s, x):
    u = np.zeros(1)
    g = np.zeros(3)
    rc = lib().orc_exact(pb.ref, s, _ptr(_f64(x), C.c_double), _ptr(u, C.c_double),
                         _ptr(g, C.c_double))
    return None if rc < 0 else (float(u[0]), g)


def f(pb, s, x) -> float:
    return lib().orc_f(pb.ref, s, _ptr(_f64(x), C.c_double))


def mu(pb, s, x):
    """(mu_s(x), grad mu_s(x)) of the problem's diffusion coefficient"""
    g = np.zeros(3)
    m = lib().orc_mu(pb.ref, s, _ptr(_f64(x), C.c_double), _ptr(g, C.c_double))
    return float(m), g


def alpha(pb, x) -> float:
    return lib().orc_alpha(pb.ref, _ptr(_f64(x), C.c_double))


def sigma(pb, x, n) -> float:
    return lib().orc_sigma(pb.ref, _ptr(_f64(x), C.c_double), _ptr(_f64(n), C.c_double))


def g(pb, x) -> float:
    return lib().orc_g(pb.ref, _ptr(_f64(x), C.c_double))


def assemble(pb, p, h: float, sign_mutation: bool = False) -> Row:
    row = Row()
    rc = lib().orc_assemble(pb.ref, _ptr(_f32(p), C.c_float), float(np.float32(h)),
                            int(sign_mutation), C.byref(row))
    if rc == -1:
        raise ValueError("OutOfDomain")
    if rc == -2:
        raise RuntimeError("DegenerateGradient")
    return row


def classify(pb, pts, h: float):
    pts = _f32(pts).reshape(-1, 3)
    n = len(pts)
    mask = np.zeros(n, np.uint8)
    cls = np.zeros(n, np.uint8)
    rc = lib().orc_classify(pb.ref, _ptr(pts, C.c_float), n, float(np.float32(h)),
                            _ptr(mask, C.c_uint8), _ptr(cls, C.c_uint8))
    if rc:
        raise ValueError("OutOfDomain")
    return mask, cls


def init_params(arch: OracleArch, seed: int) -> np.ndarray:
    th = np.zeros(arch.P, np.float32)
    lib().orc_init_params(arch.ref, seed, _ptr(th, C.c_float))
    return th


def forward(arch, theta, net, x, mode=MODE_F64) -> float:
    th = _theta(theta)
    return lib().orc_forward(arch.ref, _ptr(th, C.c_double), net, _ptr(_f64(x), C.c_double), mode)


def backward(arch, theta, net, x, cot, mode=MODE_F64) -> np.ndarray:
    th = _theta(theta)
    g_ = np.zeros(arch.P)
    lib().orc_backward(arch.ref, _ptr(th, C.c_double), net, _ptr(_f64(x), C.c_double),
                       float(cot), mode, _ptr(g_, C.c_double))
    return g_


def loss_grad(pb, arch, theta, pts, bpts, h, n_glob=None, nb_glob=None, mode=MODE_F64,
              terms=T_ALL, per_term=False, nthreads=0):
    """Returns (loss, loss_terms[4], grad[P], grad_terms[4,P] or None), all fp64."""
    th = _theta(theta)
    pts = _f32(pts).reshape(-1, 3)
    bpts = _f32(bpts).reshape(-1, 3)
    n, nb = len(pts), len(bpts)
    n_glob = n if n_glob is None else n_glob
    nb_glob = nb if nb_glob is None else nb_glob
    lt = np.zeros(4)
    gr = np.zeros(arch.P)
    gt = np.zeros((4, arch.P)) if per_term else None
    rc = lib().orc_loss_grad(pb.ref, arch.ref, _ptr(th, C.c_double), _ptr(pts, C.c_float), n,
                             _ptr(bpts, C.c_float), nb, float(np.float32(h)),
                             max(n_glob, 1), max(nb_glob, 1), mode, terms,
                             _ptr(lt, C.c_double), _ptr(gr, C.c_double),
                             _ptr(gt, C.c_double) if per_term else None, nthreads)
    if rc == -1:
        raise ValueError("OutOfDomain")
    if rc == -2:
        raise RuntimeError("DegenerateGradient")
    return float(lt.sum()), lt, gr, gt


def loss_grad_ml(pb, arch, theta, pts, bpts, h0, n_levels, level_weights=None, n_glob=None, nb_glob=None,
                 mode=MODE_F64):
    """Multi-resolution loss ("implicit cells at multi-resolutions",
    P:98 "three levels of implicit refinement"): the same centres at h_l = h0 / 2^l,
    L = (1/N) sum_p sum_l w_l r_p(h_l)^2 + (lambda_b/N_b) sum_b r_b^2, w_l = 1 by default,
    boundary term once.  Written as the definition: one single-level loss per level over the
    interior points (no boundary) plus the boundary-only loss, weighted and summed."""
    pts = _f32(pts).reshape(-1, 3)
    bpts = _f32(bpts).reshape(-1, 3)
    ng = len(pts) if n_glob is None else n_glob
    nbg = len(bpts) if nb_glob is None else nb_glob
    none = np.zeros((0, 3), np.float32)
    L, _, g, _ = loss_grad(pb, arch, theta, none, bpts, h0, n_glob=ng, nb_glob=nbg, mode=mode)
    for lev in range(n_levels):
        w = 1.0 if level_weights is None else float(level_weights[lev])
        Ll, _, gl, _ = loss_grad(pb, arch, theta, pts, none, h0 / 2 ** lev, n_glob=ng, nb_glob=nbg, mode=mode)
        L, g = L + w * Ll, g + w * gl
    return L, g


def residuals(pb, arch, theta, pts, bpts, h, mode=MODE_F64):
    th = _theta(theta)
    pts = _f32(pts).reshape(-1, 3)
    bpts = _f32(bpts).reshape(-1, 3)
    r = np.zeros(len(pts))
    rb = np.zeros(len(bpts))
    rc = lib().orc_residuals(pb.ref, arch.ref, _ptr(th, C.c_double), _ptr(pts, C.c_float),
                             len(pts), _ptr(bpts, C.c_float), len(bpts), float(np.float32(h)),
                             mode, _ptr(r, C.c_double), _ptr(rb, C.c_double))
    if rc:
        raise ValueError("assembly error %d" % rc)
    return r, rb


def residual_exact(pb, pts, h):
    """(raw, r, cls) with the manufactured solution substituted for the networks."""
    pts = _f32(pts).reshape(-1, 3)
    n = len(pts)
    raw, r, cls = np.zeros(n), np.zeros(n), np.zeros(n, np.uint8)
    rc = lib().orc_residual_exact(pb.ref, _ptr(pts, C.c_float), n, float(np.float32(h)),
                                  _ptr(raw, C.c_double), _ptr(r, C.c_double),
                                  _ptr(cls, C.c_uint8))
    if rc:
        raise ValueError("assembly error %d" % rc)
    return raw, r, cls


def evaluate(pb, arch, theta, pts, mode=MODE_F64) -> np.ndarray:
    th = _theta(theta)
    pts = _f32(pts).reshape(-1, 3)
    u = np.zeros(len(pts))
    lib().orc_eval(pb.ref, arch.ref, _ptr(th, C.c_double), _ptr(pts, C.c_float), len(pts), mode,
                   _ptr(u, C.c_double))
    return u


def error_norms(pb, arch, theta, M, mode=MODE_F64):
    """(rmse, linf) of the pair against the exact solution over the (M+1)^3 nodal grid
    (Table 1's columns)."""
    th = _theta(theta)
    out = np.zeros(2)
    rc = lib().orc_error_norms(pb.ref, arch.ref, _ptr(th, C.c_double), int(M), mode, _ptr(out, C.c_double))
    if rc:
        raise ValueError("no closed-form solution for this problem")
    return float(out[0]), float(out[1])


def convergence_order(e_coarse: float, e_fine: float) -> float:
    """log2(e_coarse / e_fine) for a resolution doubling (Table 1 "Order")."""
    if not (e_coarse > 0 and e_fine > 0):
        raise ValueError("NonPositiveError")
    return float(np.log2(e_coarse / e_fine))


def adam(theta, m, v, g_, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    th, m, v = _f64(theta).copy(), _f64(m).copy(), _f64(v).copy()
    gg = _f64(g_)
    lib().orc_adam(len(th), _ptr(th, C.c_double), _ptr(m, C.c_double), _ptr(v, C.c_double),
                   _ptr(gg, C.c_double), t, lr, b1, b2, eps)
    return th, m, v


def adam_f32(theta, m, v, g_, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    th, m, v = _f32(theta).copy(), _f32(m).copy(), _f32(v).copy()
    gg = _f32(g_)
    lib().orc_adam_f32(len(th), _ptr(th, C.c_float), _ptr(m, C.c_float), _ptr(v, C.c_float),
                       _ptr(gg, C.c_float), t, lr, b1, b2, eps)
    return th, m, v


def num_threads() -> int:
    return int(lib().orc_num_threads())
