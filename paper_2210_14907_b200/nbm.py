"""ctypes binding of libnbm.so (include/nbm.h).  Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels.  There is no CPU fallback: if the
library is missing or no CUDA device is present the calls raise.

The functions keep the C names (nbm_create, nbm_sample, nbm_loss_grad, nbm_eval,
nbm_adam_step, ...) and take torch tensors for device buffers (PyTorch supplies device
memory and streams only).  `Solver` is a thin convenience wrapper over one handle.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NBM_LIB", os.path.join(HERE, "libnbm.so"))   # override: experiments

NBM_OK = 0
ERRORS = {1: "NBM_E_INVALID_ARCH", 2: "NBM_E_INVALID_PROBLEM", 3: "NBM_E_CAPACITY", 4: "NBM_E_CUDA",
          5: "NBM_E_ARG", 6: "NBM_E_OUT_OF_DOMAIN", 7: "NBM_E_DEGENERATE", 8: "NBM_E_NONFINITE"}
LS_NONE, LS_SPHERES, LS_STAR, LS_PLANE = 0, 1, 2, 3
SRC_SINE3PI, SRC_PAIR, SRC_GAUSS = 0, 1, 2
ACT_TANH, ACT_SILU = 0, 1
PREC_FP32, PREC_BF16 = 0, 1
STENCIL_DIRECT, STENCIL_STABLE = 0, 1   # NBM_STENCIL_* (G27)
POINTS_INTERIOR, POINTS_BOUNDARY = 0, 1
TERM_UNX_MINUS, TERM_UNX_PLUS, TERM_CROSSED, TERM_BOUNDARY, TERM_ALL = 1, 2, 4, 8, 15


class NbmError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class nbm_levelset(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int), ("centers", C.POINTER(C.c_float)),
                ("radii", C.POINTER(C.c_float)), ("star_r0", C.c_float), ("star_amp", C.c_float),
                ("star_m", C.c_int), ("star_n", C.c_int), ("plane_n", C.c_float * 3),
                ("plane_c", C.c_float), ("grid_n", C.c_int), ("grid_phi", C.POINTER(C.c_float))]


class nbm_problem(C.Structure):
    _fields_ = [("box_lo", C.c_float * 3), ("box_hi", C.c_float * 3), ("ls", nbm_levelset),
                ("beta_minus", C.c_float), ("beta_plus", C.c_float), ("k_minus", C.c_float),
                ("k_plus", C.c_float), ("source", C.c_int), ("n_charges", C.c_int),
                ("q", C.POINTER(C.c_float)), ("charge_centers", C.POINTER(C.c_float)),
                ("charge_sigma", C.c_float), ("lambda_b", C.c_float), ("mu_kind", C.c_int),
                ("mu_lin", (C.c_float * 4) * 2)]


class nbm_arch(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("sizes", C.POINTER(C.c_int)), ("act", C.c_int),
                ("prec", C.c_int), ("n_nets", C.c_int), ("stencil", C.c_int)]


_lib = None


def lib():
    """Load libnbm.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, v, i64, f, u64 = C.POINTER, C.c_void_p, C.c_int64, C.c_float, C.c_uint64
        L.nbm_version.restype = C.c_char_p
        L.nbm_arch_param_count.restype = i64
        L.nbm_arch_param_count.argtypes = [P(nbm_arch)]
        L.nbm_check.argtypes = [P(nbm_problem), P(nbm_arch)]
        L.nbm_create.argtypes = [P(nbm_problem), P(nbm_arch), C.c_int, i64, P(v)]
        L.nbm_destroy.argtypes = [v]
        L.nbm_destroy.restype = None
        L.nbm_param_count.restype = i64
        L.nbm_param_count.argtypes = [v]
        L.nbm_last_error.restype = C.c_char_p
        L.nbm_last_error.argtypes = [v]
        L.nbm_status.argtypes = [v, v]
        L.nbm_init_params.argtypes = [v, u64, v, v]
        L.nbm_sample.argtypes = [v, u64, u64, C.c_int, i64, i64, f, v, v]
        L.nbm_loss_grad.argtypes = [v, v, v, i64, v, i64, f, i64, i64, C.c_uint, v, v, v]
        L.nbm_eval.argtypes = [v, v, v, i64, v, v]
        L.nbm_error_norms.argtypes = [v, v, C.c_int, v, v]
        L.nbm_classify.argtypes = [v, v, i64, f, v, v, v]
        L.nbm_adam_step.argtypes = [v, v, v, v, v, i64, f, f, f, f, v]
        L.nbm_loss_grad_ml.argtypes = [v, v, v, i64, v, i64, f, C.c_int, v, i64, i64, C.c_uint, v, v, v]
        L.nbm_sample_at.argtypes = [v, u64, v, C.c_int, i64, i64, f, v, v]
        L.nbm_adam_step_at.argtypes = [v, v, v, v, v, v, f, f, f, f, v]
        L.nbm_timing_enable.argtypes = [v, C.c_int]
        L.nbm_timing_read.argtypes = [v, P(C.c_double), P(C.c_double), P(i64)]
        L.nbm_last_launch_count.argtypes = [v]
        _lib = L
    return _lib


class Descriptors:
    """nbm_problem / nbm_arch built from an inputs.config() dict (keeps arrays alive)."""

    def __init__(self, cfg: dict):
        self._keep = []
        p = nbm_problem()
        for d in range(3):
            p.box_lo[d], p.box_hi[d] = cfg["box"][0], cfg["box"][1]
        ls = nbm_levelset()
        ls.kind = cfg["ls_kind"]
        cen = np.ascontiguousarray(np.asarray(cfg["centers"], np.float32).reshape(-1))
        rad = np.ascontiguousarray(np.asarray(cfg["radii"], np.float32).reshape(-1))
        self._keep += [cen, rad]
        ls.n = len(rad)
        ls.centers = cen.ctypes.data_as(C.POINTER(C.c_float))
        ls.radii = rad.ctypes.data_as(C.POINTER(C.c_float))
        r0, amp, m, n = cfg["star"]
        ls.star_r0, ls.star_amp, ls.star_m, ls.star_n = r0, amp, int(m), int(n)
        pn, pc = cfg["plane"]
        for d in range(3):
            ls.plane_n[d] = pn[d]
        ls.plane_c = pc
        if cfg.get("grid") is not None:
            gphi = np.ascontiguousarray(np.asarray(cfg["grid"], np.float32).reshape(-1))
            self._keep.append(gphi)
            ls.grid_n = int(round(len(gphi) ** (1.0 / 3.0))) - 1
            ls.grid_phi = gphi.ctypes.data_as(C.POINTER(C.c_float))
        p.ls = ls
        p.beta_minus, p.beta_plus = cfg["beta"]
        p.k_minus, p.k_plus = cfg["k"]
        p.source = cfg["source"]
        q = np.ascontiguousarray(np.asarray(cfg["charges_q"], np.float32).reshape(-1))
        qc = np.ascontiguousarray(np.asarray(cfg["charges_c"], np.float32).reshape(-1))
        self._keep += [q, qc]
        p.n_charges = len(q)
        p.q = q.ctypes.data_as(C.POINTER(C.c_float))
        p.charge_centers = qc.ctypes.data_as(C.POINTER(C.c_float))
        p.charge_sigma = cfg["charge_sigma"]
        p.lambda_b = cfg["lambda_b"]
        p.mu_kind = int(cfg.get("mu_kind", 0))
        if cfg.get("mu_lin") is not None:
            ml = np.asarray(cfg["mu_lin"], np.float32).reshape(2, 4)
            for s_ in range(2):
                for c_ in range(4):
                    p.mu_lin[s_][c_] = float(ml[s_, c_])
        sizes = np.ascontiguousarray(np.asarray(cfg["sizes"], np.int32))
        self._keep.append(sizes)
        a = nbm_arch()
        a.n_layers = len(sizes)
        a.sizes = sizes.ctypes.data_as(C.POINTER(C.c_int))
        a.act = cfg["act"]
        a.prec = cfg["prec"]
        a.n_nets = cfg["n_nets"]
        a.stencil = int(cfg.get("stencil", STENCIL_DIRECT))
        self.problem, self.arch = p, a


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _check(h, rc):
    if rc != NBM_OK:
        msg = lib().nbm_last_error(h)
        raise NbmError(rc, msg.decode() if msg else "")


# ---- the C-ABI calls with the same names ----

def nbm_arch_param_count(desc: Descriptors) -> int:
    return int(lib().nbm_arch_param_count(C.byref(desc.arch)))


def nbm_check(desc: Descriptors) -> int:
    return int(lib().nbm_check(C.byref(desc.problem), C.byref(desc.arch)))


def nbm_create(desc: Descriptors, device: int, max_points: int):
    h = C.c_void_p()
    rc = lib().nbm_create(C.byref(desc.problem), C.byref(desc.arch), device, max_points, C.byref(h))
    _check(None, rc)
    return h


def nbm_destroy(h) -> None:
    lib().nbm_destroy(h)


def nbm_param_count(h) -> int:
    return int(lib().nbm_param_count(h))


def nbm_status(h, stream=None) -> int:
    return int(lib().nbm_status(h, _stream(stream)))


def nbm_init_params(h, seed: int, theta, stream=None) -> None:
    _check(h, lib().nbm_init_params(h, seed, _ptr(theta), _stream(stream)))


def nbm_sample(h, seed: int, step: int, kind: int, first_index: int, n: int, h_cell: float, pts,
               stream=None) -> None:
    _check(h, lib().nbm_sample(h, seed, step, kind, first_index, n, h_cell, _ptr(pts), _stream(stream)))


def nbm_loss_grad(h, theta, pts, n: int, bpts, nb: int, h_cell: float, n_global: int, nb_global: int,
                  terms: int, loss, grad, stream=None) -> None:
    _check(h, lib().nbm_loss_grad(h, _ptr(theta), _ptr(pts), n, _ptr(bpts), nb, h_cell, n_global,
                                  nb_global, terms, _ptr(loss), _ptr(grad), _stream(stream)))


def nbm_loss_grad_ml(h, theta, pts, n: int, bpts, nb: int, h0: float, n_levels: int, level_weights,
                     n_global: int, nb_global: int, terms: int, loss, grad, stream=None) -> None:
    w = None
    if level_weights is not None:
        w = (C.c_float * n_levels)(*[float(x) for x in level_weights])
    _check(h, lib().nbm_loss_grad_ml(h, _ptr(theta), _ptr(pts), n, _ptr(bpts), nb, h0, n_levels,
                                     C.cast(w, C.c_void_p) if w is not None else None, n_global, nb_global,
                                     terms, _ptr(loss), _ptr(grad), _stream(stream)))


def nbm_classify(h, pts, n: int, h_cell: float, mask, cls, stream=None) -> None:
    _check(h, lib().nbm_classify(h, _ptr(pts), n, h_cell, _ptr(mask), _ptr(cls), _stream(stream)))


def nbm_eval(h, theta, pts, n: int, u, stream=None) -> None:
    _check(h, lib().nbm_eval(h, _ptr(theta), _ptr(pts), n, _ptr(u), _stream(stream)))


def nbm_error_norms(h, theta, M: int, out, stream=None) -> None:
    _check(h, lib().nbm_error_norms(h, _ptr(theta), int(M), _ptr(out), _stream(stream)))


def nbm_adam_step(h, theta, m, v, grad, t: int, lr: float, b1: float, b2: float, eps: float,
                  stream=None) -> None:
    _check(h, lib().nbm_adam_step(h, _ptr(theta), _ptr(m), _ptr(v), _ptr(grad), t, lr, b1, b2, eps,
                                  _stream(stream)))


def nbm_sample_at(h, seed: int, step_dev, kind: int, first_index: int, n: int, h_cell: float, pts,
                  stream=None) -> None:
    _check(h, lib().nbm_sample_at(h, seed, _ptr(step_dev), kind, first_index, n, h_cell, _ptr(pts),
                                  _stream(stream)))


def nbm_adam_step_at(h, theta, m, v, grad, t_dev, lr: float, b1: float, b2: float, eps: float,
                     stream=None) -> None:
    _check(h, lib().nbm_adam_step_at(h, _ptr(theta), _ptr(m), _ptr(v), _ptr(grad), _ptr(t_dev), lr, b1, b2,
                                     eps, _stream(stream)))


def nbm_timing_enable(h, enable: bool) -> None:
    _check(h, lib().nbm_timing_enable(h, int(enable)))


def nbm_timing_read(h):
    a, b, n = C.c_double(), C.c_double(), C.c_int64()
    _check(h, lib().nbm_timing_read(h, C.byref(a), C.byref(b), C.byref(n)))
    return a.value, b.value, n.value


def nbm_last_launch_count(h) -> int:
    return int(lib().nbm_last_launch_count(h))


class Solver:
    """One handle plus the caller-owned parameter/optimizer buffers (torch tensors).

    Everything runs on `device` through the C ABI; this class only owns buffers."""

    def __init__(self, cfg: dict, device: int = 0, max_points: int | None = None):
        import torch
        self.cfg = cfg
        self.desc = Descriptors(cfg)
        self.device = torch.device("cuda", device)
        cap = max_points or max(cfg["N"], cfg["Nb"])
        self.h = nbm_create(self.desc, device, cap)
        self.P = nbm_param_count(self.h)
        # [grad, loss] contiguous: one all-reduce per step
        self.gbuf = torch.zeros(self.P + 1, dtype=torch.float32, device=self.device)
        self.grad, self.loss = self.gbuf[: self.P], self.gbuf[self.P:]
        self.theta = torch.zeros(self.P, dtype=torch.float32, device=self.device)
        self.m = torch.zeros_like(self.theta)
        self.v = torch.zeros_like(self.theta)
        self.t = 0
        # device step counter for graph-captured steps (nbm_sample_at / nbm_adam_step_at)
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=self.device)

    def close(self):
        if self.h is not None:
            nbm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def h_cell(self) -> float:
        return self.cfg["H"] / float(1 << 24)

    def init_params(self, seed: int = 0):
        nbm_init_params(self.h, seed, self.theta)

    def sample(self, kind, seed, step, first, n, out):
        nbm_sample(self.h, seed, step, kind, first, n, self.h_cell, out)

    def loss_grad(self, pts, bpts, n_global=None, nb_global=None, terms=TERM_ALL, theta=None, levels=1,
                  level_weights=None):
        n = 0 if pts is None else pts.shape[0]
        nb = 0 if bpts is None else bpts.shape[0]
        th = self.theta if theta is None else theta
        ng = n if n_global is None else n_global
        nbg = nb if nb_global is None else nb_global
        if levels == 1 and level_weights is None:
            nbm_loss_grad(self.h, th, pts, n, bpts, nb, self.h_cell, ng, nbg, terms, self.loss, self.grad)
        else:
            nbm_loss_grad_ml(self.h, th, pts, n, bpts, nb, self.h_cell, levels, level_weights, ng, nbg, terms,
                             self.loss, self.grad)
        return self.loss, self.grad

    def adam_step(self, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        self.t += 1
        nbm_adam_step(self.h, self.theta, self.m, self.v, self.grad, self.t, lr, b1, b2, eps)

    def sample_at(self, kind, seed, first, n, out):
        """sample with the step word read from self.t_dev (graph-capturable)"""
        nbm_sample_at(self.h, seed, self.t_dev, kind, first, n, self.h_cell, out)

    def adam_step_at(self, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        """Adam with t = t_dev + 1 read and t_dev incremented on the device (graph-capturable)"""
        nbm_adam_step_at(self.h, self.theta, self.m, self.v, self.grad, self.t_dev, lr, b1, b2, eps)

    def capture_step(self, pts, bpts, first=0, bfirst=0, n_global=None, nb_global=None, lr=1e-3, seed=0,
                     allreduce=None, levels=1):
        """Capture one training step [sample interior, sample boundary, loss_grad,
        (allreduce), Adam] as CUDA graphs on the device counter self.t_dev.  Returns a
        callable that replays one step.  With `allreduce` (a callable on the [grad, loss]
        buffer) the step is captured as two graphs around an eagerly launched collective."""
        import torch
        n, nb = pts.shape[0], bpts.shape[0]

        def pre():
            self.sample_at(POINTS_INTERIOR, seed, first, n, pts)
            self.sample_at(POINTS_BOUNDARY, seed, bfirst, nb, bpts)
            self.loss_grad(pts, bpts, n_global=n_global, nb_global=nb_global, levels=levels)

        def post():
            self.adam_step_at(lr=lr)

        t0 = self.t_dev.clone()
        saved = [x.clone() for x in (self.theta, self.m, self.v)]
        side = torch.cuda.Stream(self.device)   # warm up the calls outside capture (lazy init)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            pre()
            post()
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        self.t_dev.copy_(t0)                    # the warm-up step leaves no trace
        for x, y in zip((self.theta, self.m, self.v), saved):
            x.copy_(y)
        if allreduce is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                pre()
                post()
            return g.replay
        g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            pre()
        with torch.cuda.graph(g2):
            post()

        def replay():
            g1.replay()
            allreduce(self.gbuf)
            g2.replay()
        return replay

    def eval(self, pts, out=None):
        import torch
        if out is None:
            out = torch.empty(pts.shape[0], dtype=torch.float32, device=self.device)
        nbm_eval(self.h, self.theta, pts, pts.shape[0], out)
        return out

    def error_norms(self, M: int, theta=None):
        """(rmse, linf) against the closed-form solution on the (M+1)^3 nodal grid."""
        import torch
        out = torch.empty(2, dtype=torch.float64, device=self.device)
        nbm_error_norms(self.h, self.theta if theta is None else theta, M, out)
        r = out.cpu()
        return float(r[0]), float(r[1])

    def status(self) -> int:
        return nbm_status(self.h)
