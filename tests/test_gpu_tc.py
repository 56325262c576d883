"""GPU parity of the bf16 tcgen05 path (K3t) against the oracle.

Bar (north_star): the bf16 tensor-core path matches the fp64 oracle to 2e-2 (loss relative,
gradient relative L2) in total, and per term within max(2e-2, 4 x the oracle's own
bf16-emulation deviation from fp64) (SURVEY 8c rule 2: ill-conditioned terms).  A second, tighter check compares against the
oracle's bf16 emulation (same rounding points, G16): only accumulation order and
the hardware tanh differ."""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm

from _bars import floor_tol

pytestmark = pytest.mark.gpu

TOL = 2e-2
EMU_TOL = 3e-3
TERMS = [nbm.TERM_UNX_MINUS, nbm.TERM_UNX_PLUS, nbm.TERM_CROSSED, nbm.TERM_BOUNDARY]


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _run(s, th, p, b, terms=nbm.TERM_ALL):
    loss, grad = s.loss_grad(p, b, terms=terms, theta=th)
    torch.cuda.synchronize()
    return float(loss.item()), grad.double().cpu().numpy().copy()


@pytest.mark.parametrize("name,w,nh", [("c5", 128, 2), ("c5", 128, 3), ("c5", 128, 4), ("c3", 128, 2),
                                        ("c3", 128, 3), ("c3", 128, 4), ("c5", 64, 2), ("c5", 64, 4),
                                        ("c3", 64, 4), ("c4", 256, 2), ("c4", 256, 4)])
def test_tc_parity(orc, name, w, nh):
    """c5: 32-sphere union, tanh (resident weights); c3: star interface, Gaussian charges,
    SiLU (weights streamed by TMA bulk copies, bf16 SiLU' buffers); W = 64 runs two CTAs
    per SM with M = 64 dW / tail MMAs; the W = 128 tanh training pass at 3-4 hidden layers is
    K3h (two 64-row half-tiles in flight), 2 layers K3t; c4 (W = 256) streams weights, parks
    activations and flushes per-tile dW by vector reductions."""
    cfg = inputs.config(name, width=w) if name in ("c4", "c5") else inputs.config(name)
    cfg["sizes"] = [3] + [w] * nh + [1]
    n, nb = 1 << 13, 1 << 10
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    pts = orc.sample(0, 5, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 5, 0, 0, nb, cfg["H"])
    th = orc.init_params(ar, 0)
    L, lt, g, gt = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True)
    Le, lte, ge, gte = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True, mode=orc.MODE_BF16)
    dth, dp, db = _dev(th), _dev(pts), _dev(bpts)
    gl, gg = _run(s, dth, dp, db)
    assert abs(gl - L) <= TOL * L, (gl, L)
    assert np.linalg.norm(gg - g) <= TOL * np.linalg.norm(g)
    assert abs(gl - Le) <= EMU_TOL * Le, (gl, Le)
    assert np.linalg.norm(gg - ge) <= EMU_TOL * np.linalg.norm(ge)
    for k, term in enumerate(TERMS):
        tl, tg = _run(s, dth, dp, db, terms=term)
        if lt[k] == 0.0:
            assert tl == 0.0
            continue
        # noise floor of the bf16 rounding points (SURVEY 8c rule 2): the uncrossed terms, and
        # for config 3 (h = 1/512, beta 2:80) also the crossed term, sit below bf16 resolution
        # at the configs' h; where the floor-derived tolerance would exceed 0.1 the term is not
        # asserted here (test_gpu_r2_parity.test_bf16_coarse_h_per_term resolves it at h = 1/4)
        ltol = floor_tol(TOL, abs(lte[k] - lt[k]) / lt[k])
        gtol = floor_tol(TOL, np.linalg.norm(gte[k] - gt[k]) / np.linalg.norm(gt[k]))
        if ltol is None or gtol is None:
            assert k < 2 or name == "c3", (k, name)   # only the unresolved stencil terms
            continue
        assert abs(tl - lt[k]) <= ltol * lt[k], (k, tl, lt[k], ltol)
        assert np.linalg.norm(tg - gt[k]) <= gtol * np.linalg.norm(gt[k]), (k, gtol)
    s.close()


def test_tc_eval_and_determinism(orc):
    cfg = inputs.config("c5", width=128)
    n = 3000
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    th = orc.init_params(ar, 1)
    pts = orc.sample(0, 6, 0, 0, n, cfg["H"])
    s.theta.copy_(_dev(th))
    u = s.eval(_dev(pts)).double().cpu().numpy()
    want = orc.evaluate(pb, ar, th, pts)
    assert np.abs(u - want).max() <= TOL * np.abs(want).max()        # the bf16 bar (2e-2)
    b = orc.sample(1, 6, 0, 0, 300, cfg["H"])
    l1, g1 = _run(s, s.theta, _dev(pts), _dev(b))
    l2, g2 = _run(s, s.theta, _dev(pts), _dev(b))
    assert l1 == l2 and np.array_equal(g1, g2)
    assert s.status() == 0
    s.close()


def test_tc_eval_silu_many_tiles(orc):
    """nbm_eval on the SiLU network (weights streamed through one shared-memory stage) with
    several 128-row tiles per CTA (2^15 points, 148 CTAs): every tile's forward must start from
    W_2 again (a stage left holding W_NH after the previous tile would go unnoticed with one
    tile per CTA).  The bf16 bar against the fp64 oracle, point by point."""
    cfg = inputs.config("c3")
    n = 1 << 15
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    th = orc.init_params(ar, 2)
    pts = orc.sample(0, 9, 0, 0, n, cfg["H"])
    s.theta.copy_(_dev(th))
    u = s.eval(_dev(pts)).double().cpu().numpy()
    want = orc.evaluate(pb, ar, th, pts)
    assert np.abs(u - want).max() <= TOL * np.abs(want).max()
    assert s.status() == 0
    s.close()


def test_tc_full_size_config4(orc):
    """BASELINE config 4 at its full size (2^22 interior + 2^19 boundary points per step) in
    the bench's launch configuration (K3w, CTA pairs).  At this size the fp64 oracle can
    evaluate the crossed term: its points (~0.26 %) are classified by the oracle and passed
    to it alone with the global normalisation, so the GPU's crossed term over the full batch
    must equal it (2e-2 vs fp64, 3e-3 vs the bf16 emulation).  The total is checked through a
    property that holds at any size: 4-way shard invariance (L2 reductions: deterministic
    within tolerance only, G21)."""
    cfg = inputs.config("c4")
    N, Nb = cfg["N"], cfg["Nb"]
    s = nbm.Solver(cfg, 0)
    pb, ar = orc.from_config(cfg)
    s.init_params(0)
    pts = torch.empty(N, 3, device="cuda")
    bpts = torch.empty(Nb, 3, device="cuda")
    s.sample(0, 0, 0, 0, N, pts)
    s.sample(1, 0, 0, 0, Nb, bpts)
    lx, gx = _run(s, s.theta, pts, bpts, terms=nbm.TERM_CROSSED)
    P = pts.cpu().numpy()
    _, cls = orc.classify(pb, P, cfg["h"])
    X = P[cls == 2]
    assert 5000 < len(X) < 20000
    th = orc.init_params(ar, 0)
    none = np.zeros((0, 3), np.float32)
    L, _, g, _ = orc.loss_grad(pb, ar, th, X, none, cfg["h"], n_glob=N, nb_glob=Nb)
    Le, _, ge, _ = orc.loss_grad(pb, ar, th, X, none, cfg["h"], n_glob=N, nb_glob=Nb, mode=orc.MODE_BF16)
    assert abs(lx - L) <= TOL * L, (lx, L)
    assert np.linalg.norm(gx - g) <= TOL * np.linalg.norm(g)
    assert abs(lx - Le) <= EMU_TOL * Le, (lx, Le)
    assert np.linalg.norm(gx - ge) <= EMU_TOL * np.linalg.norm(ge)
    # total over the full batch vs the sum of 4 shard calls (each rank's contribution)
    lt, gt = _run(s, s.theta, pts, bpts)
    acc_l, acc_g = 0.0, np.zeros_like(gt)
    for r in range(4):
        lo, hi, blo, bhi = r * N // 4, (r + 1) * N // 4, r * Nb // 4, (r + 1) * Nb // 4
        loss, grad = s.loss_grad(pts[lo:hi], bpts[blo:bhi], n_global=N, nb_global=Nb, theta=s.theta)
        torch.cuda.synchronize()
        acc_l += float(loss.item())
        acc_g += grad.double().cpu().numpy()
    assert abs(acc_l - lt) <= 1e-5 * lt
    assert np.linalg.norm(acc_g - gt) <= 1e-4 * np.linalg.norm(gt)
    assert s.status() == 0
    s.close()


@pytest.mark.parametrize("name,w,nh", [("c5", 128, 4), ("c4", 256, 4)])
def test_tc_multiresolution(orc, name, w, nh):
    """Multi-resolution loss on the bf16 paths (K3t per-CTA partials, K3w L2 replicas): two
    levels accumulate in the reduction; 2e-2 vs the fp64 oracle, 3e-3 vs its bf16 emulation."""
    cfg = inputs.config(name, width=w)
    cfg["sizes"] = [3] + [w] * nh + [1]
    n, nb = 1 << 12, 1 << 9
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    pts = orc.sample(0, 9, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 9, 0, 0, nb, cfg["H"])
    th = orc.init_params(ar, 0)
    loss, grad = s.loss_grad(_dev(pts), _dev(bpts), theta=_dev(th), levels=2)
    torch.cuda.synchronize()
    gl, gg = float(loss.item()), grad.double().cpu().numpy()
    L, g = orc.loss_grad_ml(pb, ar, th, pts, bpts, cfg["h"], 2)
    Le, ge = orc.loss_grad_ml(pb, ar, th, pts, bpts, cfg["h"], 2, mode=orc.MODE_BF16)
    assert abs(gl - L) <= TOL * L, (gl, L)
    assert np.linalg.norm(gg - g) <= TOL * np.linalg.norm(g)
    assert abs(gl - Le) <= EMU_TOL * Le, (gl, Le)
    assert np.linalg.norm(gg - ge) <= EMU_TOL * np.linalg.norm(ge)
    s.close()


def test_tc_grid_levelset_w256(orc):
    """bf16 W = 256 (K3w) on config 4's 32-sphere union sampled on a 128^3 grid."""
    cfg = inputs.with_grid(inputs.config("c4"), 128)
    n, nb = 1 << 12, 1 << 9
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    pts = orc.sample(0, 3, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 3, 0, 0, nb, cfg["H"])
    th = orc.init_params(ar, 0)
    L, _, g, _ = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"])
    Le, _, ge, _ = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], mode=orc.MODE_BF16)
    gl, gg = _run(s, _dev(th), _dev(pts), _dev(bpts))
    assert abs(gl - L) <= TOL * L and np.linalg.norm(gg - g) <= TOL * np.linalg.norm(g)
    assert abs(gl - Le) <= EMU_TOL * Le and np.linalg.norm(gg - ge) <= EMU_TOL * np.linalg.norm(ge)
    s.close()


def test_tc_eval_w256(orc):
    """nbm_eval on the W = 256 pair kernel (K3w forward-only path) at the bf16 bar."""
    cfg = inputs.config("c4")
    n = 3000
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    th = orc.init_params(ar, 2)
    pts = np.concatenate([orc.sample(0, 6, 0, 0, n - 100, cfg["H"]), orc.sample(1, 6, 0, 0, 100, cfg["H"])])
    s.theta.copy_(_dev(th))
    u = s.eval(_dev(pts)).double().cpu().numpy()
    want = orc.evaluate(pb, ar, th, pts)
    assert np.abs(u - want).max() <= TOL * np.abs(want).max()
    assert s.status() == 0
    s.close()


@pytest.mark.parametrize("name,w,nh", [("c5", 64, 4), ("c5", 128, 4), ("c3", 128, 4), ("c4", 256, 4)])
def test_tc_ragged_and_empty(orc, name, w, nh):
    """Edge cases on the tensor-core paths: a single crossed point, single points with one
    boundary point, partial stencil / row tiles (19, 37 points; 129 boundary points: a pair
    tile's odd half at W = 256), boundary-only, interior-only and empty calls.  Totals at the
    bf16 bar against the fp64 oracle (the per-term floor is not stable on a few residuals)."""
    cfg = inputs.config(name, width=w) if name in ("c4", "c5") else inputs.config(name)
    cfg["sizes"] = [3] + [w] * nh + [1]
    pb, ar = orc.from_config(cfg)
    s = nbm.Solver(cfg, 0, max_points=4096)
    th = orc.init_params(ar, 1)
    allp = orc.sample(0, 12, 0, 0, 4096, cfg["H"])
    allb = orc.sample(1, 12, 0, 0, 512, cfg["H"])
    _, cls = orc.classify(pb, allp, cfg["h"])
    crossed = allp[cls == 2]
    cases = [(crossed[:1], allb[:0]), (allp[:1], allb[:1]), (allp[:19], allb[:3]), (allp[:37], allb[:129]),
             (allp[:0], allb[:200]), (allp[:300], allb[:0])]
    for p_, b_ in cases:
        gl, gg = _run(s, _dev(th), _dev(p_) if len(p_) else None, _dev(b_) if len(b_) else None)
        L, _, g, _ = orc.loss_grad(pb, ar, th, p_.reshape(-1, 3), b_.reshape(-1, 3), cfg["h"])
        Le, _, ge, _ = orc.loss_grad(pb, ar, th, p_.reshape(-1, 3), b_.reshape(-1, 3), cfg["h"], mode=orc.MODE_BF16)
        ltol = floor_tol(TOL, abs(Le - L) / L)
        gtol = floor_tol(TOL, np.linalg.norm(ge - g) / np.linalg.norm(g))
        if ltol is None or gtol is None:   # interior-only rows at the config's h: unresolved
            continue
        assert abs(gl - L) <= ltol * L, (len(p_), len(b_), gl, L)
        assert np.linalg.norm(gg - g) <= gtol * np.linalg.norm(g), (len(p_), len(b_))
    gl, gg = _run(s, _dev(th), None, None)
    assert gl == 0.0 and np.all(gg == 0.0)
    assert s.status() == 0
    s.close()


@pytest.mark.parametrize("w", [64, 128, 256])
def test_tc_single_network_no_interface(orc, w):
    """Config 1's problem (no interface: one network, no crossed rows, the sin(3 pi) source) on
    the bf16 kernels (K3t W = 64, K3h W = 128, K3w W = 256): a single network run per CTA, the
    crossed-row passes skipped.  Totals at the bf16 bar against fp64 and 3e-3 against the bf16
    emulation, at h = 1/16 where the uncrossed residual is resolved in bf16."""
    cfg = inputs.config("c1")
    cfg.update(sizes=[3, w, w, w, w, 1], prec=inputs.PREC_BF16, H=inputs.h_lattice(1 / 16))
    n, nb = 1 << 12, 1 << 9
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    th = orc.init_params(ar, 1)
    pts = orc.sample(0, 3, 0, 0, n, cfg["H"])
    b = orc.sample(1, 3, 0, 0, nb, cfg["H"])
    L, _, g, _ = orc.loss_grad(pb, ar, th, pts, b, cfg["H"] / 2**24)
    Le, _, ge, _ = orc.loss_grad(pb, ar, th, pts, b, cfg["H"] / 2**24, mode=orc.MODE_BF16)
    gl, gg = _run(s, _dev(th), _dev(pts), _dev(b))
    assert abs(gl - L) <= TOL * L and np.linalg.norm(gg - g) <= TOL * np.linalg.norm(g)
    assert abs(gl - Le) <= EMU_TOL * Le and np.linalg.norm(gg - ge) <= EMU_TOL * np.linalg.norm(ge)
    assert s.status() == 0
    s.close()
