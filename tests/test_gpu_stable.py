"""GPU parity of the stable stencil form (NBM_STENCIL_STABLE, G27)
against the fp64 oracle's plain definition (the same L and dL/dtheta; only the evaluation
order differs).

Bar: the bf16 bar of the north_star (2e-2: loss relative, gradient relative L2) on the
totals and on each uncrossed term, relaxed only to 4 x the stable form's OWN bf16 floor
(its emulation, oracle/stable_stencil.py: ~0.1-4 % where the three second differences of a
random network cancel in the Laplacian) instead of the direct path's floor (~1e4 x the
signal at h = 2/1023); the GPU result also agrees with that emulation to 3e-3, and is 10x
closer to fp64 than the direct bf16 evaluation.  The crossed and boundary rows are
evaluated directly and keep the direct path's per-term rule."""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm

from _bars import floor_tol

pytestmark = pytest.mark.gpu

TOL = 2e-2
EMU_TOL = 3e-3   # vs the bf16 emulation of the form: accumulation order and MUFU only
TERMS = [nbm.TERM_UNX_MINUS, nbm.TERM_UNX_PLUS, nbm.TERM_CROSSED, nbm.TERM_BOUNDARY]


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _run(s, th, p, b, terms=nbm.TERM_ALL):
    loss, grad = s.loss_grad(p, b, terms=terms, theta=th)
    torch.cuda.synchronize()
    return float(loss.item()), grad.double().cpu().numpy().copy()


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def _stable_emulation(orc, cfg, pb, ar, th, pts, side):
    """(loss, grad) of one uncrossed term through the stable form with the CUDA path's bf16
    rounding points (oracle/stable_stencil.py); rhs b/d recovered from oracle.c's fp64
    residuals.  Its deviation from fp64 is the form's own noise floor (SURVEY 8c rule 2)."""
    from oracle import stable_stencil as st
    h = cfg["h"]
    _, cls = orc.classify(pb, pts, h)
    sel = pts[cls == side]
    P = ar.P // cfg["n_nets"]
    net = side if cfg["n_nets"] == 2 else 0
    thn = np.asarray(th, np.float64)[net * P:(net + 1) * P]
    k, beta = float(np.float32(cfg["k"][side])), float(np.float32(cfg["beta"][side]))
    cc, ch = st.residual_coefficients(k, beta, h)
    r_plain, _ = orc.residuals(pb, ar, th, sel, np.zeros((0, 3), np.float32), h)
    u, _, DU, _ = st.forward(thn, cfg["sizes"], sel.astype(np.float64), h)
    rhs = cc * u + ch * DU.sum(axis=1) - r_plain
    L, _, g = st.loss_grad_unx(thn, cfg["sizes"], sel.astype(np.float64), h, k, beta, rhs, n_glob=len(pts),
                               rnd=st.bf16)
    full = np.zeros(ar.P)
    full[net * P:(net + 1) * P] = g
    return L, full


@pytest.mark.parametrize("w,nh,k,n", [(128, 4, 0.0, 1 << 13), (128, 3, 0.0, (1 << 13) + 5), (128, 2, 0.0, 4099),
                                      (64, 4, 0.0, 1 << 13), (64, 2, 0.0, 3001), (64, 3, 2.5, 1 << 13),
                                      (256, 4, 0.0, 1 << 13), (256, 2, 1.5, 5003), (256, 3, 0.0, 77)])
def test_stable_parity(orc, w, nh, k, n):
    cfg = inputs.config("c5", width=w)
    cfg.update(sizes=[3] + [w] * nh + [1], k=(k, 2 * k), stencil=inputs.STENCIL_STABLE)
    direct = dict(cfg, stencil=inputs.STENCIL_DIRECT)
    nb = 1 << 10
    s = nbm.Solver(cfg, 0, max_points=max(n, nb))
    sd = nbm.Solver(direct, 0, max_points=max(n, nb))
    pb, ar = orc.from_config(cfg)
    pts = orc.sample(0, 5, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 5, 0, 0, nb, cfg["H"])
    th = orc.init_params(ar, 0)
    L, lt, g, gt = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True)
    _, lte, _, gte = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True, mode=orc.MODE_BF16)
    dth, dp, db = _dev(th), _dev(pts), _dev(bpts)
    gl, gg = _run(s, dth, dp, db)
    assert abs(gl - L) <= TOL * L, (gl, L)
    assert _rel(gg, g) <= TOL
    gl2, gg2 = _run(s, dth, dp, db)
    if w < 256:   # K3w flushes dW through L2 reductions: deterministic within tolerance only (G21)
        assert gl2 == gl and np.array_equal(gg2, gg)
    else:
        assert abs(gl2 - gl) <= 1e-6 * gl and _rel(gg2, gg) <= 1e-5
    for kk, term in enumerate(TERMS):
        tl, tg = _run(s, dth, dp, db, terms=term)
        if lt[kk] == 0.0:
            assert tl == 0.0
            continue
        if kk < 2:   # uncrossed: the bar up to the stable form's own bf16 floor, and far below
            # the direct evaluation's error
            Le, ge = _stable_emulation(orc, cfg, pb, ar, th, pts, kk)
            ltol = floor_tol(TOL, abs(Le - lt[kk]) / lt[kk])
            gtol = floor_tol(TOL, _rel(ge, gt[kk]))
            if ltol is not None:   # else: the form's own bf16 floor exceeds 0.1 / 4 on this draw
                assert abs(tl - lt[kk]) <= ltol * lt[kk], (kk, tl, lt[kk], ltol)
            if gtol is not None:
                assert _rel(tg, gt[kk]) <= gtol, (kk, _rel(tg, gt[kk]), gtol)
            assert abs(tl - Le) <= EMU_TOL * Le and _rel(tg, ge) <= EMU_TOL, (kk, tl, Le, _rel(tg, ge))
            dl, dg = _run(sd, dth, dp, db, terms=term)
            assert _rel(tg, gt[kk]) < 0.1 * _rel(dg, gt[kk]), (kk, _rel(tg, gt[kk]), _rel(dg, gt[kk]))
        else:        # crossed / boundary rows: evaluated directly, the direct path's rule
            ltol = floor_tol(TOL, abs(lte[kk] - lt[kk]) / lt[kk])
            gtol = floor_tol(TOL, _rel(gte[kk], gt[kk]))
            assert ltol is not None and gtol is not None
            assert abs(tl - lt[kk]) <= ltol * lt[kk], (kk, tl, lt[kk], ltol)
            assert _rel(tg, gt[kk]) <= gtol, (kk, gtol)
    s.close()
    sd.close()


def test_stable_multiresolution(orc):
    """Three implicit levels h0 / 2^l at h0 = 2/1023 through the stable form."""
    cfg = inputs.config("c5", width=64)
    cfg.update(sizes=[3, 64, 64, 64, 1], stencil=inputs.STENCIL_STABLE)
    assert cfg["H"] % 4 == 0
    n, nb = 4096, 512
    s = nbm.Solver(cfg, 0, max_points=n)
    pb, ar = orc.from_config(cfg)
    pts = orc.sample(0, 9, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 9, 0, 0, nb, cfg["H"])
    th = orc.init_params(ar, 2)
    wts = [1.0, 0.5, 0.25]
    L, g = orc.loss_grad_ml(pb, ar, th, pts, bpts, cfg["h"], 3, wts)
    loss, grad = s.loss_grad(_dev(pts), _dev(bpts), theta=_dev(th), levels=3, level_weights=wts)
    torch.cuda.synchronize()
    assert abs(float(loss.item()) - L) <= TOL * L
    assert _rel(grad.double().cpu().numpy(), g) <= TOL
    s.close()


def test_stable_unsupported_rejected():
    cfg = dict(inputs.config("c3"), stencil=inputs.STENCIL_STABLE)   # SiLU
    with pytest.raises(Exception):
        nbm.Solver(cfg, 0, max_points=16)


def test_stable_graph_replay_matches_eager_steps():
    """The stable form inside the captured CUDA-graph training step (device step counter):
    bitwise equal to the host-counter calls for 3 steps (K3t is deterministic)."""
    cfg = inputs.config("c5", width=64)
    cfg.update(sizes=[3, 64, 64, 64, 1], stencil=inputs.STENCIL_STABLE, N=1 << 14, Nb=1 << 11)
    N, Nb = cfg["N"], cfg["Nb"]
    a = nbm.Solver(cfg, 0, max_points=N)
    b = nbm.Solver(cfg, 0, max_points=N)
    a.init_params(0)
    b.init_params(0)
    pa, ba = torch.empty(N, 3, device="cuda"), torch.empty(Nb, 3, device="cuda")
    pb_, bb = torch.empty(N, 3, device="cuda"), torch.empty(Nb, 3, device="cuda")
    step = b.capture_step(pb_, bb, lr=1e-3, levels=2)
    for k in range(3):
        a.sample(nbm.POINTS_INTERIOR, 0, k, 0, N, pa)
        a.sample(nbm.POINTS_BOUNDARY, 0, k, 0, Nb, ba)
        a.loss_grad(pa, ba, levels=2)
        a.adam_step(lr=1e-3)
        step()
        torch.cuda.synchronize()
        assert torch.equal(a.gbuf, b.gbuf)
        assert torch.equal(a.theta, b.theta)
    a.close()
    b.close()


@pytest.mark.parametrize("name,w", [("c5", 128), ("c4", 256)])
def test_stable_full_size_shard_invariance(name, w):
    """At the bench's full size (2^22 + 2^19 points, the timed launch configuration): the
    stable-form total equals the sum of 4 shard calls with the global normalisation (fp32
    reduction bars), and every term is finite.  Per-point parity is size-independent and is
    checked above; this covers the tile indexing and reductions at full size."""
    cfg = inputs.config(name, width=w)
    cfg["stencil"] = inputs.STENCIL_STABLE
    N, Nb = cfg["N"], cfg["Nb"]
    s = nbm.Solver(cfg, 0)
    s.init_params(0)
    pts = torch.empty(N, 3, device="cuda")
    bpts = torch.empty(Nb, 3, device="cuda")
    s.sample(0, 0, 0, 0, N, pts)
    s.sample(1, 0, 0, 0, Nb, bpts)
    lt, gt = _run(s, s.theta, pts, bpts)
    assert np.isfinite(lt) and np.all(np.isfinite(gt)) and lt > 0
    for term in TERMS[:2]:
        tl, _ = _run(s, s.theta, pts, bpts, terms=term)
        assert np.isfinite(tl) and tl > 0
    acc_l, acc_g = 0.0, np.zeros_like(gt)
    for r in range(4):
        lo, hi, blo, bhi = r * N // 4, (r + 1) * N // 4, r * Nb // 4, (r + 1) * Nb // 4
        loss, grad = s.loss_grad(pts[lo:hi], bpts[blo:bhi], n_global=N, nb_global=Nb, theta=s.theta)
        torch.cuda.synchronize()
        acc_l += float(loss.item())
        acc_g += grad.double().cpu().numpy()
    assert abs(acc_l - lt) <= 1e-5 * lt
    # the shards move tiles between CTAs; K3t sums each CTA's dW_l in TMEM (tensor-core fp32
    # accumulation), where the difference rows' O(h^-1) / O(h^-2) gradients times O(h) / O(h^2)
    # activations partly cancel: measured 5e-4 of the gradient norm at c5-w128 (K3w's L2
    # reductions: < 1e-4), far inside the 2e-2 bf16 bar
    assert np.linalg.norm(acc_g - gt) <= (2e-3 if w < 256 else 1e-4) * np.linalg.norm(gt)
    assert s.status() == 0
    s.close()


@pytest.mark.parametrize("name,sizes,k,n,hq", [("c2", None, 0.0, 1 << 14, None), ("c2", None, 2.0, 5003, None),
                                                ("c1", None, 0.0, 4096, None), ("c5", [3, 64, 64, 64, 64, 1], 0.0, 1 << 13, None),
                                                ("c5", [3, 20, 20, 1], 0.0, 3001, None),
                                                ("c5", [3, 128, 128, 128, 1], 0.0, 4099, None),
                                                ("c5", [3, 256, 256, 1], 1.5, 2048, None),
                                                ("c2", [3, 16, 1], 0.0, 2000, None),
                                                ("c2", [3, 24, 24, 24, 24, 24, 1], 0.0, 2000, None)])
def test_stable_fp32_strict_parity(orc, name, sizes, k, n, hq):
    """fp32 stable form (K3f<STAB>): every term, the uncrossed ones included, at the STRICT fp32
    bars of the north_star (1e-5 loss, 1e-4 gradient; no noise-floor relaxation), where the
    direct fp32 evaluation needs it (c5 at h = 2/1023: the oracle's fp32 emulation of the
    direct form is off by up to 5x on the Omega- term)."""
    cfg = inputs.config(name)
    if name == "c5":
        cfg.update(prec=inputs.PREC_FP32)
    if sizes:
        cfg["sizes"] = sizes
    if k:
        cfg["k"] = (k, 2 * k)
    cfg["stencil"] = inputs.STENCIL_STABLE
    nb = max(64, n // 8)
    s = nbm.Solver(cfg, 0, max_points=max(n, nb))
    pb, ar = orc.from_config(cfg)
    pts = orc.sample(0, 3, 0, 0, n, cfg["H"])
    bpts = orc.sample(1, 3, 0, 0, nb, cfg["H"])
    th = orc.init_params(ar, 0)
    L, lt, g, gt = orc.loss_grad(pb, ar, th, pts, bpts, cfg["h"], per_term=True)
    dth, dp, db = _dev(th), _dev(pts), _dev(bpts)
    gl, gg = _run(s, dth, dp, db)
    assert abs(gl - L) <= 1e-5 * L, (gl, L)
    assert _rel(gg, g) <= 1e-4
    gl2, gg2 = _run(s, dth, dp, db)
    if cfg["sizes"][1] <= 64:
        assert gl2 == gl and np.array_equal(gg2, gg)
    else:   # K3fw: L2 reductions, deterministic within tolerance (G21)
        assert abs(gl2 - gl) <= 1e-6 * gl and _rel(gg2, gg) <= 1e-6
    for kk, term in enumerate(TERMS):
        tl, tg = _run(s, dth, dp, db, terms=term)
        if lt[kk] == 0.0:
            assert tl == 0.0
            continue
        assert abs(tl - lt[kk]) <= 1e-5 * lt[kk], (kk, tl, lt[kk])
        assert _rel(tg, gt[kk]) <= 1e-4, (kk, _rel(tg, gt[kk]))
    s.close()
