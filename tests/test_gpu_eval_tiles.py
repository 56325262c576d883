"""nbm_eval with many tiles per CTA on every kernel family (round 2).  The parity tests' eval
cases use a few thousand points, i.e. at most one tile per CTA, which cannot catch a forward-only
pass that leaves a CTA's streamed-weight stage (or ring) on the last layer after its first tile
(the SiLU kernel had exactly that bug, test_gpu_tc.test_tc_eval_silu_many_tiles).  Here 2^15
interior + 2^10 boundary points give several tiles per CTA everywhere.  Bars, point by point
and relative to max |u|: fp32 paths 1e-5 against the fp64 oracle; bf16 paths 2e-2 against the
oracle's bf16 emulation (the per-point tail of tanh.approx and accumulation order reaches
≈ 7e-3 over 33k points; a tile evaluated with the wrong weights is off by O(1)) and 5e-2
against fp64 (the max over 33k points of the bf16 rounding error; 3000-point tests hold 2e-2)."""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


CASES = [
    ("c4", 256, None, 5e-2),                   # K3w: CTA pairs, weight ring
    ("c5", 128, None, 5e-2),                   # K3t W = 128 (resident weights)
    ("c5", 64, None, 5e-2),                    # K3t W = 64, two CTAs per SM
    ("c5", 128, inputs.PREC_FP32, 1e-5),       # K3fw W = 128, streamed fp32 weights
    ("c5", 256, inputs.PREC_FP32, 1e-5),       # K3fw W = 256
    ("c2", 64, inputs.PREC_FP32X, 1e-5),       # FP32X split planes (resident weights)
    ("c5", 64, inputs.PREC_FP32X, 1e-5),       # FP32X at four hidden layers (streamed planes)
    ("c2", 64, inputs.PREC_FP32, 1e-5),        # K3f
]


@pytest.mark.parametrize("name,w,prec,tol", CASES)
def test_eval_many_tiles_per_cta(orc, name, w, prec, tol):
    cfg = inputs.config(name, width=w, prec=prec) if name in ("c4", "c5") else inputs.config(name, prec=prec)
    n, nb = 1 << 15, 1 << 10
    s = nbm.Solver(cfg, 0, max_points=n + nb)
    pb, ar = orc.from_config(cfg)
    th = orc.init_params(ar, 3)
    pts = np.concatenate([orc.sample(0, 12, 0, 0, n, cfg["H"]), orc.sample(1, 12, 0, 0, nb, cfg["H"])])
    s.theta.copy_(_dev(th))
    u = s.eval(_dev(pts)).double().cpu().numpy()
    want = orc.evaluate(pb, ar, th, pts)
    err = np.abs(u - want).max() / np.abs(want).max()
    assert err <= tol, err
    if cfg["prec"] == inputs.PREC_BF16:
        emu = orc.evaluate(pb, ar, th, pts, mode=orc.MODE_BF16)
        e_emu = np.abs(u - emu).max() / np.abs(emu).max()
        assert e_emu <= 2e-2, e_emu
    assert s.status() == 0
    s.close()


def test_eval_full_size_config4_sampled(orc):
    """nbm_eval at config 4's full size (2^22 interior points, the bench's --eval launch) on
    K3w, checked on 3000 sampled points one by one (bars as above)."""
    cfg = inputs.config("c4")
    n = 1 << 22
    s = nbm.Solver(cfg, 0, max_points=n)
    s.init_params(5)
    pb, ar = orc.from_config(cfg)
    th = s.theta.double().cpu().numpy()
    pts = torch.empty(n, 3, device="cuda")
    s.sample(nbm.POINTS_INTERIOR, 7, 3, 0, n, pts)
    u = s.eval(pts).double().cpu().numpy()
    idx = np.random.default_rng(0).choice(n, 3000, replace=False)
    idx = np.concatenate([idx, [0, n - 1]])
    sp = pts.cpu().numpy()[idx]
    assert np.array_equal(sp, orc.sample(0, 7, 3, 0, n, cfg["H"])[idx])   # the sampled inputs
    want = orc.evaluate(pb, ar, th, sp)
    assert np.abs(u[idx] - want).max() / np.abs(want).max() <= 5e-2
    emu = orc.evaluate(pb, ar, th, sp, mode=orc.MODE_BF16)
    assert np.abs(u[idx] - emu).max() / np.abs(emu).max() <= 2e-2
    assert np.all(np.isfinite(u))
    assert s.status() == 0
    s.close()
