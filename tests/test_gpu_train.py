"""GPU: evaluation-grid error norms through the C ABI against the oracle, and
the training workload on the section 4.1 problem."""
import numpy as np
import pytest
import torch

from paper_2210_14907_b200 import inputs, nbm, train

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


@pytest.mark.parametrize("name,M,cap", [("p41", 16, 1000), ("p41", 33, 1 << 16), ("c2", 20, 3001), ("c1", 8, 64)])
def test_error_norms_parity(orc, name, M, cap):
    """fp32 networks on the GPU vs fp64 in the oracle: the errors agree to the networks'
    fp32 evaluation error; chunks of `cap` points exercise the chunked path."""
    cfg = inputs.config(name)
    s = nbm.Solver(cfg, 0, max_points=cap)
    pb, ar = orc.from_config(cfg)
    th = inputs.random_theta(cfg["sizes"], cfg["n_nets"], 4)
    rmse, linf = s.error_norms(M, theta=_dev(th))
    o_rmse, o_linf = orc.error_norms(pb, ar, th, M)
    assert rmse == pytest.approx(o_rmse, rel=1e-5)
    assert linf == pytest.approx(o_linf, rel=1e-5)
    assert rmse <= linf
    r2 = s.error_norms(M, theta=_dev(th))
    assert r2 == (rmse, linf)                                          # deterministic
    s.close()


def test_error_norms_rejects_sources_without_exact_solution():
    s = nbm.Solver(inputs.config("c3"), 0, max_points=1024)
    with pytest.raises(nbm.NbmError):
        s.error_norms(4)
    with pytest.raises(nbm.NbmError):
        s.error_norms(0)
    s.close()


def test_training_reduces_error_and_is_deterministic():
    """Section 4.1 problem, N = 8, 300 epochs: the nodal-grid RMSE drops well below
    the initial network's and the loss history falls (medians of the first and last
    10 %); two runs with one seed are bitwise identical."""
    cfg = inputs.config("p41")
    r = train.train(cfg, 8, 300, log_every=10)
    assert r["rmse"] < 0.25 * r["rmse_init"]
    assert r["linf"] < r["linf_init"]
    losses = [l for _, l in r["loss_history"]]
    k = max(1, len(losses) // 10)
    assert np.median(losses[-k:]) < np.median(losses[:k])
    r2 = train.train(cfg, 8, 300, log_every=10)
    assert (r2["rmse"], r2["linf"]) == (r["rmse"], r["linf"])


def test_error_norms_on_a_sampled_level_set(orc):
    """The side of each nodal point comes from the sampled (grid) level set: the
    error norms still match the oracle's, which evaluates the same trilinear phi."""
    cfg = inputs.with_grid(inputs.config("c2"), 32)
    s = nbm.Solver(cfg, 0, max_points=2048)
    pb, ar = orc.from_config(cfg)
    th = inputs.random_theta(cfg["sizes"], cfg["n_nets"], 6)
    rmse, linf = s.error_norms(24, theta=_dev(th))
    o_rmse, o_linf = orc.error_norms(pb, ar, th, 24)
    assert rmse == pytest.approx(o_rmse, rel=1e-5)
    assert linf == pytest.approx(o_linf, rel=1e-5)
    s.close()


def test_training_multilevel_and_lr_phases():
    """train() with two implicit levels and an lr schedule of two captured graphs:
    runs, stays finite, lowers the error, and is bitwise repeatable."""
    cfg = inputs.config("p41")
    kw = dict(levels=2, lr_schedule=[(0.5, 2e-3), (0.5, 5e-4)], log_every=50)
    r = train.train(cfg, 8, 200, **kw)
    assert np.isfinite(r["rmse"]) and r["rmse"] < 0.5 * r["rmse_init"]
    r2 = train.train(cfg, 8, 200, **kw)
    assert (r2["rmse"], r2["linf"]) == (r["rmse"], r["linf"])


def test_spec_acceptance_table1_row_n16():
    """SPEC's training acceptance from Table 1 row N = 2^4 (RMSE 7.1e-3,
    L-inf 1.10e-1): the section 4.1 problem, two 5 x 10 sine networks (982 parameters), N = 16,
    10,000 epochs of Adam (lr 1e-3) through the library's CUDA-graph step -> RMSE and L-inf on the
    nodal grid within 3x of the paper's (the tolerance covers the unstated optimiser settings)."""
    cfg = inputs.config("p41")
    r = train.train(cfg, 16, 10000)
    assert 7.1e-3 / 3 <= r["rmse"] <= 3 * 7.1e-3, r["rmse"]
    assert 1.10e-1 / 3 <= r["linf"] <= 3 * 1.10e-1, r["linf"]
