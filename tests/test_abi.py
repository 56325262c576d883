"""The C-ABI library loads and exports every symbol include/nbm.h declares; the host-only
helpers validate descriptors (no GPU needed)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT
from paper_2210_14907_b200 import inputs, nbm


@pytest.fixture(scope="module")
def lib():
    from paper_2210_14907_b200 import build as b
    b.build()
    return nbm.lib()


def _declared():
    hdr = open(os.path.join(ROOT, "include", "nbm.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(nbm_[a-z_]+)\s*\(", hdr)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert "nbm_loss_grad" in names and "nbm_create" in names and len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_version(lib):
    assert b"sm_100a" in lib.nbm_version()


def test_host_param_count_and_check(lib):
    cfg = inputs.config("c2")
    d = nbm.Descriptors(cfg)
    assert nbm.nbm_arch_param_count(d) == inputs.param_count(cfg["sizes"], 2) == 17282
    assert nbm.nbm_check(d) == 0
    bad = dict(cfg, beta=(0.0, 10.0))
    assert nbm.nbm_check(nbm.Descriptors(bad)) == 2          # NBM_E_INVALID_PROBLEM
    bad = dict(cfg, sizes=[4, 64, 1])
    assert nbm.nbm_check(nbm.Descriptors(bad)) == 1          # NBM_E_INVALID_ARCH
    bad = dict(cfg, box=(-1.0, 2.0))
    assert nbm.nbm_check(nbm.Descriptors(bad)) == 2
    c1 = inputs.config("c1")
    assert nbm.nbm_arch_param_count(nbm.Descriptors(c1)) == 1217


def test_all_configs_are_valid_descriptors(lib):
    for name in ("c1", "c2"):
        assert nbm.nbm_check(nbm.Descriptors(inputs.config(name))) == 0


def test_stable_stencil_descriptor_rules(lib):
    """NBM_STENCIL_STABLE (G27) needs a bf16 tanh tensor-core kernel (W in {64, 128, 256})."""
    S = inputs.STENCIL_STABLE
    ok = dict(inputs.config("c5", width=128), stencil=S)
    assert nbm.nbm_check(nbm.Descriptors(ok)) == 0
    assert nbm.nbm_check(nbm.Descriptors(dict(inputs.config("c5", width=64), stencil=S))) == 0
    assert nbm.nbm_check(nbm.Descriptors(dict(inputs.config("c4"), stencil=S))) == 0
    assert nbm.nbm_check(nbm.Descriptors(dict(inputs.config("c2"), stencil=S))) == 0   # fp32 W <= 64
    assert nbm.nbm_check(nbm.Descriptors(dict(inputs.config("c5", width=128, prec=inputs.PREC_FP32), stencil=S))) == 0
    for bad in (dict(inputs.config("c2"), stencil=S, prec=inputs.PREC_FP32X),           # fp32x
                dict(inputs.config("c3"), stencil=S),                     # SiLU
                dict(inputs.config("c5", width=128), stencil=2)):         # unknown mode
        assert nbm.nbm_check(nbm.Descriptors(bad)) == 1
