"""Pins of the oracle's Philox4x32-10 and lattice sampler.

Pinned against: published known-answer vectors, cuRAND's own Philox routine
(compiled for the host), and distributional / structural properties of
S:339-344 UniformRandom sampling."""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2210_14907_b200 import inputs


def test_philox_known_answers(orc):
    kat = json.load(open(os.path.join(GOLDEN, "philox_kat.json")))
    for v in kat["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        out = [int(x, 16) for x in v["out"]]
        assert list(orc.philox(ctr, key)) == out


CURAND_HOST = r"""
#include <cstdio>
#include <cstdint>
#include <vector_types.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = {c0, c1, c2, c3}; uint2 k = {k0, k1};
    uint4 r = curand_Philox4x32_10(c, k);
    std::printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
"""


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_philox_matches_curand_library_routine(orc, tmp_path):
    src = tmp_path / "ph.cu"
    src.write_text(CURAND_HOST)
    exe = tmp_path / "ph"
    subprocess.check_call(["nvcc", "-O1", "-o", str(exe), str(src)])
    rng = np.random.default_rng(5)
    rows = rng.integers(0, 2**32, size=(256, 6), dtype=np.uint64)
    rows[0] = 0
    rows[1] = 2**32 - 1
    inp = "\n".join(" ".join(str(int(v)) for v in r) for r in rows) + "\n"
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout
    ref = np.array([[int(t) for t in line.split()] for line in out.strip().splitlines()])
    for r, want in zip(rows, ref):
        got = orc.philox(r[:4], r[4:])
        assert list(got) == list(want)


@pytest.mark.parametrize("h", [1 / 32, 1 / 128, 2 / 1023])
def test_interior_points_on_lattice_and_in_shrunken_cube(orc, h):
    H = inputs.h_lattice(h)
    hq = H / 2**24
    pts = orc.sample(0, 7, 3, 0, 1 << 14, H)
    ints = pts.astype(np.float64) * 2**24
    assert np.all(ints == np.round(ints))                      # lattice (G9)
    assert np.all(np.abs(pts) <= 1 - hq)                        # S:339 margin
    # all six arms p +- h e_d are exact fp32 values inside the box
    for d in range(3):
        for s in (+1, -1):
            q = pts[:, d].astype(np.float64) + s * hq
            assert np.all(q.astype(np.float32).astype(np.float64) == q)
            assert np.all(np.abs(q) <= 1.0)


def test_uniform_margin_example(orc):
    spec = json.load(open(os.path.join(GOLDEN, "spec_vectors.json")))["training"]["uniform_margin"]
    H = inputs.h_lattice(2.0 / spec["N"])
    pts = orc.sample(0, 0, 0, 0, spec["n"], H)
    assert pts.shape == (spec["n"], 3)
    assert np.all(np.abs(pts) <= spec["bound"])


def test_interior_moments_within_5_sigma(orc):
    H = inputs.h_lattice(1 / 128)
    a = 1 - H / 2**24
    n = 1 << 16
    pts = orc.sample(0, 123, 0, 0, n, H).astype(np.float64)
    var = a * a / 3.0
    for d in range(3):
        assert abs(pts[:, d].mean()) < 5 * np.sqrt(var / n)
        # Var of x^2 for U[-a,a] is 4a^4/45
        assert abs((pts[:, d] ** 2).mean() - var) < 5 * np.sqrt(4 * a**4 / 45 / n)
    # independence of axes: correlation coefficients small
    c = np.corrcoef(pts.T)
    assert np.all(np.abs(c[np.triu_indices(3, 1)]) < 5 / np.sqrt(n))


def test_boundary_points_on_faces(orc):
    n = 60000
    b = orc.sample(1, 9, 0, 0, n, inputs.h_lattice(1 / 32)).astype(np.float64)
    on_face = np.abs(b) == 1.0
    assert np.all(on_face.sum(1) >= 1)
    ints = b * 2**24
    assert np.all(ints == np.round(ints))
    assert np.all(np.abs(b) <= 1.0)
    # face frequencies ~ 1/6 (chi-square with 5 dof, 99.99% quantile ~ 25.7)
    face = np.argmax(on_face, axis=1) * 2 + (np.take_along_axis(b, np.argmax(on_face, 1)[:, None], 1)[:, 0] < 0)
    cnt = np.bincount(face, minlength=6)
    chi2 = ((cnt - n / 6) ** 2 / (n / 6)).sum()
    assert chi2 < 25.7
    # tangential coordinates ~ U[-1,1]
    tang = b[~on_face]
    assert abs(tang.mean()) < 5 * np.sqrt(1 / 3 / len(tang))


def test_shard_and_step_structure(orc):
    H = inputs.h_lattice(1 / 128)
    full = orc.sample(0, 42, 5, 0, 1000, H)
    parts = np.concatenate([orc.sample(0, 42, 5, 0, 300, H), orc.sample(0, 42, 5, 300, 700, H)])
    assert np.array_equal(full, parts)                 # shard invariance
    assert np.array_equal(full, orc.sample(0, 42, 5, 0, 1000, H))   # determinism
    assert not np.array_equal(full, orc.sample(0, 42, 6, 0, 1000, H))  # resampled per step
    assert not np.array_equal(full, orc.sample(0, 43, 5, 0, 1000, H))  # seed matters
