"""Shared tolerance logic of the parity tests (no method arithmetic).

SURVEY 8c rule 2: an ill-conditioned term is compared at max(bar, 4 x the oracle's own
emulation deviation from fp64) -- the noise floor of any correct implementation at that
precision.  A floor-derived tolerance above CAP (0.1) would make the assertion unable to
fail, so such a term is not asserted there: `floor_tol` returns None and the caller records
it as unresolved at that h (the coarse-h tests, where every floor is below the cap, cover the
same kernels' stencil epilogues with the bar binding)."""
import numpy as np

CAP = 0.1


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


def floor_tol(bar, floor_dev, factor=4.0):
    t = max(bar, factor * floor_dev)
    return t if t <= CAP else None


def param_blocks(sizes, n_nets):
    """(name, lo, hi) of every parameter block W_l, b_l per network (G17 layout)."""
    out, off = [], 0
    for net in range(n_nets):
        for l in range(1, len(sizes)):
            fi, fo = sizes[l - 1], sizes[l]
            out.append((f"net{net}.W{l}", off, off + fi * fo))
            off += fi * fo
            out.append((f"net{net}.b{l}", off, off + fo))
            off += fo
    return out


def check_blocks(got, want, emu, sizes, n_nets, bar, factor=4.0):
    """Per-block relative gradient error: each W_l / b_l of each network within
    max(bar, factor x the emulation's deviation of that block) (capped, see floor_tol).
    Returns the number of blocks asserted."""
    n = 0
    for name, lo, hi in param_blocks(sizes, n_nets):
        w = want[lo:hi]
        if not np.any(w):
            assert not np.any(got[lo:hi]), name
            continue
        tol = floor_tol(bar, rel(emu[lo:hi], w), factor) if emu is not None else bar
        if tol is None:
            continue
        err = rel(got[lo:hi], w)
        assert err <= tol, (name, err, tol)
        n += 1
    return n
