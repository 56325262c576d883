"""Multi-process data parallelism through libnbm ("distributing collocation
points across multiple processors ... aggregating these locally computed updates"): two ranks,
each a separate process driving the library on cuda:0, sample their contiguous shards of one
global batch, run the CUDA-graph step of bench.py (Solver.capture_step with the all-reduce
between the two graphs) and must reproduce the single-process run on the whole batch: the
all-reduced loss at every step within 1e-6, theta after the steps within the fp32 bar, and the
two ranks' theta bitwise equal (Adam replicated on identical sums); theta within 1e-3 of the
steps' displacement of the single-process run (summation order differs)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
WORKER = os.path.join(HERE, "_mp_worker.py")


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_two_rank_capture_step_matches_single_process(tmp_path):
    steps, n = 4, 1 << 13
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK="0", WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, WORKER, str(tmp_path / f"r{r}.npz"), str(steps), str(n)], env=env))
    for p in procs:
        assert p.wait(timeout=600) == 0
    env = dict(os.environ, RANK="0", LOCAL_RANK="0", WORLD_SIZE="1")
    subprocess.run([sys.executable, WORKER, str(tmp_path / "single.npz"), str(steps), str(2 * n)], env=env,
                   check=True, timeout=600)
    r0, r1, one = (np.load(tmp_path / f) for f in ("r0.npz", "r1.npz", "single.npz"))
    for r in (r0, r1, one):
        assert int(r["status"]) == 0 and int(r["t"]) == steps
    assert np.array_equal(r0["theta"], r1["theta"])                 # replicated Adam, identical sums
    assert np.array_equal(r0["losses"], r1["losses"])
    assert len(r0["losses"]) == steps
    np.testing.assert_allclose(r0["losses"], one["losses"], rtol=1e-6)
    init = np.asarray(r0["theta0"], np.float64)
    moved = np.linalg.norm(one["theta"] - init)                   # the 4 Adam steps' displacement
    assert moved > 0
    assert np.linalg.norm(one["theta"].astype(np.float64) - r0["theta"]) <= 1e-3 * moved
