"""Host logic of the training workload (train.py): epoch sizing and the
convergence order, no GPU needed."""
import math

import pytest

from paper_2210_14907_b200 import train


def test_epoch_plan_covers_the_epoch():
    # N = 8: one step of all 512 interior points and 6 * 9^2 = 486 boundary points
    assert train.epoch_plan(8, 16384) == (1, 512, 486)
    # N = 128: 2^21 interior points in 128 steps of 16384; 6 * 129^2 = 99846 boundary points
    assert train.epoch_plan(128, 16384) == (128, 16384, math.ceil(99846 / 128))
    for N in (4, 16, 32, 64, 256):
        for batch in (1000, 4096, 16384):
            steps, n, nb = train.epoch_plan(N, batch)
            assert n <= batch or steps == 1
            assert steps * n >= N ** 3 and (steps - 1) * n < N ** 3      # the epoch, no extra step
            assert steps * nb >= 6 * (N + 1) ** 2


@pytest.mark.parametrize("N", [0, 3, 6, 12])
def test_epoch_plan_rejects_non_powers_of_two(N):
    with pytest.raises(ValueError):
        train.epoch_plan(N, 16384)


def test_convergence_order_matches_table1_example():
    assert train.convergence_order(3.7e-2, 7.1e-3) == pytest.approx(2.38, abs=0.01)
    with pytest.raises(ValueError):
        train.convergence_order(0.0, 1.0)
