"""World-size-2 gloo test of the data-parallel host logic:
contiguous shards, globally normalised per-rank contributions and one
all-reduce(sum) of [grad, loss] reproduce the single-process loss and gradient,
and every rank ends with identical values (so replicated Adam stays in lockstep)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_14907_b200 import dp, inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = inputs.config("c2")
    cfg.update(sizes=[3, 8, 8, 1])
    pb, ar = oracle.from_config(cfg)
    N, Nb = 512, 64
    lo, hi = dp.shard(rank, world, N)
    blo, bhi = dp.shard(rank, world, Nb)
    # each rank samples only its own indices from the shared counter-based stream
    pts = oracle.sample(0, 0, 3, lo, hi - lo, cfg["H"])
    b = oracle.sample(1, 0, 3, blo, bhi - blo, cfg["H"])
    th = oracle.init_params(ar, 0)
    L, _, g, _ = oracle.loss_grad(pb, ar, th, pts, b, cfg["h"], n_glob=N, nb_glob=Nb, nthreads=1)
    buf = torch.tensor(np.concatenate([g, [L]]), dtype=torch.float64)
    dp.allreduce_sum_(buf)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), buf.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_allreduce_matches_single_process(tmp_path, orc):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r0 = np.load(tmp_path / "r0.npy")
    r1 = np.load(tmp_path / "r1.npy")
    assert np.array_equal(r0, r1)
    cfg = inputs.config("c2")
    cfg.update(sizes=[3, 8, 8, 1])
    pb, ar = orc.from_config(cfg)
    pts = orc.sample(0, 0, 3, 0, 512, cfg["H"])
    b = orc.sample(1, 0, 3, 0, 64, cfg["H"])
    th = orc.init_params(ar, 0)
    L, _, g, _ = orc.loss_grad(pb, ar, th, pts, b, cfg["h"])
    assert r0[-1] == pytest.approx(L, rel=1e-13)
    assert np.allclose(r0[:-1], g, rtol=1e-11, atol=1e-14 * np.abs(g).max())


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 4096, 1 << 22):
        for world in (1, 2, 3, 4, 8):
            ranges = [dp.shard(r, world, n) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
