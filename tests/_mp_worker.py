"""Worker of test_gpu_multiproc.py (not a test module): one rank of the data-parallel training
step through the C ABI, the step captured by Solver.capture_step with the all-reduce between
the two graphs.  The all-reduce is gloo over host-staged buffers, so the two
processes sharing cuda:0 never run kernels that wait on each other.
usage: python _mp_worker.py OUT.npz STEPS N_PER_RANK   (RANK / WORLD_SIZE / MASTER_* from the env)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2210_14907_b200 import dp, inputs, nbm  # noqa: E402


def main():
    out, steps, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    rank, world, _ = dp.env_rank_world()
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo")
    cfg = inputs.config("c2")
    nb = n // 8
    s = nbm.Solver(cfg, 0, max_points=n)
    s.init_params(0)
    theta0 = s.theta.cpu().numpy()
    pts = torch.empty(n, 3, device="cuda")
    bpts = torch.empty(nb, 3, device="cuda")
    losses = []

    def allreduce(buf):   # host-staged gloo all-reduce of [grad, loss] (the bench's NCCL call on one box)
        h = buf.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM)
        buf.copy_(h.to(buf.device))
        losses.append(float(h[-1]))

    step = s.capture_step(pts, bpts, first=rank * n, bfirst=rank * nb, n_global=n * world, nb_global=nb * world,
                          lr=cfg["lr"], allreduce=allreduce if world > 1 else None)
    for _ in range(steps):
        step()
        if world == 1:
            torch.cuda.synchronize()
            losses.append(float(s.loss.item()))
    torch.cuda.synchronize()
    np.savez(out, theta=s.theta.cpu().numpy(), theta0=theta0, losses=np.array(losses), status=s.status(),
             t=int(s.t_dev.item()))
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
