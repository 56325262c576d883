"""Data parallelism over collocation points ("distributing collocation
points across multiple processors to compute gradient updates and then
aggregating these locally computed updates").

Rank r of P owns the contiguous global index ranges given by `shard` for the
interior and the boundary points.  It samples them itself from the shared
counter-based stream (no data moves), computes its contribution to the
*global* mean (normalised by the global counts, G18), and one all-reduce(sum)
of the flat [grad(P_theta), loss] buffer yields the exact global L and dL/dtheta
on every rank.  Adam then runs replicated on bitwise-identical inputs.

torch.distributed is plumbing only: the all-reduce runs over NCCL (NVLink /
NVSwitch) on the GPU box and over gloo in the CPU tests.
"""
from __future__ import annotations

import os


def shard(rank: int, world: int, n: int) -> tuple[int, int]:
    """[first, last) of rank's contiguous share of n global indices."""
    return rank * n // world, (rank + 1) * n // world


def env_rank_world() -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def allreduce_sum_(buf, group=None) -> None:
    """In-place sum over ranks of the flat [grad, loss] buffer (one collective per step)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
