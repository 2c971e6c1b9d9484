"""Process-group plumbing for the multi-GPU paths (torch.distributed only moves
host-side bookkeeping: the NCCL unique id, timings; all data-path exchange is
in libhysco).  DESIGN.md §8.

* batch DP (configs[3]): each rank corrects its own pairs, no collective on the
  data path; the job time is the max over ranks.
* slab decomposition (configs[4]): rank r owns planes slab_bounds(n1, P, r) of
  every pair; libhysco exchanges one halo plane and allreduces the per-pair
  scalars over NCCL (hysco_create_slab).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import hysco as H


def env():
    """(rank, world, local_rank) from the torchrun environment."""
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def slab_bounds(n1, world, rank):
    return H.slab_bounds(n1, world, rank)


def share_nccl_id(group=None):
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf = torch.tensor(list(H.hysco_nccl_unique_id()), dtype=torch.uint8)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if dist.get_backend(group) == "nccl":
            b = buf.cuda()
            dist.broadcast(b, 0, group=group)
            buf = b.cpu()
        else:
            dist.broadcast(buf, 0, group=group)
    return bytes(buf.tolist())


def max_over_ranks(x: float, device=None) -> float:
    """Job time = max over ranks (B200 bench contract)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
