"""View sharding and the surfel-gradient all-reduce.

The refine objective is a sum over views (mapper.py:300-307), so views are
block-partitioned across ranks; every rank holds a full surfel replica, renders
its own views, and one all-reduce(SUM) of the packed 13N gradient block plus
the scalar loss makes every rank's Adam step identical.  One process per GPU,
``torch.distributed`` for the plumbing: NCCL on B200 (NVLink/NVSwitch), gloo
in the CPU tests.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

__all__ = ["shard_views", "world", "allreduce_grads", "init_from_env"]


def shard_views(n_views: int, rank: int, world_size: int) -> list:
    """Contiguous block partition of view indices; sizes differ by at most one."""
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_views, world_size)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return list(range(start, stop))


def world(group=None) -> tuple:
    """(rank, world_size) of the group, (0, 1) when torch.distributed is not initialised."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def allreduce_grads(grads: torch.Tensor, loss: torch.Tensor | None = None, group=None) -> None:
    """In-place SUM all-reduce of the packed gradient block (and the loss accumulator).

    The float64 loss is folded into the same collective as a float32 tail only when
    dtypes agree; otherwise it gets its own (tiny) all-reduce.
    """
    _, ws = world(group)
    if ws == 1:
        return
    dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
    if loss is not None:
        dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)


def init_from_env(backend: str = "nccl") -> tuple:
    """Initialise the default process group from torchrun's env (127.0.0.1 rendezvous)."""
    if not (dist.is_available() and "RANK" in os.environ and "WORLD_SIZE" in os.environ):
        return 0, 1
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist.get_rank(), dist.get_world_size()
