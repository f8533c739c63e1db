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

__all__ = ["shard_views", "world", "allreduce_grads", "init_from_env", "SEGMENTS", "shard_rows",
           "ShardedOptimizerState", "sharded_step"]

# packed parameter block segments (floats per surfel): means, quats, scales, opacity, colour
SEGMENTS = (3, 4, 2, 1, 3)


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


def shard_rows(n: int, world_size: int) -> int:
    """Surfels per optimizer shard: ceil(n / world), so every rank's reduce-scatter chunk has
    the same size (the last shard is zero-padded)."""
    return (n + world_size - 1) // world_size


class ShardedOptimizerState:
    """ZeRO-1 style optimizer sharding: rank r owns surfels [r c, (r + 1) c) of every packed
    segment, holds Adam moments for those c surfels only, and updates only them."""

    def __init__(self, n: int, group=None, device=None, dtype=torch.float32):
        self.rank, self.world_size = world(group)
        self.group = group
        self.n = n
        self.c = shard_rows(n, self.world_size)
        f = dict(device=device, dtype=dtype)
        self.m1 = torch.zeros(13 * self.c, **f)
        self.m2 = torch.zeros(13 * self.c, **f)
        self.params = torch.zeros(13 * self.c, **f)
        self.grads = torch.zeros(13 * self.c, **f)
        self._pad = torch.zeros(self.world_size * self.c * 4, **f)  # one segment, padded
        self._gather = torch.zeros(self.world_size * self.c * 4, **f)

    def _segments(self, flat, rows):
        out, off = [], 0
        for w in SEGMENTS:
            out.append(flat[off:off + w * rows].view(rows, w))
            off += w * rows
        return out


def sharded_step(params: torch.Tensor, grads: torch.Tensor, state: ShardedOptimizerState, adam_fn,
                 mask: torch.Tensor | None = None, group=None) -> None:
    """reduce-scatter(SUM) the packed gradient block by surfel shard, run ``adam_fn`` on this
    rank's shard (packed over its c surfels: ``adam_fn(shard_params, shard_grads, m1, m2, c,
    shard_mask)``), then all-gather the updated parameters into every rank's replica.  Moves
    the same bytes as the all-reduce it replaces and cuts the optimizer's HBM traffic and
    moment memory by the world size."""
    n, c, W, r = state.n, state.c, state.world_size, state.rank
    lo, hi = r * c, min((r + 1) * c, n)
    gseg = state._segments(grads, n)
    pseg = state._segments(params, n)
    sg = state._segments(state.grads, c)
    sp = state._segments(state.params, c)
    for k, w in enumerate(SEGMENTS):
        pad = state._pad[:W * c * w].view(W * c, w)
        pad[:n].copy_(gseg[k])
        pad[n:].zero_()
        dist.reduce_scatter_tensor(sg[k], pad, op=dist.ReduceOp.SUM, group=group)
        sp[k].zero_()
        if hi > lo:
            sp[k][:hi - lo].copy_(pseg[k][lo:hi])
    smask = None
    if mask is not None:
        smask = torch.zeros(c, dtype=mask.dtype, device=mask.device)
        if hi > lo:
            smask[:hi - lo].copy_(mask[lo:hi])
    adam_fn(state.params, state.grads, state.m1, state.m2, c, smask)
    for k, w in enumerate(SEGMENTS):
        out = state._gather[:W * c * w].view(W * c, w)
        dist.all_gather_into_tensor(out, sp[k].contiguous(), group=group)
        pseg[k].copy_(out[:n])


def init_from_env(backend: str = "nccl") -> tuple:
    """Initialise the default process group from torchrun's env (127.0.0.1 rendezvous)."""
    if not (dist.is_available() and "RANK" in os.environ and "WORLD_SIZE" in os.environ):
        return 0, 1
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist.get_rank(), dist.get_world_size()
