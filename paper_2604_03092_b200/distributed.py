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
           "ShardedOptimizerState", "sharded_step", "to_shard_major", "from_shard_major"]

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
    """Surfels per optimizer shard: ceil(n / world), so every rank's slice of the packed blocks
    has the same size (the last shard is zero-padded)."""
    return (n + world_size - 1) // world_size


def to_shard_major(flat: torch.Tensor, n: int, c: int) -> torch.Tensor:
    """Plain packed block (13 n) -> the shard-major layout of s2d_view_set_layout (13 W c, W =
    ceil(n / c)): shard s = [means 3c | quats 4c | scales 2c | opacities c | colors 3c] of
    surfels [s c, (s + 1) c), zero-padded."""
    w = (n + c - 1) // c
    out = flat.new_zeros((w, 13 * c))
    off, col = 0, 0
    for d in SEGMENTS:
        seg = flat.new_zeros((w * c, d))
        seg[:n] = flat[off:off + d * n].view(n, d)
        out[:, col * c:(col + d) * c] = seg.view(w, c * d)
        off += d * n
        col += d
    return out.view(-1)


def from_shard_major(flat: torch.Tensor, n: int, c: int) -> torch.Tensor:
    """Inverse of to_shard_major: the plain packed block (13 n)."""
    w = (n + c - 1) // c
    blk = flat.view(w, 13 * c)
    parts, col = [], 0
    for d in SEGMENTS:
        parts.append(blk[:, col * c:(col + d) * c].reshape(w * c, d)[:n].reshape(-1))
        col += d
    return torch.cat(parts)


class ShardedOptimizerState:
    """ZeRO-1 style optimizer sharding over the shard-major packed blocks: rank r owns the
    contiguous slice [13 r c, 13 (r + 1) c) of the parameter and gradient blocks (surfels
    [r c, (r + 1) c)), holds Adam moments for those c surfels only, and updates only them."""

    def __init__(self, n: int, group=None, device=None, dtype=torch.float32, mask=None):
        self.rank, self.world_size = world(group)
        self.group = group
        self.n = n
        self.c = shard_rows(n, self.world_size)
        f = dict(device=device, dtype=dtype)
        self.m1 = torch.zeros(13 * self.c, **f)
        self.m2 = torch.zeros(13 * self.c, **f)
        self.grads = torch.zeros(13 * self.c, **f)  # this rank's summed gradients (reduce-scatter)
        self.mask = None
        if mask is not None:
            self.mask = self.shard_mask(mask)

    def shard_mask(self, mask: torch.Tensor) -> torch.Tensor:
        lo, hi = self.rank * self.c, min((self.rank + 1) * self.c, self.n)
        m = torch.zeros(self.c, dtype=mask.dtype, device=mask.device)
        if hi > lo:
            m[:hi - lo] = mask[lo:hi]
        return m

    def slice(self, block: torch.Tensor) -> torch.Tensor:
        """This rank's contiguous slice of a shard-major block."""
        return block[13 * self.rank * self.c:13 * (self.rank + 1) * self.c]


def sharded_step(params: torch.Tensor, grads: torch.Tensor, state: ShardedOptimizerState, adam_fn,
                 mask: torch.Tensor | None = None, group=None) -> None:
    """One sharded optimizer step on shard-major blocks (13 W c): ONE reduce-scatter (SUM) of the
    gradient block leaves rank r the summed gradients of its surfels, ``adam_fn(p, g, m1, m2, c,
    shard_mask)`` updates its contiguous parameter slice in place, and ONE all-gather writes
    every rank's slice back into every replica (in place under NCCL).  No staging copies: the
    same bytes over NVLink as the all-reduce it replaces, with the optimizer's HBM traffic and
    moment memory divided by the world size."""
    # gloo has no device reduce-scatter / all-gather: device blocks go through host copies
    # (the multi-rank tests on one GPU); NCCL moves them in place over NVLink
    host = dist.get_backend(group) != "nccl" and grads.is_cuda
    if host:
        out = torch.empty(state.grads.shape, dtype=state.grads.dtype)
        dist.reduce_scatter_tensor(out, grads.cpu(), op=dist.ReduceOp.SUM, group=group)
        state.grads.copy_(out)
    else:
        dist.reduce_scatter_tensor(state.grads, grads, op=dist.ReduceOp.SUM, group=group)
    mine = state.slice(params)
    smask = state.mask if mask is None else state.shard_mask(mask)
    adam_fn(mine, state.grads, state.m1, state.m2, state.c, smask)
    if host:
        full = torch.empty(params.shape, dtype=params.dtype)
        dist.all_gather_into_tensor(full, mine.cpu(), group=group)
        params.copy_(full)
    else:
        src = mine if dist.get_backend(group) == "nccl" else mine.clone()
        dist.all_gather_into_tensor(params, src, group=group)


def init_from_env(backend: str = "nccl") -> tuple:
    """Initialise the default process group from torchrun's env (127.0.0.1 rendezvous)."""
    if not (dist.is_available() and "RANK" in os.environ and "WORLD_SIZE" in os.environ):
        return 0, 1
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist.get_rank(), dist.get_world_size()
