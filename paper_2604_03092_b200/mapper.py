"""Refinement on the GPU path.

* :func:`refine` — drop-in for ``surfelslam.mapper.refine`` (mapper.py:276-349):
  backtracking gradient descent on the colours/opacities of the surfels bound
  to the given keyframes, L-inf normalised step, halving, clip to [0, 1],
  warm-started step; the summed loss never increases.  The map stays resident
  on the device for the whole call; every trial is V x (forward + backward)
  through the fused kernels.
* :func:`transform_surfels`, :func:`fuse`, :func:`prune` — drop-ins for the map
  maintenance around refinement (mapper.py:184-260): the map is rendered on the GPU
  and the per-candidate / per-pixel / per-surfel decisions run in the map.cu kernels.
* :class:`AdamRefiner` — the multi-view refinement of BASELINE configs 4-5:
  every iteration renders this rank's views forward+backward (L1 RGB + depth),
  all-reduces the packed 13N gradient block over NCCL, and applies the fused
  Adam step (lr 1e-3 means, 5e-3 the rest) to all surfel parameters.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .distributed import (ShardedOptimizerState, allreduce_grads, from_shard_major, shard_views, sharded_step,
                          to_shard_major, world)
from .engine import (DeviceContext, ImageBuffers, View, camera_struct, config_struct, forward_checked,
                     pack_params, unpack_params)
from .geometry import as_packed_pose
from .rasterizer import (DEFAULT_RASTER_CONFIG, CameraIntrinsics, LossWeights, RasterConfig, SurfelArrays,
                         loss_struct)

__all__ = ["FusionConfig", "RefinementConfig", "RefinementReport", "GlobalSurfelMap", "transform_surfels",
           "fuse", "prune", "refine", "psnr", "AdamConfig", "ViewLoss", "AdamRefiner"]

PSNR_EXACT = float("inf")


def psnr(rendered, target) -> float:
    """10 log10(1/MSE) over all channels of [0,1] images; inf on MSE=0 (evaluation.py:63-72)."""
    rendered = np.asarray(rendered, dtype=float)
    target = np.asarray(target, dtype=float)
    if rendered.shape != target.shape:
        raise ValueError("image dimensions differ")
    mse = float(np.mean((rendered - target) ** 2))
    if mse == 0.0:
        return PSNR_EXACT
    return 10.0 * math.log10(1.0 / mse)


@dataclass(frozen=True)
class FusionConfig:
    """mapper.py:53-62"""

    accum_threshold: float = 0.5
    prune_rgb_error: float = 0.2
    prune_depth_error_frac: float = 0.10
    prune_contribution_floor: float = 0.1

    def __post_init__(self):
        if not 0 < self.accum_threshold < 1:
            raise ValueError("accum_threshold must be in (0, 1)")
        if min(self.prune_rgb_error, self.prune_depth_error_frac, self.prune_contribution_floor) <= 0:
            raise ValueError("prune thresholds must be positive")


@dataclass(frozen=True)
class RefinementConfig:
    """mapper.py:64-70"""

    iterations: int = 20
    keyframes: int = 4
    initial_step: float = 0.1
    min_step: float = 1e-6
    loss: LossWeights = field(default_factory=LossWeights)


@dataclass
class RefinementReport:
    """mapper.py:268-273"""

    losses: list
    psnr_before: float
    psnr_after: float
    accepted_steps: int


@dataclass
class GlobalSurfelMap:
    """World-frame surfel store with keyframe bindings (mapper.py:73-103)."""

    surfels: SurfelArrays = field(default_factory=SurfelArrays.empty)
    keyframe_poses: dict = field(default_factory=dict)

    def __len__(self):
        return len(self.surfels)

    @property
    def keyframe_index(self):
        """keyframe_id -> surfel indices; covers every surfel exactly once."""
        out = {}
        for i, kf in enumerate(np.asarray(self.surfels.keyframe_ids)):
            out.setdefault(int(kf), []).append(i)
        return out

    def insert(self, new: SurfelArrays):
        unknown = set(np.unique(np.asarray(new.keyframe_ids)).tolist()) - set(self.keyframe_poses)
        if unknown:
            raise KeyError(f"surfels bound to unregistered keyframes {sorted(unknown)}")
        self.surfels = SurfelArrays.concatenate([self.surfels, new])

    def remove(self, indices):
        keep = np.ones(len(self.surfels), dtype=bool)
        keep[np.asarray(indices, dtype=int)] = False
        self.surfels = self.surfels.select(keep)

    def copy(self) -> "GlobalSurfelMap":
        return GlobalSurfelMap(self.surfels.copy(), dict(self.keyframe_poses))


# --------------------------------------------------------------------------- map maintenance

def _stream():
    return torch.cuda.current_stream().cuda_stream


def _host_block(t: torch.Tensor, n: int) -> dict:
    return {k: v.double().cpu().numpy() for k, v in unpack_params(t, n).items()}


def transform_surfels(surfels: SurfelArrays, t) -> SurfelArrays:
    """Camera->world per the node pose (mapper.py:184-197): means by the Sim(3) action,
    rotations left-composed and canonicalised, tangent scales times the pose scale.
    Computed by k_transform (float64 in the reference's order, float32 result)."""
    arrays = SurfelArrays.from_surfels(surfels)
    n = len(arrays)
    if n == 0:
        return arrays.copy()
    ctx = DeviceContext.get()
    pin = pack_params(arrays, ctx.device)
    out = torch.empty_like(pin)
    N.check(N.lib().s2d_transform_surfels(_stream(), N.as_doubles(as_packed_pose(t)), N.dptr(pin), n,
                                          N.dptr(out)), "s2d_transform_surfels")
    P = _host_block(out, n)
    return SurfelArrays(P["means"], P["quats"], P["scales"], P["opacities"], P["colors"],
                        np.array(arrays.confidences, copy=True), np.array(arrays.keyframe_ids, copy=True),
                        np.array(arrays.submap_ids, copy=True))


def fuse(map_: GlobalSurfelMap, new_surfels: SurfelArrays, keyframe_id: int, pose, intr: CameraIntrinsics,
         cfg: FusionConfig = FusionConfig(), raster_cfg: RasterConfig = DEFAULT_RASTER_CONFIG,
         submap_id: int = -1) -> dict:
    """Insert camera-frame surfels where the map's accumulation is still low (mapper.py:200-230).

    The map's accumulation is rendered on the GPU from the keyframe pose; k_fuse_gate looks
    up each candidate's own pixel; the kept candidates are warped to the world frame by
    k_transform and appended."""
    if keyframe_id not in map_.keyframe_poses:
        map_.keyframe_poses[keyframe_id] = pose
    cand = SurfelArrays.from_surfels(new_surfels)
    n_cand = len(cand)
    if n_cand == 0:
        return {"candidates": 0, "inserted": 0}
    ctx = DeviceContext.get()
    dev = ctx.device
    cp = pack_params(cand, dev)
    if len(map_) == 0:
        keep = np.ones(n_cand, dtype=bool)
    else:
        from .rasterizer import _device_render
        _, _, img, _, _, _ = _device_render(map_.surfels, pose, intr, raster_cfg, normal=False)
        keep_t = torch.empty(n_cand, dtype=torch.uint8, device=dev)
        N.check(N.lib().s2d_fuse_gate(_stream(), N.dptr(img.accumulation), ctypes.byref(camera_struct(intr)),
                                      N.dptr(cp), n_cand, float(cfg.accum_threshold), N.dptr(keep_t)),
                "s2d_fuse_gate")
        keep = keep_t.cpu().numpy().astype(bool)
    world = transform_surfels(cand.select(keep), pose)
    world.keyframe_ids = np.full(len(world), keyframe_id, np.int64)
    world.submap_ids = np.full(len(world), submap_id, np.int64)
    map_.insert(world)
    return {"candidates": n_cand, "inserted": int(keep.sum())}


def prune(map_: GlobalSurfelMap, keyframe_id: int, observed_rgb, observed_depth, intr: CameraIntrinsics,
          cfg: FusionConfig = FusionConfig(), raster_cfg: RasterConfig = DEFAULT_RASTER_CONFIG) -> int:
    """Remove surfels that contribute to pixels with large reconstruction error (mapper.py:238-260).

    Render (GPU), k_prune_mark over the pixels, the forward's per-surfel max weight over
    the marked pixels, k_prune_keep; the victims are removed from the map."""
    if len(map_) == 0:
        return 0
    pose = map_.keyframe_poses[keyframe_id]
    from .rasterizer import _device_render
    arrays, params, img, _, view, _ = _device_render(map_.surfels, pose, intr, raster_cfg, normal=False)
    dev = params.device
    n = len(arrays)
    orgb = torch.from_numpy(np.ascontiguousarray(np.asarray(observed_rgb, dtype=np.float32))).to(dev)
    odep = torch.from_numpy(np.ascontiguousarray(np.asarray(observed_depth, dtype=np.float32))).to(dev)
    if orgb.shape != (intr.height, intr.width, 3) or odep.shape != (intr.height, intr.width):
        raise ValueError("observation dimensions do not match the camera")
    npx = intr.width * intr.height
    marked = torch.empty((intr.height, intr.width), dtype=torch.uint8, device=dev)
    N.check(N.lib().s2d_prune_mark(_stream(), N.dptr(img.color), N.dptr(img.depth), N.dptr(img.accumulation),
                                   N.dptr(orgb), N.dptr(odep), npx, float(cfg.prune_rgb_error),
                                   float(cfg.prune_depth_error_frac), N.dptr(marked)), "s2d_prune_mark")
    if not bool(marked.any()):
        return 0
    max_all = torch.zeros(n, device=dev)
    max_marked = torch.zeros(n, device=dev)
    forward_checked(view, params, n, as_packed_pose(pose), camera_struct(intr), config_struct(raster_cfg), img,
                    max_all, max_marked, marked)
    keep = torch.empty(n, dtype=torch.uint8, device=dev)
    N.check(N.lib().s2d_prune_keep(_stream(), N.dptr(max_marked), n, float(cfg.prune_contribution_floor),
                                   N.dptr(keep)), "s2d_prune_keep")
    victims = np.flatnonzero(keep.cpu().numpy() == 0)
    if len(victims):
        map_.remove(victims)
    return int(len(victims))


class _ViewSet:
    """Device-resident targets + one reusable workspace for a list of views."""

    def __init__(self, intr, poses, rgbs, depths, raster_cfg, device):
        self.ctx = DeviceContext.get(device)
        self.dev = self.ctx.device
        self.intr = intr
        self.cam = camera_struct(intr)
        self.cfg = config_struct(raster_cfg)
        self.poses = [as_packed_pose(p) for p in poses]
        self.rgb = [torch.from_numpy(np.asarray(r, dtype=np.float32)).to(self.dev) for r in rgbs]
        self.depth = [torch.from_numpy(np.asarray(d, dtype=np.float32)).to(self.dev) for d in depths]
        self.view = View(self.ctx)
        self.img = ImageBuffers.allocate(intr.height, intr.width, self.dev, normal=False)


def refine(map_: GlobalSurfelMap, keyframe_ids, observations, intr: CameraIntrinsics,
           cfg: RefinementConfig = RefinementConfig(),
           raster_cfg: RasterConfig = DEFAULT_RASTER_CONFIG) -> RefinementReport:
    """Backtracking GD on colours/opacities of the surfels bound to ``keyframe_ids``
    (mapper.py:276-349).  ``observations`` maps keyframe_id -> (rgb, depth).

    The map stays on the device: every trial is the views' fused forward + backward
    (s2d_forward / s2d_backward), the L-inf norm and the clipped step run in
    s2d_refine_gnorm / s2d_refine_gd.  Like the reference, a trial clips every surfel's
    colour and opacity to [0, 1] (np.clip over the whole arrays, mapper.py:334-335), and the
    last rejected trial restores the previous state (mapper.py:346-347)."""
    keyframe_ids = [k for k in keyframe_ids if k in observations]
    poses = [map_.keyframe_poses[k] for k in keyframe_ids]
    target_mask = np.isin(np.asarray(map_.surfels.keyframe_ids), np.asarray(keyframe_ids, dtype=np.int64))
    n = len(map_.surfels)
    if not keyframe_ids:
        return RefinementReport([], float("inf"), float("inf"), 0)
    vs = _ViewSet(intr, poses, [observations[k][0] for k in keyframe_ids],
                  [observations[k][1] for k in keyframe_ids], raster_cfg, None)
    dev = vs.dev
    L = N.lib()
    params = pack_params(map_.surfels, dev) if n else torch.zeros(13, device=dev)
    grads = [torch.zeros_like(params), torch.zeros_like(params)]  # current / trial
    loss_acc = torch.zeros(1, dtype=torch.float64, device=dev)
    lw = cfg.loss

    def view_psnrs():
        vals = []
        for v in range(len(poses)):
            forward_checked(vs.view, params, n, vs.poses[v], vs.cam, vs.cfg, vs.img)
            vals.append(psnr(vs.img.color.cpu().numpy(), observations[keyframe_ids[v]][0]))
        finite = [x for x in vals if math.isfinite(x)]
        return float(np.mean(finite)) if finite else float("inf")

    def total_loss_and_grads(g):
        """Sum over the views of the reference loss and its gradients (mapper.py:300-313)."""
        g.zero_()
        loss_acc.zero_()
        for v in range(len(poses)):
            forward_checked(vs.view, params, n, vs.poses[v], vs.cam, vs.cfg, vs.img)
            vs.view.backward(params, n, vs.img,
                             loss_struct(N.LOSS_MSE, lw.mse, lw.depth, True, vs.rgb[v], vs.depth[v]),
                             g, loss_acc)
        return float(loss_acc.item())

    psnr_before = view_psnrs()
    if cfg.iterations == 0 or not target_mask.any() or n == 0:
        return RefinementReport([], psnr_before, psnr_before, 0)
    mask_t = torch.from_numpy(target_mask.astype(np.uint8)).to(dev)
    gn = torch.zeros(1, device=dev)
    params0 = torch.empty_like(params)
    stream = _stream()
    loss = total_loss_and_grads(grads[0])
    losses = [loss]
    accepted = 0
    step_scale = cfg.initial_step
    for _ in range(cfg.iterations):
        N.check(L.s2d_refine_gnorm(stream, N.dptr(grads[0]), n, N.dptr(mask_t), N.dptr(gn)), "s2d_refine_gnorm")
        gnorm = float(gn.item())
        if gnorm < 1e-14:
            break
        step = step_scale / gnorm
        params0.copy_(params)
        improved = False
        while step >= cfg.min_step / gnorm:
            N.check(L.s2d_refine_gd(stream, N.dptr(params), N.dptr(params0), N.dptr(grads[0]), n, float(step),
                                    N.dptr(mask_t)), "s2d_refine_gd")
            new_loss = total_loss_and_grads(grads[1])
            if new_loss < loss:
                loss = new_loss
                grads.reverse()
                losses.append(loss)
                accepted += 1
                improved = True
                step_scale = min(2.0 * step * gnorm, cfg.initial_step)
                break
            step *= 0.5
        if not improved:
            params.copy_(params0)
            break
    if accepted:
        P = unpack_params(params, n)
        cols = np.clip(np.asarray(map_.surfels.colors, dtype=float), 0.0, 1.0)
        ops = np.clip(np.asarray(map_.surfels.opacities, dtype=float), 0.0, 1.0)
        idx = np.flatnonzero(target_mask)
        cols[idx] = P["colors"].double().cpu().numpy()[idx]
        ops[idx] = P["opacities"].double().cpu().numpy()[idx]
        map_.surfels.colors = cols
        map_.surfels.opacities = ops
    return RefinementReport(losses, psnr_before, view_psnrs(), accepted)


# --------------------------------------------------------------------------- Adam refinement


@dataclass(frozen=True)
class AdamConfig:
    lr_means: float = 1e-3
    lr_rest: float = 5e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    scale_min: float = 1e-7

    def struct(self) -> N.AdamCfg:
        return N.AdamCfg(self.lr_means, self.lr_rest, self.beta1, self.beta2, self.eps, self.scale_min)


@dataclass(frozen=True)
class ViewLoss:
    """Per-view loss of the Adam refinement: L1 RGB + w_depth * L1 depth (BASELINE config 4)."""

    kind: str = "l1"
    w_rgb: float = 1.0
    w_depth: float = 0.1
    depth_mask: bool = False

    def code(self) -> int:
        return {"l1": N.LOSS_L1, "mse": N.LOSS_MSE}[self.kind]

    def fusable(self) -> bool:
        """The seeds need no whole-image reduction (s2d_forward_backward's one-kernel path)."""
        return (self.kind == "l1" and not self.depth_mask) or (self.kind == "mse" and self.w_depth == 0.0)


class _Lane:
    """One stream's worth of view state: workspace and render buffers."""

    def __init__(self, ctx, h, w, dev):
        self.stream = torch.cuda.Stream(dev)
        self.view = View(ctx)
        self.img = ImageBuffers.allocate(h, w, dev, normal=False)


class AdamRefiner:
    """Multi-view fused-Adam refinement of all surfel parameters, views sharded over ranks.

    With N > 1 ranks the optimizer is sharded by default (``shard_optimizer``): the packed
    parameter and gradient blocks use the shard-major layout (s2d_view_set_layout, c =
    ceil(n / N) surfels per rank), so ONE reduce-scatter leaves each rank the summed gradients
    of its contiguous slice, the fused Adam kernel updates that slice in place (moments for c
    surfels), and ONE in-place all-gather refreshes every replica.

    ``targets_rgb[v]`` (H,W,3) / ``targets_depth[v]`` (H,W) may be numpy arrays, device
    tensors, or (``host_targets=True``) host tensors that are pinned and copied in every
    step on a copy stream, each view's first reader of them (the fused raster kernel, or the
    backward) waiting for its own copy (the end-to-end path: the transfers overlap the
    projections, sorts and the other views' compute).
    ``inflight`` views run concurrently on separate streams.

    ``step(sync=False)`` queues an iteration without a host round trip: the Adam step is
    skipped on the device when a view overflowed its pair capacity (the overflow word of the
    views' accumulated stats, all-reduced over ranks), and the host notices it one iteration
    later, regrows the capacity and re-runs the skipped iterations, so the sequence of applied
    steps is exactly that of a synchronous loop.  The loss of every iteration is copied to
    pinned host memory on the device's queue; ``losses()`` returns them.
    """

    def __init__(self, surfels, intr: CameraIntrinsics, poses, targets_rgb, targets_depth,
                 loss: ViewLoss = ViewLoss(), adam: AdamConfig = AdamConfig(),
                 raster_cfg: RasterConfig = DEFAULT_RASTER_CONFIG, mask=None, group=None, device=None,
                 host_targets: bool = False, inflight: int = 16, shard_optimizer: bool | None = None,
                 cuda_graph: bool = False, fused: bool = True):
        self.ctx = DeviceContext.get(device)
        self.dev = self.ctx.device
        self.group = group
        self.rank, self.world_size = world(group)
        self.intr = intr
        self.cam = camera_struct(intr)
        self.cfg = config_struct(raster_cfg)
        if isinstance(surfels, torch.Tensor):
            plain = surfels.to(self.dev, torch.float32).contiguous()
            self.n = plain.numel() // 13
        else:
            self.n = len(surfels)
            plain = pack_params(surfels, self.dev)
        # N > 1: ZeRO-1 style optimizer sharding over the shard-major blocks unless disabled
        self.sharded = (self.world_size > 1) if shard_optimizer is None else bool(shard_optimizer)
        self.mask = None if mask is None else torch.as_tensor(np.asarray(mask, dtype=np.uint8)).to(self.dev)
        if self.sharded:
            self.opt_state = ShardedOptimizerState(self.n, group, self.dev, mask=self.mask)
            self.shard = self.opt_state.c
            self.params = to_shard_major(plain, self.n, self.shard) if self.shard < self.n else plain
            self.m1, self.m2 = self.opt_state.m1, self.opt_state.m2
        else:
            self.shard = self.n
            self.params = plain
            self.m1 = torch.zeros_like(self.params)
            self.m2 = torch.zeros_like(self.params)
        self.grads = torch.zeros_like(self.params)
        self.all_poses = [as_packed_pose(p) for p in poses]
        self.my_views = shard_views(len(self.all_poses), self.rank, self.world_size)
        self.loss_cfg = loss
        # forward, loss and backward of a view in one raster kernel where the loss allows it
        self.fused = bool(fused) and loss.fusable()
        self.adam = adam.struct()
        self.host_targets = host_targets
        h, w = intr.height, intr.width
        self.rgb, self.depth = {}, {}
        for v in self.my_views:
            r, d = targets_rgb[v], targets_depth[v]
            if host_targets:
                r = torch.as_tensor(np.asarray(r, dtype=np.float32)) if not isinstance(r, torch.Tensor) else r
                d = torch.as_tensor(np.asarray(d, dtype=np.float32)) if not isinstance(d, torch.Tensor) else d
                self.rgb[v] = r.float().contiguous().pin_memory()
                self.depth[v] = d.float().contiguous().pin_memory()
            else:
                self.rgb[v] = torch.as_tensor(np.asarray(r, dtype=np.float32) if not isinstance(r, torch.Tensor) else r).to(self.dev, torch.float32)
                self.depth[v] = torch.as_tensor(np.asarray(d, dtype=np.float32) if not isinstance(d, torch.Tensor) else d).to(self.dev, torch.float32)
        self.inflight = max(1, int(inflight))
        self.active_lanes = self.inflight
        self.lanes = [_Lane(self.ctx, h, w, self.dev) for _ in range(self.inflight)]
        for lane in self.lanes:
            N.check(N.lib().s2d_view_set_layout(lane.view.handle, self.shard if self.shard < self.n else 0),
                    "s2d_view_set_layout")
        if host_targets:
            # end-to-end path: every view's targets go up on a copy stream at the start of the
            # step, into per-view device buffers; a view's raster kernel (the fused path) or
            # backward, the only reader, waits for its own copy, so the transfers overlap the
            # projections, sorts and the other views
            self.copy_stream = torch.cuda.Stream(self.dev)
            self.dev_rgb = {v: torch.empty((h, w, 3), device=self.dev) for v in self.my_views}
            self.dev_depth = {v: torch.empty((h, w), device=self.dev) for v in self.my_views}
        self.view = self.lanes[0].view  # the first lane (phase timing / inspection)
        self.loss_acc = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.stats_acc = torch.zeros(8, dtype=torch.int32, device=self.dev)
        self.step_count = 0
        # CUDA graph of one step's views (forward, stats, backward on every lane stream): one
        # launch per step instead of ~4 library calls per view from Python
        self.cuda_graph = bool(cuda_graph)
        self._graph = None
        self._graph_launches = 0
        self.kernel_launches = 0  # library kernels launched by step() (graph replays included)
        self.regrows = 0  # iterations re-run after a view overflowed the pair capacity
        self.h2d_bytes_per_step = (sum(self.rgb[v].numel() + self.depth[v].numel() for v in self.my_views) * 4
                                   if host_targets else 0)
        self._pending = []  # queued iterations: (step, pinned stats, pinned loss, done event)
        self._losses = []
        self._size_pairs()

    def _size_pairs(self):
        """One forward per view to size the pair capacity (1.3 x the largest view)."""
        mx = 0
        lane = self.lanes[0]
        for v in self.my_views:
            st = forward_checked(lane.view, self.params, self.n, self.all_poses[v], self.cam, self.cfg, lane.img)
            mx = max(mx, st.pairs)
        self._reserve(int(mx * 1.3) + 4096)

    def _reserve(self, pairs):
        for lane in self.lanes:
            lane.view.reserve_pairs(pairs)

    def compute_grads(self):
        """grads <- sum over this rank's views of d(loss)/d(params); loss_acc <- sum of losses.

        Views are dealt round-robin to `active_lanes` streams, each with its own workspace
        and image buffers, so one view's projection/sort overlaps another's compositing;
        gradients, loss and stats accumulate atomically into shared buffers.
        """
        main = torch.cuda.current_stream(self.dev)
        self.grads.zero_()
        self.loss_acc.zero_()
        self.stats_acc.zero_()
        lanes = self.lanes[: self.active_lanes]
        for lane in lanes:
            lane.stream.wait_stream(main)
        copied = {}
        if self.host_targets:
            cs = self.copy_stream
            cs.wait_stream(main)
            with torch.cuda.stream(cs):
                for v in self.my_views:
                    self.dev_rgb[v].copy_(self.rgb[v], non_blocking=True)
                    self.dev_depth[v].copy_(self.depth[v], non_blocking=True)
                    copied[v] = torch.cuda.Event()
                    copied[v].record(cs)
        lc = self.loss_cfg
        for j, v in enumerate(self.my_views):
            lane = lanes[j % len(lanes)]
            s = lane.stream
            if self.host_targets:
                trgb, tdep = self.dev_rgb[v], self.dev_depth[v]
            else:
                trgb, tdep = self.rgb[v], self.depth[v]
            ls = loss_struct(lc.code(), lc.w_rgb, lc.w_depth, lc.depth_mask, trgb, tdep)
            if self.fused:
                # the raster kernel waits for this view's target upload, the projection and
                # sorts before it do not
                lane.view.forward_backward(self.params, self.n, self.all_poses[v], self.cam, self.cfg, None, ls,
                                           self.grads, self.loss_acc, stream=s, wait_event=copied.get(v))
                lane.view.accumulate_stats(self.stats_acc, stream=s)
                continue
            lane.view.forward(self.params, self.n, self.all_poses[v], self.cam, self.cfg, lane.img, stream=s)
            lane.view.accumulate_stats(self.stats_acc, stream=s)
            if self.host_targets:
                s.wait_event(copied[v])
            lane.view.backward(self.params, self.n, lane.img, ls, self.grads, self.loss_acc, stream=s)
        for lane in lanes:
            main.wait_stream(lane.stream)
        if self.host_targets:
            main.wait_stream(self.copy_stream)

    def _capture(self):
        """Capture compute_grads into a CUDA graph.  The pair capacities must already fit (an
        eager step sized them): the library does not allocate while they do."""
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        l0 = N.lib().s2d_launch_count()
        with torch.cuda.graph(g):
            self.compute_grads()
        self._graph_launches = N.lib().s2d_launch_count() - l0
        self._graph = g

    def _enqueue(self):
        """Queue one iteration: views forward+backward, collectives, the gated Adam step, and the
        stats / loss copies to pinned host memory."""
        l0 = N.lib().s2d_launch_count()
        if self.cuda_graph and self.step_count > 0:
            if self._graph is None:
                self._capture()
            self._graph.replay()
            self.kernel_launches += self._graph_launches
        else:
            self.compute_grads()
        step = self.step_count + 1
        overflow = self.stats_acc[4:5]
        if self.world_size > 1:
            # every rank must skip together: the overflow word (and the max pair count) over ranks
            import torch.distributed as dist
            dist.all_reduce(self.stats_acc, op=dist.ReduceOp.MAX, group=self.group)
        if self.sharded:
            allreduce_grads(self.loss_acc, None, self.group)
            sharded_step(self.params, self.grads, self.opt_state,
                         lambda p, g, m1, m2, c, m: self._adam(p, g, m1, m2, c, m, step, overflow), None, self.group)
        else:
            allreduce_grads(self.grads, self.loss_acc, self.group)
            self._adam(self.params, self.grads, self.m1, self.m2, self.n, self.mask, step, overflow)
        self.kernel_launches += N.lib().s2d_launch_count() - l0
        hs = torch.empty(8, dtype=torch.int32).pin_memory()
        hl = torch.empty(1, dtype=torch.float64).pin_memory()
        hs.copy_(self.stats_acc, non_blocking=True)
        hl.copy_(self.loss_acc, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        self.step_count = step
        self._pending.append((step, hs, hl, ev))

    def _resolve(self, keep: int):
        """Settle all but the newest `keep` queued iterations (waits for them).  On an overflow,
        the iterations from the overflowing one on were all skipped on the device (the
        parameters did not change, so each overflowed again): regrow and re-run them."""
        while len(self._pending) > keep:
            step, hs, hl, ev = self._pending[0]
            ev.synchronize()
            if int(hs[4]):
                redo = len(self._pending)
                torch.cuda.synchronize(self.dev)
                self._pending.clear()
                self.step_count = step - 1
                self._reserve(int(hs[1]) * 5 // 4 + 4096)
                self._graph = None  # buffers may have moved: capture again
                self.regrows += 1
                for _ in range(redo):
                    self._enqueue()
                continue
            self._losses.append(float(hl[0]))
            self._pending.pop(0)

    def step(self, sync: bool = True):
        """One refine iteration; with ``sync`` returns the total loss over ALL views (all
        ranks), else queues it (``losses()`` collects the values)."""
        self._resolve(keep=1)  # the previous iteration is checked while this one is queued
        self._enqueue()
        if sync:
            self._resolve(keep=0)
            return self._losses[-1]
        return None

    def losses(self) -> list:
        """Losses of all iterations so far (waits for the queued ones)."""
        self._resolve(keep=0)
        return list(self._losses)

    def _adam(self, params, grads, m1, m2, n, mask, step, skip=None):
        N.check(N.lib().s2d_adam_step_gated(torch.cuda.current_stream(self.dev).cuda_stream, N.dptr(params),
                                            N.dptr(grads), N.dptr(m1), N.dptr(m2), int(n), int(step), self.adam,
                                            N.dptr(mask), N.dptr(skip)), "s2d_adam_step_gated")

    def plain_params(self) -> torch.Tensor:
        """The parameters in the plain packed layout (13 n)."""
        self._resolve(keep=0)
        return from_shard_major(self.params, self.n, self.shard) if self.shard < self.n else self.params

    def plain_grads(self) -> torch.Tensor:
        """The last iteration's summed gradients (this rank's views; plain layout)."""
        return from_shard_major(self.grads, self.n, self.shard) if self.shard < self.n else self.grads

    def surfel_arrays(self) -> SurfelArrays:
        P = unpack_params(self.plain_params(), self.n)
        return SurfelArrays(*[P[k].double().cpu().numpy() for k in ("means", "quats", "scales", "opacities",
                                                                     "colors")])
