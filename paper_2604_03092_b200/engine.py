"""Device-level engine over the C ABI: contexts, views, packed parameters.

PyTorch is plumbing here (device memory, streams); all compute runs in
``lib/libsurfel2d.so``.  A :class:`View` owns one workspace arena and the
state of its last forward, so ``forward`` then ``backward`` on the same view
is the fused render+gradient path of one camera (rasterizer.py:360-399).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .geometry import as_packed_pose

__all__ = [
    "pack_params", "unpack_params", "DeviceContext", "View", "ImageBuffers", "camera_struct",
    "config_struct", "default_device", "PARAM_SEGMENTS",
]

# packed parameter block layout [means 3n | quats 4n | scales 2n | opacities n | colors 3n]
PARAM_SEGMENTS = (("means", 3), ("quats", 4), ("scales", 2), ("opacities", 1), ("colors", 3))


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise N.NativeLibraryError("no CUDA device: this package has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def pack_params(arrays, device=None) -> torch.Tensor:
    """SurfelArrays-like (numpy/torch fields) -> packed float32 (13n,) tensor on the device."""
    device = device or default_device()
    parts = []
    for name, k in PARAM_SEGMENTS:
        a = getattr(arrays, name)
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32)))
        parts.append(t.reshape(-1).to(device=device, dtype=torch.float32))
    return torch.cat(parts).contiguous()


def unpack_params(flat: torch.Tensor, n: int) -> dict:
    """Views (no copy) of the packed block as (n, k) tensors."""
    out, off = {}, 0
    for name, k in PARAM_SEGMENTS:
        out[name] = flat[off:off + k * n].view(n, k) if k > 1 else flat[off:off + n]
        off += k * n
    return out


def camera_struct(intr) -> N.Camera:
    return N.Camera(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy), int(intr.width),
                    int(intr.height))


def config_struct(cfg) -> N.RasterCfg:
    mode = {"affine": 0, "ray": 1}[getattr(cfg, "splat_mode", "affine")]
    return N.RasterCfg(float(cfg.weight_clamp), float(cfg.termination_transmittance),
                       float(cfg.footprint_sigma), float(cfg.near_plane), float(cfg.max_condition),
                       float(cfg.max_view_angle_deg), float(cfg.center_margin_frac), mode, 0)


@dataclass
class ImageBuffers:
    """Device render targets (torch tensors); None = not produced."""

    color: torch.Tensor | None = None
    depth: torch.Tensor | None = None
    accumulation: torch.Tensor | None = None
    normal: torch.Tensor | None = None
    max_w: torch.Tensor | None = None
    arg_w: torch.Tensor | None = None

    @classmethod
    def allocate(cls, h, w, device, normal=True, argmax=False):
        f = dict(device=device, dtype=torch.float32)
        return cls(torch.empty((h, w, 3), **f), torch.empty((h, w), **f), torch.empty((h, w), **f),
                   torch.empty((h, w, 3), **f) if normal else None,
                   torch.empty((h, w), **f) if argmax else None,
                   torch.empty((h, w), device=device, dtype=torch.int32) if argmax else None)

    def struct(self) -> N.Image:
        return N.Image(N.dptr(self.color), N.dptr(self.depth), N.dptr(self.accumulation),
                       N.dptr(self.normal), N.dptr(self.max_w), N.dptr(self.arg_w))


class _DevArray:
    """Zero-copy __cuda_array_interface__ wrapper of a raw device pointer."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _wrap(ptr, shape, typestr, device) -> torch.Tensor:
    if int(np.prod(shape)) == 0:
        dt = {"<u4": torch.int32, "<i4": torch.int32, "<i2": torch.int16, "<f8": torch.float64,
              "|u1": torch.uint8, "<f4": torch.float32}[typestr]
        return torch.empty(shape, dtype=dt, device=device)
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device=device)


class DeviceContext:
    """One C-ABI context per CUDA device (created lazily, process-wide)."""

    _lock = threading.Lock()
    _instances: dict = {}

    def __init__(self, device_index: int):
        L = N.lib()
        h = N.c_p()
        N.check(L.s2d_ctx_create(int(device_index), ctypes.byref(h)), "s2d_ctx_create")
        self.handle = h
        self.device = torch.device("cuda", device_index)
        self._tls = threading.local()

    @classmethod
    def get(cls, device=None) -> "DeviceContext":
        device = torch.device(device) if device is not None else default_device()
        idx = device.index if device.index is not None else torch.cuda.current_device()
        with cls._lock:
            if idx not in cls._instances:
                cls._instances[idx] = DeviceContext(idx)
            return cls._instances[idx]

    def thread_view(self) -> "View":
        """A per-thread reusable view (workspace arena) for one-shot render calls."""
        v = getattr(self._tls, "view", None)
        if v is None:
            v = View(self)
            self._tls.view = v
        return v

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            N.lib().s2d_ctx_destroy(self.handle)
        except Exception:
            pass


class View:
    """A camera view's workspace arena + forward state (s2d_view)."""

    def __init__(self, ctx: DeviceContext):
        self.ctx = ctx
        h = N.c_p()
        N.check(N.lib().s2d_view_create(ctx.handle, ctypes.byref(h)), "s2d_view_create")
        self.handle = h
        self.device = ctx.device
        self._last = None  # (n, h, w)

    def __del__(self):  # pragma: no cover
        try:
            N.lib().s2d_view_destroy(self.handle)
        except Exception:
            pass

    @staticmethod
    def _stream(stream):
        s = stream if stream is not None else torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def forward(self, params: torch.Tensor, n: int, pose, cam: N.Camera, cfg: N.RasterCfg,
                image: ImageBuffers, max_all=None, max_marked=None, mask=None, stream=None):
        pose8 = N.as_doubles(as_packed_pose(pose))
        img = image.struct()
        N.check(N.lib().s2d_forward(self.handle, self._stream(stream), N.dptr(params), int(n), pose8,
                                    ctypes.byref(cam), ctypes.byref(cfg), ctypes.byref(img),
                                    N.dptr(max_all), N.dptr(max_marked), N.dptr(mask)), "s2d_forward")
        self._last = (int(n), int(cam.height), int(cam.width))

    def backward(self, params: torch.Tensor, n: int, image: ImageBuffers, loss: N.Loss,
                 grads: torch.Tensor, loss_accum: torch.Tensor | None = None, stream=None):
        img = image.struct()
        N.check(N.lib().s2d_backward(self.handle, self._stream(stream), N.dptr(params), int(n),
                                     ctypes.byref(img), ctypes.byref(loss), N.dptr(grads),
                                     N.dptr(loss_accum)), "s2d_backward")

    def forward_backward(self, params: torch.Tensor, n: int, pose, cam: N.Camera, cfg: N.RasterCfg,
                         image: ImageBuffers | None, loss: N.Loss, grads: torch.Tensor,
                         loss_accum: torch.Tensor | None = None, stream=None, wait_event=None):
        """s2d_forward_backward: render + loss + backward in one raster kernel for the losses
        without the whole-image depth mask (else forward then backward).  `image` may be None
        on the fused path; `wait_event` (torch.cuda.Event) is waited for before the loss
        targets are read."""
        pose8 = N.as_doubles(as_packed_pose(pose))
        img = image.struct() if image is not None else None
        ev = ctypes.c_void_p(wait_event.cuda_event) if wait_event is not None else None
        N.check(N.lib().s2d_forward_backward(self.handle, self._stream(stream), N.dptr(params), int(n), pose8,
                                             ctypes.byref(cam), ctypes.byref(cfg),
                                             ctypes.byref(img) if img is not None else None, ctypes.byref(loss),
                                             N.dptr(grads), N.dptr(loss_accum), ev), "s2d_forward_backward")
        self._last = (int(n), int(cam.height), int(cam.width))

    def stats(self) -> N.ViewStats:
        st = N.ViewStats()
        N.check(N.lib().s2d_view_stats_host(self.handle, ctypes.byref(st)), "s2d_view_stats_host")
        return st

    def accumulate_stats(self, acc: torch.Tensor, stream=None):
        N.check(N.lib().s2d_view_stats_accumulate(self.handle, self._stream(stream), N.dptr(acc)),
                "s2d_view_stats_accumulate")

    def set_timing(self, enable: bool):
        N.check(N.lib().s2d_view_set_timing(self.handle, int(bool(enable))), "s2d_view_set_timing")

    PHASES = ("project", "depth_sort", "tile_bin", "raster_fwd", "raster_bwd", "project_bwd")

    def timing(self, reset: bool = True) -> dict:
        """Accumulated per-phase milliseconds (synchronises)."""
        out = (ctypes.c_double * 8)()
        N.check(N.lib().s2d_view_timing(self.handle, out, int(reset)), "s2d_view_timing")
        d = {k: out[i] for i, k in enumerate(self.PHASES)}
        d["n_forward"] = int(out[6])
        d["n_backward"] = int(out[7])
        return d

    def reserve_pairs(self, pairs: int):
        N.check(N.lib().s2d_view_reserve_pairs(self.handle, int(pairs)), "s2d_view_reserve_pairs")

    def inspect(self) -> dict:
        """Copies of the last forward's depth order, tile lists, bboxes, depths and flags."""
        d = N.ViewDebug()
        N.check(N.lib().s2d_view_inspect(self.handle, ctypes.byref(d)), "s2d_view_inspect")
        st = self.stats()
        n, h, w = self._last
        dev = self.device
        v, p = d.drawn, st.pairs_stored
        out = {
            "order": _wrap(d.order, (v,), "<i4", dev).clone(),  # drawn surfels (non-empty bbox)
            "pair_tiles": _wrap(d.pair_tiles, (p,), "<i4", dev).clone() & 0xFFFF,  # low 16 bits: tile id
            "pair_ids": _wrap(d.pair_ids, (p,), "<i4", dev).clone(),
            "ranges": _wrap(d.ranges, (d.ntiles, 2), "<i4", dev).clone(),
            "bbox": _wrap(d.bbox, (n, 4), "<i2", dev).clone() if n else torch.zeros((0, 4), dtype=torch.int16),
            "z": _wrap(d.z, (n,), "<f8", dev).clone() if n else torch.zeros(0, dtype=torch.float64),
            "flags": _wrap(d.flags, (n,), "|u1", dev).clone() if n else torch.zeros(0, dtype=torch.uint8),
            "records": _wrap(d.records, (n, 16), "<f4", dev).clone() if n else torch.zeros((0, 16)),
            "pixel_state": _wrap(d.pixel_state, (h * w, 2), "<i4", dev).clone(),
            "stream_lengths": _wrap(d.stream_lengths, (d.ntiles, 8, 2), "<i4", dev).clone(),
            "streams": _wrap(d.streams, (16 * p, 4), "<i4", dev).clone() if p else None,
            "tiles_x": d.tiles_x,
            "stats": st,
        }
        return out


def forward_checked(view: View, params, n, pose, cam, cfg, image, max_all=None, max_marked=None,
                    mask=None) -> N.ViewStats:
    """Forward + synchronous stats read; grows the pair capacity and re-runs on overflow."""
    for _ in range(4):
        if max_all is not None:
            max_all.zero_()
        if max_marked is not None:
            max_marked.zero_()
        view.forward(params, n, pose, cam, cfg, image, max_all, max_marked, mask)
        st = view.stats()
        if not st.overflow:
            return st
        view.reserve_pairs(st.pairs + st.pairs // 4 + 4096)
    raise RuntimeError("pair capacity could not be sized")  # pragma: no cover
