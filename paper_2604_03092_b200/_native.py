"""ctypes binding of ``lib/libsurfel2d.so`` (the C ABI in ``include/surfel2d.h``).

There is no CPU fallback: if the library is missing or cannot be loaded, every
entry point raises :class:`NativeLibraryError`.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_2604_03092_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("S2D_LIB_PATH") or os.path.join(_HERE, "lib", "libsurfel2d.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "surfel2d.h")

S2D_OK = 0
SPLAT_AFFINE = 0
SPLAT_RAY = 1
S2D_ERR_INVALID = 1
S2D_ERR_CUDA = 2
S2D_ERR_OOM = 3
S2D_ERR_STATE = 4

LOSS_MSE = 0
LOSS_L1 = 1
LOSS_EXTERNAL = 2

c_p = ctypes.c_void_p


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or failed to load (no CPU fallback exists)."""


class Camera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class RasterCfg(ctypes.Structure):
    _fields_ = [("weight_clamp", ctypes.c_double), ("termination_transmittance", ctypes.c_double),
                ("footprint_sigma", ctypes.c_double), ("near_plane", ctypes.c_double),
                ("max_condition", ctypes.c_double), ("max_view_angle_deg", ctypes.c_double),
                ("center_margin_frac", ctypes.c_double), ("splat_mode", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class Image(ctypes.Structure):
    _fields_ = [("color", c_p), ("depth", c_p), ("accumulation", c_p), ("normal", c_p),
                ("max_w", c_p), ("arg_w", c_p)]


class ViewStats(ctypes.Structure):
    _fields_ = [("visible", ctypes.c_int32), ("pairs", ctypes.c_int32),
                ("degenerate", ctypes.c_int32), ("n_mask", ctypes.c_int32),
                ("overflow", ctypes.c_int32), ("guard_hits", ctypes.c_int32),
                ("pairs_stored", ctypes.c_int32), ("blended", ctypes.c_int32)]


class ViewDebug(ctypes.Structure):
    _fields_ = [("order", c_p), ("pair_tiles", c_p), ("pair_ids", c_p), ("ranges", c_p),
                ("bbox", c_p), ("z", c_p), ("flags", c_p), ("records", c_p),
                ("pixel_state", c_p), ("ntiles", ctypes.c_int32), ("tiles_x", ctypes.c_int32),
                ("pair_capacity", ctypes.c_int64), ("drawn", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("stream_lengths", c_p), ("streams", c_p)]


class Loss(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("depth_mask", ctypes.c_int32),
                ("w_rgb", ctypes.c_double), ("w_depth", ctypes.c_double),
                ("target_rgb", c_p), ("target_depth", c_p), ("d_color", c_p), ("d_depth", c_p),
                ("d_normal", c_p), ("d_accumulation", c_p)]


class AdamCfg(ctypes.Structure):
    _fields_ = [("lr_means", ctypes.c_double), ("lr_rest", ctypes.c_double),
                ("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("eps", ctypes.c_double),
                ("scale_min", ctypes.c_double)]


_lib = None
_load_error = None

_SIGNATURES = {
    "s2d_last_error": (ctypes.c_char_p, []),
    "s2d_version": (ctypes.c_int32, []),
    "s2d_ctx_create": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(c_p)]),
    "s2d_ctx_destroy": (ctypes.c_int, [c_p]),
    "s2d_view_create": (ctypes.c_int, [c_p, ctypes.POINTER(c_p)]),
    "s2d_view_destroy": (ctypes.c_int, [c_p]),
    "s2d_view_stats_device": (ctypes.c_int, [c_p, ctypes.POINTER(c_p)]),
    "s2d_view_stats_host": (ctypes.c_int, [c_p, ctypes.POINTER(ViewStats)]),
    "s2d_view_stats_accumulate": (ctypes.c_int, [c_p, c_p, c_p]),
    "s2d_view_reserve_pairs": (ctypes.c_int, [c_p, ctypes.c_int64]),
    "s2d_view_set_layout": (ctypes.c_int, [c_p, ctypes.c_int64]),
    "s2d_view_inspect": (ctypes.c_int, [c_p, ctypes.POINTER(ViewDebug)]),
    "s2d_launch_count": (ctypes.c_int64, []),
    "s2d_view_set_timing": (ctypes.c_int, [c_p, ctypes.c_int32]),
    "s2d_view_timing": (ctypes.c_int, [c_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32]),
    "s2d_pose_inverse": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "s2d_forward": (ctypes.c_int, [c_p, c_p, c_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(Camera), ctypes.POINTER(RasterCfg),
                                   ctypes.POINTER(Image), c_p, c_p, c_p]),
    "s2d_backward": (ctypes.c_int, [c_p, c_p, c_p, ctypes.c_int64, ctypes.POINTER(Image),
                                    ctypes.POINTER(Loss), c_p, c_p]),
    "s2d_forward_backward": (ctypes.c_int, [c_p, c_p, c_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(Camera), ctypes.POINTER(RasterCfg),
                                            ctypes.POINTER(Image), ctypes.POINTER(Loss), c_p, c_p, c_p]),
    "s2d_adam_step": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_p, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.POINTER(AdamCfg), c_p]),
    "s2d_adam_step_gated": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_p, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.POINTER(AdamCfg), c_p, c_p]),
    "s2d_render_host": (ctypes.c_int, [c_p, c_p] + [c_p] * 5 + [ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                                           ctypes.POINTER(Camera), ctypes.POINTER(RasterCfg)]
                        + [c_p] * 4 + [ctypes.POINTER(ctypes.c_int32)]),
    "s2d_refine_gd": (ctypes.c_int, [c_p, c_p, c_p, c_p, ctypes.c_int64, ctypes.c_double, c_p]),
    "s2d_refine_gnorm": (ctypes.c_int, [c_p, c_p, ctypes.c_int64, c_p, c_p]),
    "s2d_transform_surfels": (ctypes.c_int, [c_p, ctypes.POINTER(ctypes.c_double), c_p, ctypes.c_int64, c_p]),
    "s2d_fuse_gate": (ctypes.c_int, [c_p, c_p, ctypes.POINTER(Camera), c_p, ctypes.c_int64, ctypes.c_double, c_p]),
    "s2d_prune_mark": (ctypes.c_int, [c_p] * 6 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double, c_p]),
    "s2d_prune_keep": (ctypes.c_int, [c_p, c_p, ctypes.c_int64, ctypes.c_double, c_p]),
}


def lib():
    """The loaded CUDA library; raises NativeLibraryError if unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not found: build the CUDA extension first (__graft_entry__.build()); "
            "there is no CPU fallback")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - environment dependent
        _load_error = e
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    old_ok = os.environ.get("S2D_ALLOW_OLD_LIB") == "1"  # A/B runs against an older build only
    for name, (res, args) in _SIGNATURES.items():
        if old_ok and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def header_functions():
    """Names of the functions declared in include/surfel2d.h."""
    with open(HEADER_PATH) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(s2d_\w+)\s*\(", text, flags=re.M)))


def check(rc: int, what: str = "") -> None:
    if rc == S2D_OK:
        return
    msg = lib().s2d_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == S2D_ERR_INVALID:
        raise ValueError(text)
    if rc == S2D_ERR_OOM:
        raise MemoryError(text)
    raise RuntimeError(text)


def dptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def as_doubles(a):
    import numpy as np
    arr = (ctypes.c_double * len(a))(*[float(x) for x in np.asarray(a, dtype=float).reshape(-1)])
    return arr
