"""ctypes binding of libssb200.so (the C ABI declared in include/ssb_api.h).

The library is built in-tree (``python -m paper_2602_08642_b200.build``) and
loaded from ``paper_2602_08642_b200/lib/``.  There is no fallback: if the
library is missing or fails to load, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

SSB_MAX_LEVELS = 8
SSB_F32, SSB_BF16, SSB_F64 = 0, 1, 2
SSB_BLEND_NATIVE, SSB_BLEND_TIED = 0, 1
RULES = {"stochastic": 0, "relaxed": 1, "gumbel": 2}
VARIANTS = {"stochastic": 0, "relaxed": 1, "straight-through": 2, "gumbel": 3}
SSB_EUNSUPPORTED = -3  # ssb_api.h

# every symbol include/ssb_api.h declares (tests check the .so exports them all)
EXPORTS = (
    "ssb_version", "ssb_last_error", "ssb_launch_count", "ssb_set_launch_events",
    "ssb_pyr_logit_channels", "ssb_pyr_level_dims", "ssb_pyr_tape_bytes",
    "ssb_pyr_workspace_bytes", "ssb_pyr_forward", "ssb_pyr_backward",
    "ssb_softmax_channels", "ssb_gather", "ssb_upsample2", "ssb_avgpool2",
    "ssb_uniform_grid", "ssb_uniform_at", "ssb_density_workspace_bytes", "ssb_normalize_density",
    "ssb_allocate", "ssb_stochastic_core", "ssb_estimate", "ssb_place_fused", "ssb_place",
    "ssb_warp", "ssb_warp_backward_workspace_bytes", "ssb_warp_backward",
    "ssb_score_grad_workspace_bytes", "ssb_score_grad",
    "ssb_tonemap", "ssb_tonemap_backward", "ssb_losses_workspace_bytes", "ssb_losses", "ssb_epilogue",
    "ssb_pyr_forward_level", "ssb_pool2_strided", "ssb_halo_put", "ssb_flag_wait", "ssb_enable_peer",
    "ssb_infer_small_workspace_bytes", "ssb_infer_small",
)

vp = C.c_void_p


class PyrDesc(C.Structure):
    _fields_ = [("batch", C.c_int32), ("channels", C.c_int32), ("height", C.c_int32),
                ("width", C.c_int32), ("levels", C.c_int32), ("ksize", C.c_int32),
                ("image_dtype", C.c_int32), ("logit_dtype", C.c_int32),
                ("has_prev", C.c_int32), ("has_demod", C.c_int32),
                ("blend_mode", C.c_int32), ("reserved", C.c_int32)]


class PyrFwdIO(C.Structure):
    _fields_ = [("noisy", vp), ("demod", vp), ("prev", vp),
                ("logits", vp * SSB_MAX_LEVELS), ("out", vp)]


class PyrBwdIO(C.Structure):
    _fields_ = [("noisy", vp), ("demod", vp), ("prev", vp),
                ("logits", vp * SSB_MAX_LEVELS), ("out", vp), ("upstream", vp),
                ("g_logits", vp * SSB_MAX_LEVELS), ("g_noisy", vp), ("g_demod", vp),
                ("g_prev", vp), ("accumulate_logits", C.c_int32), ("reserved", C.c_int32)]


class AllocDesc(C.Structure):
    _fields_ = [("B", C.c_int32), ("H", C.c_int32), ("W", C.c_int32), ("rule", C.c_int32),
                ("dithered", C.c_int32), ("mask_size", C.c_int32), ("seed", C.c_uint64),
                ("frame0", C.c_int64), ("gumbel_temp", C.c_double)]


class EstimateDesc(C.Structure):
    _fields_ = [("B", C.c_int32), ("H", C.c_int32), ("W", C.c_int32), ("variant", C.c_int32),
                ("capacity", C.c_int32), ("reserved", C.c_int32), ("lam", C.c_double),
                ("gumbel_temp", C.c_double), ("density_floor", C.c_double)]


class PlaceDesc(C.Structure):
    _fields_ = [("B", C.c_int32), ("H", C.c_int32), ("W", C.c_int32), ("capacity", C.c_int32),
                ("variant", C.c_int32), ("reserved", C.c_int32), ("seed", C.c_uint64),
                ("frame0", C.c_int64), ("budget", C.c_double)]


class PyrLevelDesc(C.Structure):
    _fields_ = [("batch", C.c_int32), ("channels", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("ksize", C.c_int32), ("image_dtype", C.c_int32), ("logit_dtype", C.c_int32),
                ("blend_mode", C.c_int32), ("has_coarse", C.c_int32), ("coarse_height", C.c_int32),
                ("coarse_width", C.c_int32), ("reserved", C.c_int32)]


class PlaceCfg(C.Structure):
    _fields_ = [("lam", C.c_double), ("gumbel_temp", C.c_double), ("density_floor", C.c_double)]


class PlaceIO(C.Structure):
    _fields_ = [("scores", C.c_void_p), ("bank", C.c_void_p), ("noisy", C.c_void_p), ("grad", C.c_void_p),
                ("spp", C.c_void_p), ("taken", C.c_void_p), ("drawn", C.c_void_p)]


class SSBError(RuntimeError):
    pass


_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    # SSB_LIB_PATH: an alternative build of the library (A/B measurements of
    # two builds on one box; symbols it lacks are left unbound)
    return os.environ.get("SSB_LIB_PATH") or _build.LIB


def load(build_if_missing: bool = False):
    """Load libssb200.so (once).  Raises if it is absent: no CPU fallback."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            if not build_if_missing:
                raise SSBError(f"libssb200.so not built ({path}); run "
                               "`python -m paper_2602_08642_b200.build`")
            _build.build()
        lib = C.CDLL(path)
        P = C.POINTER
        sigs = {
            "ssb_version": (C.c_int, []),
            "ssb_last_error": (C.c_char_p, []),
            "ssb_launch_count": (C.c_ulonglong, []),
            "ssb_set_launch_events": (C.c_int, [vp, C.c_int, P(C.c_int)]),
            "ssb_pyr_logit_channels": (C.c_int, [P(PyrDesc), C.c_int]),
            "ssb_pyr_level_dims": (C.c_int, [P(PyrDesc), C.c_int, P(C.c_int32), P(C.c_int32)]),
            "ssb_pyr_tape_bytes": (C.c_int, [P(PyrDesc), P(C.c_size_t)]),
            "ssb_pyr_workspace_bytes": (C.c_int, [P(PyrDesc), P(C.c_size_t)]),
            "ssb_pyr_forward": (C.c_int, [P(PyrDesc), P(PyrFwdIO), vp, vp]),
            "ssb_pyr_backward": (C.c_int, [P(PyrDesc), P(PyrBwdIO), vp, vp, vp]),
            "ssb_softmax_channels": (C.c_int, [C.c_int] * 6 + [vp, vp, vp]),
            "ssb_gather": (C.c_int, [C.c_int] * 6 + [vp, vp, vp, vp]),
            "ssb_upsample2": (C.c_int, [C.c_int] * 7 + [vp, vp, vp, vp]),
            "ssb_avgpool2": (C.c_int, [C.c_int] * 5 + [vp, vp, vp]),
            "ssb_uniform_grid": (C.c_int, [C.c_uint64, C.c_int64, vp, C.c_int, C.c_int, C.c_int,
                                           C.c_uint64, vp, vp]),
            "ssb_uniform_at": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, vp, vp]),
            "ssb_density_workspace_bytes": (C.c_int, [C.c_int, C.c_int, C.c_int, P(C.c_size_t)]),
            "ssb_normalize_density": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, C.c_double, vp,
                                                vp, vp]),
            "ssb_allocate": (C.c_int, [P(AllocDesc), vp, vp, vp, vp, vp, vp, vp]),
            "ssb_stochastic_core": (C.c_int, [P(EstimateDesc)] + [vp] * 10),
            "ssb_estimate": (C.c_int, [P(EstimateDesc)] + [vp] * 11),
            "ssb_place_fused": (C.c_int, [P(PlaceDesc)] + [vp] * 7),
            "ssb_place": (C.c_int, [P(PlaceDesc), P(PlaceCfg), P(PlaceIO), vp, vp]),
            "ssb_infer_small_workspace_bytes": (C.c_int, [C.c_int] * 4 + [P(C.c_size_t)]),
            "ssb_infer_small": (C.c_int, [P(PlaceDesc), vp, vp, vp, C.c_int, C.c_int, vp, vp, vp, vp, vp]),
            "ssb_pyr_forward_level": (C.c_int, [P(PyrLevelDesc)] + [vp] * 6),
            "ssb_pool2_strided": (C.c_int, [C.c_int] * 5 + [vp, C.c_longlong, C.c_longlong, vp, vp,
                                                             C.c_longlong, C.c_longlong, vp]),
            "ssb_halo_put": (C.c_int, [vp, C.c_longlong, vp, C.c_longlong, C.c_int, C.c_int, C.c_int,
                                       C.c_int, vp, C.c_int, vp]),
            "ssb_flag_wait": (C.c_int, [vp, C.c_int, vp]),
            "ssb_enable_peer": (C.c_int, [C.c_int, C.c_int]),
            "ssb_warp": (C.c_int, [C.c_int] * 5 + [vp] * 5),
            "ssb_warp_backward_workspace_bytes": (C.c_int, [C.c_int, C.c_int, C.c_int, P(C.c_size_t)]),
            "ssb_warp_backward": (C.c_int, [C.c_int] * 5 + [vp] * 5),
            "ssb_score_grad_workspace_bytes": (C.c_int, [C.c_int] * 3 + [P(C.c_size_t)]),
            "ssb_score_grad": (C.c_int, [C.c_int] * 6 + [vp, vp, vp, C.c_double, C.c_double,
                                                         vp, vp, vp]),
            "ssb_tonemap": (C.c_int, [C.c_int] * 4 + [P(C.c_double)] + [vp] * 3),
            "ssb_tonemap_backward": (C.c_int, [C.c_int] * 4 + [P(C.c_double)] + [vp] * 4),
            "ssb_losses_workspace_bytes": (C.c_int, [C.c_int, P(C.c_size_t)]),
            "ssb_losses": (C.c_int, [C.c_int] * 4 + [vp] * 14),
            "ssb_epilogue": (C.c_int, [C.c_int] * 4 + [P(C.c_double)] + [vp] * 12),
        }
        alt = bool(os.environ.get("SSB_LIB_PATH"))
        for name, (res, args) in sigs.items():
            if alt and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str) -> int:
    if rc < 0:
        msg = load().ssb_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise SSBError(f"{what} failed ({rc}): {msg}")
    return rc
