"""Drop-in for ``sparse_sampler.pyramid`` (reference pkg/src/sparse_sampler/pyramid.py)
computed by the sm_100a kernels.

Same names, signatures, array layouts (HWC float64) and ValueError behaviour
as the reference; the work runs on the GPU through libssb200.  ``LEVELS`` is
read at call time, like the reference (pyramid.py:24); kernel fields of any
level count and of kernel size k in {3, 5, 7} (inferred from the coarsest
level's k*k channels) are accepted.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .. import ops
from . import _dev, _types
from ._types import DemodMap, PyramidGrads, PyramidStack  # noqa: F401  (re-exported)

LEVELS = 5
DENOISE_TAPS = 25
UPSAMPLE_TAPS = 4
TEMPORAL_TAPS = 25
DEMOD_FLOOR = 1e-3
OFFSETS5 = [(dy, dx) for dy in range(-2, 3) for dx in range(-2, 3)]
_levels_source = None  # set by install(): read LEVELS from the reference module


def _levels() -> int:
    return _levels_source.LEVELS if _levels_source is not None else LEVELS


def level_dims(width: int, height: int) -> list[tuple[int, int]]:
    """ref pyramid.py:33-38"""
    return ops.level_shapes(height, width, _levels())


def kernel_channels(level: int) -> int:
    """ref pyramid.py:41-46 (the reference layout always carries the
    temporal group at level 0)."""
    if level == 0:
        return DENOISE_TAPS + UPSAMPLE_TAPS + TEMPORAL_TAPS
    if level < _levels() - 1:
        return DENOISE_TAPS + UPSAMPLE_TAPS
    return DENOISE_TAPS


@dataclass
class KernelField:
    """Per-level, per-pixel kernel logits (ref pyramid.py:49-75)."""

    logits: list

    def __post_init__(self):
        if len(self.logits) != _levels():
            raise ValueError(f"kernel field needs {_levels()} levels")
        self.logits = [np.asarray(l, dtype=np.float64) for l in self.logits]
        h, w = self.logits[0].shape[:2]
        for l, (dims, arr) in enumerate(zip(level_dims(w, h), self.logits)):
            expect = (dims[0], dims[1], kernel_channels(l))
            if arr.shape != expect:
                raise ValueError(f"level {l} logits must have shape {expect}, got {arr.shape}")

    @property
    def width(self) -> int:
        return self.logits[0].shape[1]

    @property
    def height(self) -> int:
        return self.logits[0].shape[0]


def zero_kernel_field(width: int, height: int) -> KernelField:
    return KernelField([np.zeros((h, w, kernel_channels(l)))
                        for l, (h, w) in enumerate(level_dims(width, height))])


def _geometry(logits) -> tuple[int, int]:
    L = len(logits)
    k2 = np.asarray(logits[-1]).shape[-1]
    k = int(round(np.sqrt(k2)))
    if L < 2 or k * k != k2 or k not in (3, 5, 7):
        raise ValueError("kernel field must have >= 2 levels and k*k logits (k in 3, 5, 7) "
                         "at the coarsest level")
    return L, k


def _level0_active(k: int, L: int, temporal: bool) -> int:
    return k * k + (4 if L > 1 else 0) + (k * k if temporal else 0)


def normalize_kernels(kf, include_temporal: bool = True) -> list[np.ndarray]:
    """Joint per-pixel softmax per level (ref pyramid.py:93-109)."""
    L, k = _geometry(kf.logits)
    out = []
    for l, z in enumerate(kf.logits):
        z = np.asarray(z, dtype=np.float64)
        active = z.shape[-1]
        if l == 0 and not include_temporal:
            active = min(active, _level0_active(k, L, False))
        w = ops.softmax_channels(_dev.to_planar(z), active=active)
        out.append(_dev.to_hwc(w))
    return out


def build_pyramid(noisy) -> PyramidStack:
    """Low-pass pyramid by iterated count-correct 2x2 pooling (ref :159-166)."""
    data = noisy.data if hasattr(noisy, "data") and not isinstance(noisy, np.ndarray) else noisy
    t = _dev.to_planar(data)
    return _types.make("PyramidStack", [_dev.to_hwc(x) for x in ops.build_pyramid(t, _levels())])


def gather5(image: np.ndarray, weights: np.ndarray) -> np.ndarray:
    """k x k clamp-to-edge gather; weights (H, W, k*k) (ref :184-187)."""
    weights = np.asarray(weights, dtype=np.float64)
    k = int(round(np.sqrt(weights.shape[-1])))
    if k * k != weights.shape[-1]:
        raise ValueError("gather weights need k*k channels")
    return _dev.to_hwc(ops.gather(_dev.to_planar(image), _dev.to_planar(weights), k))


def upsample2(coarse: np.ndarray, weights: np.ndarray) -> np.ndarray:
    """2x2 learned upsample, clamped parents (ref :234-241)."""
    return _dev.to_hwc(ops.upsample2(_dev.to_planar(coarse), _dev.to_planar(weights)))


@dataclass
class ReconTape:
    """Opaque device tape (callers only pass it back, ref pyramid.py:264-281)."""
    dev: ops.PyramidTape
    k: int
    levels: int
    temporal: bool
    ref_channels: list
    channels: int


def reconstruct_core(noisy: np.ndarray, kf, prev_warped: np.ndarray | None = None,
                     demod: np.ndarray | None = None):
    """Coarse-to-fine reconstruction; returns (out, tape) (ref :292-345).

    Any channel count C (all channels share the kernels)."""
    noisy = np.asarray(noisy, dtype=np.float64)
    if noisy.ndim != 3:
        raise ValueError("noisy must be (H, W, C)")
    logits = kf.logits
    L, k = _geometry(logits)
    h, w, c = noisy.shape
    shapes = ops.level_shapes(h, w, L)
    temporal = prev_warped is not None
    dev_logits = []
    for l, (z, (hl, wl)) in enumerate(zip(logits, shapes)):
        z = np.asarray(z, dtype=np.float64)
        if z.shape[:2] != (hl, wl):
            raise ValueError(f"level {l} logits do not match the input size")
        need = ops.logit_channels(l, L, k, has_prev=temporal)
        if l == 0:
            if z.shape[-1] < need:
                raise ValueError("level-0 logits lack the temporal group")
            # the unread temporal group is dropped on the device: the caller's
            # contiguous array crosses PCIe as it lies (no host-side copy)
            dev_logits.append(_dev.to_planar(z)[:, :need].contiguous())
            continue
        elif z.shape[-1] != need:
            raise ValueError(f"level {l} logits must carry {need} channels")
        dev_logits.append(_dev.to_planar(z))
    n = _dev.to_planar(noisy)
    dm = _dev.to_planar(demod) if demod is not None else None
    pv = _dev.to_planar(prev_warped) if temporal else None
    for name, arr in (("demod", demod), ("prev_warped", prev_warped)):
        if arr is not None and np.shape(arr) != noisy.shape:
            raise ValueError(f"{name} must match the input's shape")
    out, tape = ops.pyramid_forward(n, dev_logits, dm, pv, ksize=k)
    ref_ch = [np.asarray(z).shape[-1] for z in logits]
    return _dev.to_hwc(out), ReconTape(tape, k, L, temporal, ref_ch, c)


def reconstruct(pyr, kf, prev_warped=None, demod=None):
    """Filter surface returning a clamped RadianceImage (ref :348-359)."""
    prev = prev_warped.data if prev_warped is not None else None
    dem = demod.values if demod is not None else None
    out, _ = reconstruct_core(pyr.levels[0], kf, prev, dem)
    return _types.make("RadianceImage", np.maximum(out, 0.0))


def reconstruct_backward(tape: ReconTape, upstream: np.ndarray,
                         want_param_grads: bool = True):
    """Exact gradients of sum(upstream * out) (ref :362-449)."""
    up = np.asarray(upstream, dtype=np.float64)
    g = ops.pyramid_backward(tape.dev, _dev.to_planar(up), want_param_grads=want_param_grads)
    torch.cuda.synchronize()
    glogits = None
    if want_param_grads:
        glogits = []
        for l, gz in enumerate(g.logits):
            if gz.shape[1] != tape.ref_channels[l]:
                # the reference layout's (zero) temporal gradients, padded on the device
                full = torch.zeros((1, tape.ref_channels[l]) + tuple(gz.shape[2:]), dtype=gz.dtype,
                                   device=gz.device)
                full[:, :gz.shape[1]] = gz
                gz = full
            glogits.append(_dev.to_hwc(gz))
    gdemod = _dev.to_hwc(g.demod) if g.demod is not None else None
    gprev = _dev.to_hwc(g.prev) if g.prev is not None else None
    return _types.make("PyramidGrads", logits=glogits, demod=gdemod, input=_dev.to_hwc(g.input),
                       prev=gprev)
