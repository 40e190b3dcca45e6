"""Drop-in for the temporal warp of ``sparse_sampler.images``
(reference pkg/src/sparse_sampler/images.py:88-147) on the GPU.

warp_array(prev, motion) -> (out, validity) and warp_backward(grad_out,
motion) -> grad_prev, HWC float64 numpy in and out like the reference.  The
transpose is a deterministic gather in the reference's own summation order,
so in the default float64 precision both match the reference bit for bit.
"""

from __future__ import annotations

import numpy as np

from .. import ops
from . import _dev


def _check(img, motion):
    img, motion = np.asarray(img, dtype=np.float64), np.asarray(motion, dtype=np.float64)
    if img.shape[:2] != motion.shape[:2]:
        raise ValueError("warp: image and motion dimensions must match")
    if motion.ndim != 3 or motion.shape[2] != 2:
        raise ValueError("motion must be (H, W, 2)")
    return img, motion


def warp_array(prev, motion):
    prev, motion = _check(prev, motion)
    squeeze = prev.ndim == 2
    out, val = ops.warp(_dev.to_planar(prev), _dev.to_planar(motion))
    out = _dev.to_hwc(out)
    return (out[:, :, 0] if squeeze else out), _dev.to_host(val[0]).astype(np.float64)


def warp_backward(grad_out, motion):
    grad_out, motion = _check(grad_out, motion)
    squeeze = grad_out.ndim == 2
    g = _dev.to_hwc(ops.warp_backward(_dev.to_planar(grad_out), _dev.to_planar(motion)))
    return g[:, :, 0] if squeeze else g
