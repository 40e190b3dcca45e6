"""Drop-in for ``sparse_sampler.tonemap`` (reference pkg/src/sparse_sampler/
tonemap.py:87-118) on the GPU: tonemap_array and tonemap_backward, HWC float64
numpy in and out; the TmoParams container is the reference's (any object with
exposure / contrast / saturation / toe / shoulder)."""

from __future__ import annotations

import numpy as np

from .. import ops
from . import _dev


def _params(p):
    return (p.exposure, p.contrast, p.saturation, p.toe, p.shoulder)


def _rows(a):
    """(..., 3) -> (1, N, 3): the operator is per pixel over the last (RGB)
    axis, so any leading shape -- (H, W, 3) images, the (K, H, W, 3) seed
    batches of estimators.EstimatorLossPipeline and the (H, W, K, 3) stacks of
    optimize._chain_forward_batch -- runs as one row of N pixels."""
    if a.ndim < 1 or a.shape[-1] != 3:
        raise ValueError("tonemap: radiance must be (..., 3) RGB")
    return a.reshape(1, -1, 3)


def tonemap_array(radiance, p):
    rad = np.asarray(radiance, dtype=np.float64)
    out = _dev.to_hwc(ops.tonemap(_dev.to_planar(_rows(rad)), _params(p)))
    return out.reshape(rad.shape)


def tonemap_backward(radiance, p, upstream):
    rad = np.asarray(radiance, dtype=np.float64)
    up = np.asarray(upstream, dtype=np.float64)
    if up.shape != rad.shape:
        up = np.broadcast_to(up, np.broadcast_shapes(up.shape, rad.shape))
        rad = np.broadcast_to(rad, up.shape)
    g = ops.tonemap_backward(_dev.to_planar(_rows(rad)), _params(p), _dev.to_planar(_rows(up)))
    return _dev.to_hwc(g).reshape(rad.shape)
