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


def tonemap_array(radiance, p):
    rad = np.asarray(radiance, dtype=np.float64)
    return _dev.to_hwc(ops.tonemap(_dev.to_planar(rad), _params(p)))


def tonemap_backward(radiance, p, upstream):
    rad = np.asarray(radiance, dtype=np.float64)
    up = np.asarray(upstream, dtype=np.float64)
    if up.shape != rad.shape:
        raise ValueError("tonemap_backward: upstream must match the radiance")
    return _dev.to_hwc(ops.tonemap_backward(_dev.to_planar(rad), _params(p), _dev.to_planar(up)))
