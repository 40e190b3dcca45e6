"""Drop-in for the training losses of ``sparse_sampler.losses`` (reference
pkg/src/sparse_sampler/losses.py:58-91) on the GPU: spatial_loss,
temporal_loss, combined_loss with the reference's signatures, validation and
return values; plus ``loss_gradients`` (the inline gradient of
optimize.evaluate_step, optimize.py:219-231).  MaskImage objects are accepted
(anything with ``.weights``)."""

from __future__ import annotations

import numpy as np

from .. import ops
from . import _dev

TEMPORAL_WEIGHT = 1.25


def _img(a):
    return _dev.to_planar(np.asarray(a, dtype=np.float64))


def _map(a):
    return _dev.to_dev(np.asarray(a, dtype=np.float64)[None], _dev.dtype())


def spatial_loss(out, ref, mask):
    out, ref = np.asarray(out, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    if out.shape != ref.shape:
        raise ValueError("spatial loss: image dimensions must match")
    r = ops.losses(_img(out), _img(ref), mask=_map(mask.weights))
    return _dev.to_host(r["spatial_map"][0]).astype(np.float64), float(r["losses"][0, 0])


def temporal_loss(out_t, out_warped_prev, ref_t, ref_warped_prev, validity=None):
    arrs = [np.asarray(a, dtype=np.float64) for a in (out_t, out_warped_prev, ref_t, ref_warped_prev)]
    for a in arrs[1:]:
        if a.shape != arrs[0].shape:
            raise ValueError("temporal loss: image dimensions must match")
    r = ops.losses(_img(arrs[0]), _img(arrs[2]), _img(arrs[1]), _img(arrs[3]),
                   validity=None if validity is None else _map(validity))
    return _dev.to_host(r["temporal_map"][0]).astype(np.float64), float(r["losses"][0, 1])


def combined_loss(spatial_map, temporal_map):
    spatial_map = np.asarray(spatial_map, dtype=np.float64)
    temporal_map = np.asarray(temporal_map, dtype=np.float64)
    if spatial_map.shape != temporal_map.shape:
        raise ValueError("combined loss: map dimensions must match")
    per_pixel = np.maximum(TEMPORAL_WEIGHT * temporal_map, spatial_map)  # host: an elementwise max
    return per_pixel, float(per_pixel.mean())


def loss_gradients(ldr1, ref, ldr0_w, ref_w, validity, mask):
    """(g_ldr1, g_ldr0_w) of the combined loss as optimize.py:219-231 forms them."""
    r = ops.losses(_img(ldr1), _img(ref), _img(ldr0_w), _img(ref_w), validity=_map(validity),
                   mask=_map(mask.weights), want_maps=False, want_grads=True)
    return _dev.to_hwc(r["g_ldr1"]), _dev.to_hwc(r["g_ldr0_w"])
