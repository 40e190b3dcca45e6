"""Tonemap and training losses -- CPU oracle (test-only).

Restates `pkg/src/sparse_sampler/tonemap.py` (`log_augment` :36-43,
`filmic` :45-57, `filmic_derivative` :60-69, `srgb_encode` :72-78,
`srgb_derivative` :81-84, `tonemap_array` :87-88, `tonemap_backward`
:95-118) and `losses.py` (`spatial_loss` :58-64, `temporal_loss` :67-83,
`combined_loss` :86-91), plus the loss gradients exactly as
`optimize.evaluate_step` forms them (`optimize.py:219-231`).  Images are
(H, W, 3) float64; maps (H, W).
"""

from __future__ import annotations

import numpy as np

LOG_FLOOR = 1e-8
TEMPORAL_WEIGHT = 1.25


def log_augment(rad, exposure, contrast, saturation):
    c = np.log(np.maximum(rad, LOG_FLOOR))
    m = c.mean(axis=-1, keepdims=True)
    return contrast * (m + saturation * (c - m) + exposure)


def filmic(x, toe, shoulder):
    out = 0.5 * (1.0 + x)
    out = np.where(x < toe - 1.0, 0.5 * toe * np.exp(np.minimum((x + 1.0 - toe) / toe, 0.0)), out)
    return np.where(x >= 1.0 - shoulder,
                    1.0 - 0.5 * shoulder * np.exp(np.minimum(-(x + shoulder - 1.0) / shoulder, 0.0)), out)


def filmic_derivative(x, toe, shoulder):
    d = np.full(x.shape, 0.5)
    d = np.where(x < toe - 1.0, 0.5 * np.exp(np.minimum((x + 1.0 - toe) / toe, 0.0)), d)
    return np.where(x >= 1.0 - shoulder, 0.5 * np.exp(np.minimum(-(x + shoulder - 1.0) / shoulder, 0.0)), d)


def srgb_encode(v):
    return np.where(v <= 0.0031308, v * 12.92, 1.055 * np.power(np.clip(v, 0.0, None), 1.0 / 2.4) - 0.055)


def srgb_derivative(v):
    return np.where(v <= 0.0031308, 12.92, (1.055 / 2.4) * np.power(np.clip(v, 1e-300, None), 1.0 / 2.4 - 1.0))


def tonemap(rad, tmo):
    """tmo = (exposure, contrast, saturation, toe, shoulder)."""
    e, c, s, toe, sh = tmo
    return srgb_encode(filmic(log_augment(rad, e, c, s), toe, sh))


def tonemap_backward(rad, tmo, up):
    e, c, s, toe, sh = tmo
    x = log_augment(rad, e, c, s)
    y = filmic(x, toe, sh)
    gx = up * srgb_derivative(y) * filmic_derivative(x, toe, sh)
    gc = c * (s * gx + (1.0 - s) / 3.0 * gx.sum(axis=-1, keepdims=True))
    return np.where(rad > LOG_FLOOR, gc / np.maximum(rad, LOG_FLOOR), 0.0)


def losses(ldr1, ref, ldr0_w=None, ref_w=None, validity=None, mask=None):
    """(sp_map, tm_map, cb_map, (sp, tm, cb)) like losses.py; tm_map = 0
    without a history frame."""
    w = np.ones(ldr1.shape[:2]) if mask is None else mask
    sp_map = np.abs(ldr1 - ref).mean(axis=-1) * w
    sp = float(sp_map.mean())
    if ldr0_w is None:
        tm_map, tm = np.zeros(ldr1.shape[:2]), 0.0
    else:
        delta = (ldr1 - ldr0_w) - (ref - ref_w)
        tm_map = np.abs(delta).mean(axis=-1)
        if validity is not None:
            valid = validity >= 1.0
            tm_map = np.where(valid, tm_map, 0.0)
            tm = float(tm_map.sum() / max(int(valid.sum()), 1))
        else:
            tm = float(tm_map.mean())
    cb_map = np.maximum(TEMPORAL_WEIGHT * tm_map, sp_map)
    return sp_map, tm_map, cb_map, (sp, tm, float(cb_map.mean()))


def loss_grads(ldr1, ref, ldr0_w=None, ref_w=None, validity=None, mask=None):
    """(g_ldr1, g_ldr0_w) of the combined loss, optimize.py:219-231."""
    sp_map, tm_map, cb_map, _ = losses(ldr1, ref, ldr0_w, ref_w, validity, mask)
    w = np.ones(ldr1.shape[:2]) if mask is None else mask
    n_pix = cb_map.size
    wins = (TEMPORAL_WEIGHT * tm_map) > sp_map
    g_sp = (~wins).astype(np.float64) / n_pix
    g_tm = np.where(wins, TEMPORAL_WEIGHT / n_pix, 0.0)
    g1 = np.sign(ldr1 - ref) * (g_sp * w)[..., None] / 3.0
    if ldr0_w is None:
        return g1, None
    st = np.sign((ldr1 - ldr0_w) - (ref - ref_w))
    return g1 + st * g_tm[..., None] / 3.0, -st * g_tm[..., None] / 3.0
