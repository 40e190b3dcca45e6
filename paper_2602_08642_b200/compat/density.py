"""Drop-in for the hot-path part of ``sparse_sampler.density``
(reference pkg/src/sparse_sampler/density.py:13-69,173-233) on the GPU.

normalize_density (frame-global softmax, deterministic two-pass reduction),
allocate (stochastic and dithered u, floor/frac, take rules) and
holdout_taken.  Decisions are float64 on the device, so base / frac / u /
taken are bit-identical to the reference.  The void-and-cluster mask builder
is a serial CPU precompute and stays out of scope (any object with ``.rank``
and ``.size`` -- e.g. the reference's DitherMask -- is accepted).
"""

from __future__ import annotations

import numpy as np

from .. import ops
from . import _dev, _types
from ._types import DensityMap, SampleAllocation  # noqa: F401

UNIFORM_FRACTION = 1.0 / 8.0
TAKE_RULES = ("stochastic", "relaxed", "gumbel")
_RULE_VARIANT = {"stochastic": "stochastic", "relaxed": "relaxed", "gumbel": "gumbel"}


def normalize_density(scores, budget: float):
    """budget/8 floor + 7/8 budget distributed by a frame-global softmax."""
    scores = np.asarray(scores, dtype=np.float64)
    if not np.isfinite(scores).all():
        raise ValueError("scores must be finite")
    if budget <= 0:
        raise ValueError("budget must be positive")
    if scores.ndim != 2:
        raise ValueError("density map must be 2-D")
    spp = ops.normalize_density(_dev.to_dev(scores), float(budget))[0]
    return _types.make("DensityMap", _dev.to_host(spp), budget)


def uniform_density(width: int, height: int, budget: float):
    return normalize_density(np.zeros((height, width)), budget)


def holdout_taken(rule: str, u, frac, gumbel_temp: float = 1.0):
    """Whether the fractional extra sample is taken under `rule` (ref :196-206)."""
    if rule not in _RULE_VARIANT:
        raise ValueError(f"unknown take rule {rule!r}")
    u, frac = np.broadcast_arrays(np.asarray(u, dtype=np.float64), np.asarray(frac, dtype=np.float64))
    shape = u.shape
    z = np.zeros(shape + (3,))
    # the estimator core's `drawn` flag is exactly the take rule's decision
    _, _, _, drawn = ops.stochastic_core(_RULE_VARIANT[rule], _dev.to_dev(np.ones(shape)),
                                         _dev.to_dev(frac), _dev.to_dev(u), _dev.to_dev(z),
                                         _dev.to_dev(z), gumbel_temp=gumbel_temp)
    return _dev.to_host(drawn)


def allocate(density, mode: str = "stochastic", mask=None, frame: int = 0, seed: int = 0,
             rule: str = "stochastic", gumbel_temp: float = 1.0):
    """Integer counts + holdout variate + take decision (ref :209-233)."""
    if mode not in ("stochastic", "dithered"):
        raise ValueError(f"unknown allocation mode {mode!r}")
    if mode == "dithered" and mask is None:
        raise ValueError("dithered allocation requires a mask")
    if rule not in TAKE_RULES:
        raise ValueError(f"unknown take rule {rule!r}")
    spp = _dev.to_dev(density.spp)
    rank = np.asarray(mask.rank) if mode == "dithered" else None
    base, frac, u, taken = ops.allocate(spp, mode=mode, rank=rank, frame0=frame, seed=seed,
                                        rule=rule, gumbel_temp=gumbel_temp)
    return _types.make("SampleAllocation", _dev.to_host(base[0]), _dev.to_host(frac[0]),
                       _dev.to_host(u[0]), _dev.to_host(taken[0]))


def score_gradient(scores, budget: float, g_inputs, grad_densities, blur: float = 1.5):
    """The sampler half of optimize.evaluate_step (optimize.py:244-251) as one
    GPU call: g_spp = sum over frames of sum_c g_input * grad_density, blurred
    by gaussian_filter(blur, mode="nearest"), then
    7/8 * budget * N * softmax_backward(softmax(scores), g_spp).
    scores (H, W); g_inputs / grad_densities: sequences over frames of (H, W, C)."""
    scores = np.asarray(scores, dtype=np.float64)
    gi = np.stack([np.asarray(a, dtype=np.float64) for a in g_inputs])
    gd = np.stack([np.asarray(a, dtype=np.float64) for a in grad_densities])
    if gi.shape != gd.shape or gi.shape[1:3] != scores.shape:
        raise ValueError("score gradient: dimensions must match")
    dt = _dev.dtype()
    gi_t = _dev.to_dev(np.ascontiguousarray(gi.transpose(0, 3, 1, 2))[None], dt)
    gd_t = _dev.to_dev(np.ascontiguousarray(gd.transpose(0, 3, 1, 2))[None], dt)
    out = ops.score_grad(_dev.to_dev(scores, dt)[None], gi_t, gd_t, float(budget), float(blur))
    return _dev.to_host(out[0]).astype(np.float64)
