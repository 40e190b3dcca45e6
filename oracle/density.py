"""Density normalisation and stochastic allocation -- CPU oracle (test-only).

Restates `pkg/src/sparse_sampler/density.py`:
* spp = b/8 + 7/8 * b * N * softmax(scores), frame-global softmax (`:43-65`)
* allocation: base = floor(spp), frac = spp - base, u from the allocation
  stream (stochastic mode) or a tiled, per-frame shifted rank mask (dithered
  mode) (`:209-233`)
* take rules stochastic / relaxed / gumbel (`:196-206`)
"""

from __future__ import annotations

import numpy as np

from . import rng
from .estimators import gumbel_gate

UNIFORM_FRACTION = 1.0 / 8.0


def softmax_global(values: np.ndarray) -> np.ndarray:
    e = np.exp(values - values.max())
    return e / e.sum()


def softmax_global_backward(w: np.ndarray, gw: np.ndarray) -> np.ndarray:
    return w * (gw - (w * gw).sum())


def normalize_density(scores, budget: float) -> np.ndarray:
    scores = np.asarray(scores, dtype=np.float64)
    if not np.isfinite(scores).all():
        raise ValueError("scores must be finite")
    if budget <= 0:
        raise ValueError("budget must be positive")
    adaptive = (1.0 - UNIFORM_FRACTION) * budget * scores.size
    return UNIFORM_FRACTION * budget + adaptive * softmax_global(scores)


def validate_density(spp: np.ndarray, budget: float) -> None:
    """DensityMap.__post_init__ checks (ref density.py:22-32)."""
    if spp.ndim != 2:
        raise ValueError("density map must be 2-D")
    if budget <= 0:
        raise ValueError("budget must be positive")
    total = budget * spp.size
    if abs(spp.sum() - total) > 1e-4 * total:
        raise ValueError("density does not sum to the frame budget")
    if (spp < budget / 8.0 * (1 - 1e-12)).any():
        raise ValueError("density below the uniform floor budget/8")


def holdout_taken(rule: str, u, frac, gumbel_temp: float = 1.0):
    if rule == "stochastic":
        return u < frac
    if rule == "relaxed":
        return (frac > 0) & (u >= 1.0 - frac)
    if rule == "gumbel":
        return gumbel_gate(u, frac, gumbel_temp) > 1e-4
    raise ValueError(f"unknown take rule {rule!r}")


def dithered_u(rank: np.ndarray, frame: int, width: int, height: int) -> np.ndarray:
    t = rank.shape[0]
    ys, xs = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    sy, sx = (frame * 7) % t, (frame * 13) % t
    return (rank[(ys + sy) % t, (xs + sx) % t] + 0.5) / (t * t)


def allocate(spp: np.ndarray, mode: str = "stochastic", rank=None, frame: int = 0,
             seed: int = 0, rule: str = "stochastic", gumbel_temp: float = 1.0):
    """Returns (base int64, frac, u, taken)."""
    base = np.floor(spp).astype(np.int64)
    frac = spp - base
    h, w = spp.shape
    if mode == "stochastic":
        u = rng.uniform_grid(seed, frame, w, h, rng.STREAM_ALLOC)
    elif mode == "dithered":
        if rank is None:
            raise ValueError("dithered allocation requires a mask")
        u = dithered_u(np.asarray(rank), frame, w, h)
    else:
        raise ValueError(f"unknown allocation mode {mode!r}")
    return base, frac, u, holdout_taken(rule, u, frac, gumbel_temp)
