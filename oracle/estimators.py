"""Stochastic-rounding radiance estimators -- CPU oracle (test-only).

Restates `pkg/src/sparse_sampler/estimators.py:70-149`: the shared
`stochastic_core` for the stochastic / relaxed / straight-through / gumbel
variants, and the bank read of `_bank_inputs` (prefix sum of the first
min(base, S-1) samples plus the holdout sample at that index).
"""

from __future__ import annotations

import numpy as np

GATE_FLOOR = 1e-4
LOGIT_CLAMP = 1e-6


def ramp_gain(lam: float) -> float:
    return 2.0 * lam / (2.0 * lam - 1.0)


def relaxed_ramp(u, frac, lam: float):
    raw = np.zeros(np.broadcast(u, frac).shape)
    np.divide(u + frac - 1.0, frac, out=raw, where=frac > 0)
    return np.clip(lam * raw, 0.0, 1.0)


def gumbel_gate(u, frac, temp: float):
    pc = np.clip(frac, LOGIT_CLAMP, 1.0 - LOGIT_CLAMP)
    uc = np.clip(u, LOGIT_CLAMP, 1.0 - LOGIT_CLAMP)
    z = (np.log(pc) - np.log1p(-pc) + np.log(uc) - np.log1p(-uc)) / temp
    return 1.0 / (1.0 + np.exp(-z))


def stochastic_core(variant, spp, frac, u, base_sum, holdout, lam=10.0,
                    gumbel_temp=1.0, density_floor=1e-8):
    """Returns (noisy, grad, contrib, drawn); spp/frac/u (..., H, W),
    base_sum/holdout (..., H, W, 3)."""
    s = np.maximum(spp, density_floor)[..., None]
    if variant == "stochastic":
        drawn = u < frac
        contrib = np.where(drawn[..., None], holdout, 0.0)
        noisy = (base_sum + contrib) / s
        grad = -noisy / s
    elif variant == "relaxed":
        ramp = relaxed_ramp(u, frac, lam)
        gain = ramp_gain(lam)
        drawn = (frac > 0) & (u >= 1.0 - frac)
        contrib = np.where(drawn[..., None], holdout * (gain * ramp)[..., None], 0.0)
        noisy = (base_sum + contrib) / s
        slope = np.zeros(np.broadcast(u, frac).shape)
        np.divide(lam * (1.0 - u), frac * frac, out=slope, where=drawn & (ramp < 1.0))
        grad = (holdout * (gain * slope)[..., None] - noisy) / s
    elif variant == "straight-through":
        taken = u < frac
        drawn = frac > 0
        contrib = np.where(taken[..., None], holdout, 0.0)
        noisy = (base_sum + contrib) / s
        grad = (np.where(drawn[..., None], holdout, 0.0) - noisy) / s
    elif variant == "gumbel":
        gate = gumbel_gate(u, frac, gumbel_temp)
        drawn = gate > GATE_FLOOR
        contrib = np.where(drawn[..., None], holdout * gate[..., None], 0.0)
        noisy = (base_sum + contrib) / s
        pc = np.clip(frac, LOGIT_CLAMP, 1.0 - LOGIT_CLAMP)
        dgate = np.where((frac > LOGIT_CLAMP) & (frac < 1.0 - LOGIT_CLAMP),
                         gate * (1.0 - gate) / (gumbel_temp * pc * (1.0 - pc)), 0.0)
        grad = (np.where(drawn[..., None], holdout * dgate[..., None], 0.0) - noisy) / s
    else:
        raise ValueError(f"{variant!r} is not a stochastic variant")
    return noisy, grad, contrib, drawn


def bank_inputs(base: np.ndarray, samples: np.ndarray):
    """samples (H, W, S, 3): (prefix sum of the first min(base, S-1) samples,
    sample at min(base, S-1)) (ref estimators.py:136-139, banks.py:61-73)."""
    cap = samples.shape[2]
    idx = np.minimum(base, cap - 1)
    csum = np.zeros(samples.shape[:2] + (cap + 1, 3))
    np.cumsum(samples, axis=2, out=csum[:, :, 1:])
    ii = idx.astype(np.intp)[:, :, None, None]
    base_sum = np.take_along_axis(csum, ii, axis=2)[:, :, 0]
    holdout = np.take_along_axis(samples, ii, axis=2)[:, :, 0]
    return base_sum, holdout


def estimate(variant, spp, base, frac, u, samples, lam=10.0, gumbel_temp=1.0,
             density_floor=1e-8):
    """`_stochastic_estimate` (ref estimators.py:142-149): returns
    (noisy_clamped, grad, contrib, samples_used)."""
    base_sum, holdout = bank_inputs(base, samples)
    noisy, grad, contrib, drawn = stochastic_core(variant, spp, frac, u, base_sum, holdout,
                                                  lam, gumbel_temp, density_floor)
    used = np.minimum(base, samples.shape[2] - 1) + drawn.astype(np.int64)
    return np.maximum(noisy, 0.0), grad, contrib, used
