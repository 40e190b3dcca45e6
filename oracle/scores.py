"""Estimator backward to the density scores -- CPU oracle (test-only).

Restates the sampler half of `optimize.evaluate_step`
(`pkg/src/sparse_sampler/optimize.py:244-251`):
  g_spp = sum over frames of sum_c g_input * grad_density,
  blurred by scipy.ndimage.gaussian_filter(g_spp, sigma, mode="nearest"),
  g_scores = (7/8 * budget * N) * softmax_backward(softmax(scores), g_spp)
(`density.py:43-52`).  The blur is a third-party call (scipy 1.18.x, in this
image); its published algorithm is restated here: separable 1-D correlations
along axis 0 then axis 1 with weights exp(-x^2 / (2 sigma^2)), |x| <=
int(4 sigma + 0.5), normalised to sum 1, edges replicated ("nearest").
"""

from __future__ import annotations

import numpy as np

from .density import softmax_global, softmax_global_backward


def gaussian_weights(sigma: float) -> np.ndarray:
    r = int(4.0 * sigma + 0.5)
    x = np.arange(-r, r + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    return phi / phi.sum()


def gaussian_nearest(img: np.ndarray, sigma: float) -> np.ndarray:
    wts = gaussian_weights(sigma)
    r = (len(wts) - 1) // 2
    out = np.asarray(img, dtype=np.float64)
    for axis in (0, 1):
        pad = [(0, 0), (0, 0)]
        pad[axis] = (r, r)
        p = np.pad(out, pad, mode="edge")
        n = out.shape[axis]
        acc = np.take(p, np.arange(r, r + n), axis=axis) * wts[r]
        for j in range(r, 0, -1):
            lo = np.take(p, np.arange(r - j, r - j + n), axis=axis)
            hi = np.take(p, np.arange(r + j, r + j + n), axis=axis)
            acc = acc + (lo + hi) * wts[r + j]
        out = acc
    return out


def score_grad(scores, budget, g_inputs, grad_densities, sigma=1.5):
    """scores (H, W); g_inputs / grad_densities: lists over frames of (H, W, C)."""
    g_spp = None
    for gi, gd in zip(g_inputs, grad_densities):
        s = (gi * gd).sum(axis=-1)
        g_spp = s if g_spp is None else g_spp + s
    if sigma > 0:
        g_spp = gaussian_nearest(g_spp, sigma)
    w = softmax_global(np.asarray(scores, dtype=np.float64))
    return (7.0 / 8.0) * budget * w.size * softmax_global_backward(w, g_spp)
