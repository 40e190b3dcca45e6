"""Temporal warp -- CPU oracle (test-only).

Restates `pkg/src/sparse_sampler/images.py`:
* `warp_array` (`:88-119`): every output pixel samples the previous frame at
  (x + mx, y + my) with bilinear weights over the four taps (0,0), (0,1),
  (1,0), (1,1); taps outside the frame weigh zero (their indices are clipped),
  validity = the in-frame weight sum;
* `warp_backward` (`:122-147`): its transpose, accumulated tap by tap in
  raster order (the reference's `np.add.at`).
Images are (H, W, C) float64, motion (H, W, 2) = (mx, my).
"""

from __future__ import annotations

import numpy as np

TAPS = ((0, 0), (0, 1), (1, 0), (1, 1))  # (dy, dx), images.py:106-107


def _taps(motion: np.ndarray):
    h, w = motion.shape[:2]
    ys, xs = np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64), indexing="ij")
    sx, sy = xs + motion[:, :, 0], ys + motion[:, :, 1]
    x0, y0 = np.floor(sx), np.floor(sy)
    fx, fy = sx - x0, sy - y0
    for dy, dx in TAPS:
        wt = (fx if dx else 1 - fx) * (fy if dy else 1 - fy)
        tx, ty = x0 + dx, y0 + dy
        inside = (tx >= 0) & (tx < w) & (ty >= 0) & (ty < h)
        yield (np.where(inside, wt, 0.0), np.clip(ty, 0, h - 1).astype(np.intp),
               np.clip(tx, 0, w - 1).astype(np.intp))


def warp_array(prev: np.ndarray, motion: np.ndarray):
    if prev.shape[:2] != motion.shape[:2]:
        raise ValueError("warp: image and motion dimensions must match")
    out = np.zeros(prev.shape, dtype=np.float64)
    validity = np.zeros(prev.shape[:2], dtype=np.float64)
    for wi, iy, ix in _taps(motion):
        out += wi[:, :, None] * prev[iy, ix]
        validity += wi
    return out, validity


def warp_backward(grad_out: np.ndarray, motion: np.ndarray) -> np.ndarray:
    h, w = grad_out.shape[:2]
    gp = np.zeros(grad_out.shape, dtype=np.float64)
    flat = gp.reshape(h * w, -1)
    for wi, iy, ix in _taps(motion):
        np.add.at(flat, (iy * w + ix).ravel(), (wi[:, :, None] * grad_out).reshape(h * w, -1))
    return gp
