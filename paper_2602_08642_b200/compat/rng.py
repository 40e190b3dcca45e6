"""Drop-in for ``sparse_sampler.rng``'s uniform variates
(reference pkg/src/sparse_sampler/rng.py:21-81) computed on the GPU with the
identical splitmix64 key hash, so every variate is bit-identical."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .. import ops
from . import _dev

STREAM_ALLOC = 0
STREAM_TAKE = 1
STREAM_SAMPLE_BASE = 16


@dataclass(frozen=True)
class PixelRngKey:
    seed: int
    frame: int
    x: int
    y: int
    stream: int


def uniform_grid(seed: int, frame: int, width: int, height: int, stream: int) -> np.ndarray:
    u = ops.uniform_grid(int(seed), height, width, frame0=int(frame), stream_id=int(stream),
                         device=_dev.device())
    return _dev.to_host(u[0])


def uniform_grid_batch(seed: int, frames, width: int, height: int, stream: int) -> np.ndarray:
    u = ops.uniform_grid(int(seed), height, width, frames=np.asarray(frames, dtype=np.int64),
                         stream_id=int(stream), device=_dev.device())
    return _dev.to_host(u)


def pixel_uniform(key: PixelRngKey) -> float:
    """One variate (ref rng.py:51-54): a single-thread launch, not a grid."""
    return float(ops.uniform_at(int(key.seed), int(key.frame), int(key.x), int(key.y), int(key.stream),
                                device=_dev.device()).item())
