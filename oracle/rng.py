"""Counter-based per-pixel uniforms -- CPU oracle (test-only).

Restates `pkg/src/sparse_sampler/rng.py:21-63,73-81`: a splitmix64 finaliser
chained over the key words (seed, frame, x, y, stream) with wrapping uint64
arithmetic; the variate is the top 53 bits scaled by 2**-53.
"""

from __future__ import annotations

import numpy as np

STREAM_ALLOC = 0
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)
SCALE53 = 1.0 / float(1 << 53)


def splitmix_finalize(z):
    z = (z ^ (z >> np.uint64(30))) * MIX1
    z = (z ^ (z >> np.uint64(27))) * MIX2
    return z ^ (z >> np.uint64(31))


def key_hash(seed, frame, x, y, stream):
    with np.errstate(over="ignore"):
        h = splitmix_finalize(np.uint64(seed) + GOLDEN)
        for word in (frame, x, y, stream):
            h = splitmix_finalize(h ^ (np.asarray(word, dtype=np.uint64) * GOLDEN + GOLDEN))
    return h


def uniform_grid(seed: int, frame: int, width: int, height: int, stream: int) -> np.ndarray:
    xs = np.arange(width, dtype=np.uint64)[None, :]
    ys = np.arange(height, dtype=np.uint64)[:, None]
    return (key_hash(seed, frame, xs, ys, stream) >> np.uint64(11)).astype(np.float64) * SCALE53


def uniform_grid_batch(seed: int, frames, width: int, height: int, stream: int) -> np.ndarray:
    fs = np.asarray(frames, dtype=np.uint64)[:, None, None]
    xs = np.arange(width, dtype=np.uint64)[None, None, :]
    ys = np.arange(height, dtype=np.uint64)[None, :, None]
    return (key_hash(seed, fs, xs, ys, stream) >> np.uint64(11)).astype(np.float64) * SCALE53


def uniform_bits(seed: int, frame: int, width: int, height: int, stream: int) -> np.ndarray:
    """The 53-bit integer behind each variate (u = bits * 2**-53)."""
    xs = np.arange(width, dtype=np.uint64)[None, :]
    ys = np.arange(height, dtype=np.uint64)[:, None]
    return key_hash(seed, frame, xs, ys, stream) >> np.uint64(11)
