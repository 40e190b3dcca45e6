"""Result/argument containers with the reference's field names and checks.

When ``install()`` patches the reference package, the compat functions return
the reference's own container classes instead (``bind_reference_types``), so
``isinstance`` checks and downstream code behave exactly as before.
Reference: images.py:12-34 (RadianceImage), density.py:17-40,173-190,
estimators.py:44-67, pyramid.py:51-90,127-138,264-289.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class RadianceImage:
    data: np.ndarray

    def __post_init__(self):
        self.data = np.asarray(self.data, dtype=np.float64)
        if self.data.ndim != 3 or self.data.shape[2] != 3:
            raise ValueError("radiance image must have shape (H, W, 3)")
        if not np.isfinite(self.data).all():
            raise ValueError("radiance values must be finite")
        if (self.data < 0).any():
            raise ValueError("radiance values must be non-negative")

    @property
    def width(self) -> int:
        return self.data.shape[1]

    @property
    def height(self) -> int:
        return self.data.shape[0]


@dataclass
class DensityMap:
    spp: np.ndarray
    budget: float

    def __post_init__(self):
        self.spp = np.asarray(self.spp, dtype=np.float64)
        if self.spp.ndim != 2:
            raise ValueError("density map must be 2-D")
        if self.budget <= 0:
            raise ValueError("budget must be positive")
        total = self.budget * self.spp.size
        if abs(self.spp.sum() - total) > 1e-4 * total:
            raise ValueError("density does not sum to the frame budget")
        if (self.spp < self.budget / 8.0 * (1 - 1e-12)).any():
            raise ValueError("density below the uniform floor budget/8")

    @property
    def width(self) -> int:
        return self.spp.shape[1]

    @property
    def height(self) -> int:
        return self.spp.shape[0]


@dataclass
class SampleAllocation:
    base: np.ndarray
    frac: np.ndarray
    u: np.ndarray
    taken: np.ndarray

    @property
    def width(self) -> int:
        return self.base.shape[1]

    @property
    def height(self) -> int:
        return self.base.shape[0]


VARIANTS = ("deterministic", "stochastic", "relaxed", "straight-through", "gumbel")


@dataclass
class EstimatorConfig:
    variant: str = "relaxed"
    lam: float = 10.0
    gumbel_temp: float = 1.0
    density_floor: float = 1e-8

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown estimator variant {self.variant!r}")
        if self.lam < 1.0:
            raise ValueError("ramp temperature must be >= 1")
        if self.gumbel_temp <= 0:
            raise ValueError("gumbel temperature must be positive")
        if self.density_floor <= 0:
            raise ValueError("density floor must be positive")


@dataclass
class EstimatorResult:
    noisy: RadianceImage
    grad_density: np.ndarray
    holdout_contrib: np.ndarray
    samples_used: np.ndarray


@dataclass
class DemodMap:
    values: np.ndarray

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float64)
        if not np.isfinite(self.values).all() or (self.values <= 0).any():
            raise ValueError("demodulation map must be finite and strictly positive")


@dataclass
class PyramidStack:
    levels: list

    @property
    def width(self) -> int:
        return self.levels[0].shape[1]

    @property
    def height(self) -> int:
        return self.levels[0].shape[0]


@dataclass
class PyramidGrads:
    logits: list | None
    demod: np.ndarray | None
    input: np.ndarray
    prev: np.ndarray | None


# classes the compat functions construct; install() may rebind them
TYPES = {"RadianceImage": RadianceImage, "DensityMap": DensityMap,
         "SampleAllocation": SampleAllocation, "EstimatorResult": EstimatorResult,
         "PyramidStack": PyramidStack, "PyramidGrads": PyramidGrads}


def bind_reference_types(mapping: dict) -> dict:
    """Make compat functions construct the given classes; returns the old map."""
    old = dict(TYPES)
    TYPES.update({k: v for k, v in mapping.items() if k in TYPES})
    return old


def make(name, *args, **kw):
    return TYPES[name](*args, **kw)
