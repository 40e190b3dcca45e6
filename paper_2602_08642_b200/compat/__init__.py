"""Reference-signature drop-ins for the sparse-sampler hot path, on the GPU.

    from paper_2602_08642_b200 import compat
    compat.install()          # patch an importable `sparse_sampler` package in place
    ...
    compat.uninstall()

``install()`` patches both the defining modules (sparse_sampler.pyramid,
.density, .estimators, .rng, .images, .tonemap, .losses) and every module that bound the names at import
time (sparse_sampler.optimize, sparse_sampler.estimators, the package
namespace), and makes the patched functions return the
reference's own container classes.  Without the reference installed, the
compat modules are usable directly with the same API.
"""

from __future__ import annotations

import importlib
import importlib.util
import sys

from . import _dev, _types, density, estimators, images, losses, pyramid, rng, tonemap  # noqa: F401
from ._dev import precision, set_precision  # noqa: F401

# name -> compat module providing it, per reference module
PATCHES = {
    "pyramid": ["normalize_kernels", "build_pyramid", "gather5", "upsample2", "reconstruct_core",
                "reconstruct", "reconstruct_backward"],
    "density": ["normalize_density", "uniform_density", "allocate", "holdout_taken"],
    "estimators": ["stochastic_core", "estimate", "estimate_stochastic", "estimate_relaxed",
                   "estimate_straight_through", "estimate_gumbel"],
    "rng": ["uniform_grid", "uniform_grid_batch", "pixel_uniform"],
    "images": ["warp_array", "warp_backward"],
    "tonemap": ["tonemap_array", "tonemap_backward"],
    "losses": ["spatial_loss", "temporal_loss"],
}
_COMPAT = {"pyramid": pyramid, "density": density, "estimators": estimators, "rng": rng,
           "images": images, "tonemap": tonemap, "losses": losses}
_saved: list = []
_saved_types: dict | None = None


def install(package: str = "sparse_sampler") -> list:
    """Route the reference package's hot-path functions to the GPU.  Returns
    the list of (module, name) pairs patched."""
    global _saved_types
    if _saved:
        return [(m.__name__, n) for m, n, _ in _saved]
    root = importlib.import_module(package)
    mods = {k: importlib.import_module(f"{package}.{k}") for k in PATCHES}
    importers = [root] + [importlib.import_module(f"{package}.{m}")
                          for m in ("optimize", "estimators", "density", "cli")
                          if importlib.util.find_spec(f"{package}.{m}")]
    # keep the reference's containers so results are the classes callers expect
    ref_types = {}
    for cls in ("RadianceImage",):
        ref_types[cls] = getattr(importlib.import_module(f"{package}.images"), cls)
    for cls in ("DensityMap", "SampleAllocation"):
        ref_types[cls] = getattr(mods["density"], cls)
    ref_types["EstimatorResult"] = mods["estimators"].EstimatorResult
    ref_types["PyramidStack"] = mods["pyramid"].PyramidStack
    ref_types["PyramidGrads"] = mods["pyramid"].PyramidGrads
    _saved_types = _types.bind_reference_types(ref_types)
    estimators._fallthrough["estimate_deterministic"] = mods["estimators"].estimate_deterministic
    # the compat pyramid reads LEVELS at call time from the reference module
    for modname, names in PATCHES.items():
        for name in names:
            new = getattr(_COMPAT[modname], name)
            for target in [mods[modname]] + importers:
                if hasattr(target, name) and getattr(target, name) is not new:
                    _saved.append((target, name, getattr(target, name)))
                    setattr(target, name, new)
    pyramid._levels_source = mods["pyramid"]
    return [(m.__name__, n) for m, n, _ in _saved]


def uninstall() -> None:
    global _saved_types
    while _saved:
        target, name, old = _saved.pop()
        setattr(target, name, old)
    if _saved_types is not None:
        _types.bind_reference_types(_saved_types)
        _saved_types = None
    estimators._fallthrough.clear()
    pyramid._levels_source = None


def installed() -> bool:
    return bool(_saved)


del sys
