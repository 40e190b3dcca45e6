"""Drop-in for the hot-path part of ``sparse_sampler.estimators``
(reference pkg/src/sparse_sampler/estimators.py:44-196) on the GPU.

``stochastic_core`` and the bank-reading ``estimate`` / ``estimate_*`` run in
float64 on the device (bit-identical to the reference for the stochastic,
relaxed and straight-through variants; the gumbel gate's log/exp agree to
~1e-15).  The deterministic-rounding estimator (a prior-work baseline) and the
gradient-comparison harness are outside the hot path: ``estimate`` forwards
the deterministic variant to the function it replaced when installed into the
reference, and raises otherwise.
"""

from __future__ import annotations

import numpy as np

from .. import ops
from . import _dev, _types
from ._types import EstimatorConfig, EstimatorResult  # noqa: F401

_fallthrough = {}  # name -> replaced reference function (set by install())


def stochastic_core(variant: str, spp, frac, u, base_sum, holdout, cfg):
    """Shared forward/backward math of the stochastic variants; broadcasts
    over leading axes like the reference (ref :90-133)."""
    spp, frac, u = (np.asarray(a, dtype=np.float64) for a in (spp, frac, u))
    base_sum = np.asarray(base_sum, dtype=np.float64)
    holdout = np.asarray(holdout, dtype=np.float64)
    shape = np.broadcast_shapes(spp.shape, frac.shape, u.shape, base_sum.shape[:-1],
                                holdout.shape[:-1])
    b = lambda a, s: np.ascontiguousarray(np.broadcast_to(a, s))  # noqa: E731
    noisy, grad, contrib, drawn = ops.stochastic_core(
        variant, _dev.to_dev(b(spp, shape)), _dev.to_dev(b(frac, shape)), _dev.to_dev(b(u, shape)),
        _dev.to_dev(b(base_sum, shape + (3,))), _dev.to_dev(b(holdout, shape + (3,))),
        lam=cfg.lam, gumbel_temp=cfg.gumbel_temp, density_floor=cfg.density_floor)
    return _dev.to_host(noisy), _dev.to_host(grad), _dev.to_host(contrib), _dev.to_host(drawn)


def _stochastic_estimate(variant, density, alloc, bank, cfg):
    samples = getattr(bank, "samples", None)
    if samples is not None:
        # materialised SampleBank (H, W, S, 3): the bank read is fused on device
        noisy, grad, contrib, used, _ = ops.estimate(
            variant, _dev.to_dev(density.spp), _dev.to_dev(alloc.base, None).long(),
            _dev.to_dev(alloc.frac), _dev.to_dev(alloc.u), _dev.to_dev(samples),
            lam=cfg.lam, gumbel_temp=cfg.gumbel_temp, density_floor=cfg.density_floor)
        return _types.make("EstimatorResult", _types.make("RadianceImage", _dev.to_host(noisy[0])),
                           _dev.to_host(grad[0]), _dev.to_host(contrib[0]), _dev.to_host(used[0]))
    # lazily drawn bank (renderer stand-in): read its samples, core on device
    idx = np.minimum(alloc.base, bank.capacity - 1)
    base_sum, holdout = bank.prefix_sum(idx), bank.sample_at(idx)
    noisy, grad, contrib, drawn = stochastic_core(variant, density.spp, alloc.frac, alloc.u,
                                                  base_sum, holdout, cfg)
    used = idx + drawn.astype(np.int64)
    return _types.make("EstimatorResult", _types.make("RadianceImage", np.maximum(noisy, 0.0)),
                       grad, contrib, used)


def estimate_stochastic(density, alloc, bank, cfg=None):
    return _stochastic_estimate("stochastic", density, alloc, bank,
                                cfg or EstimatorConfig(variant="stochastic"))


def estimate_relaxed(density, alloc, bank, cfg=None):
    return _stochastic_estimate("relaxed", density, alloc, bank,
                                cfg or EstimatorConfig(variant="relaxed"))


def estimate_straight_through(density, alloc, bank, cfg=None):
    return _stochastic_estimate("straight-through", density, alloc, bank,
                                cfg or EstimatorConfig(variant="straight-through"))


def estimate_gumbel(density, alloc, bank, cfg=None):
    return _stochastic_estimate("gumbel", density, alloc, bank,
                                cfg or EstimatorConfig(variant="gumbel"))


def estimate(variant: str, density, alloc, bank, cfg, ref=None):
    """ref :188-196.  The deterministic-rounding estimator (a prior-work
    baseline outside the hot path, estimators.py:171-185) is NOT run on the
    GPU: installed into the reference it is forwarded to the reference's own
    CPU function (documented behaviour); standalone it
    raises NotImplementedError."""
    if variant == "deterministic":
        if ref is None:
            raise ValueError("deterministic estimator needs a reference image")
        if "estimate_deterministic" in _fallthrough:
            return _fallthrough["estimate_deterministic"](density, bank, ref)
        raise NotImplementedError("the deterministic estimator is not part of the GPU hot path")
    if alloc is None:
        raise ValueError("stochastic variants need a sample allocation")
    return _stochastic_estimate(variant, density, alloc, bank, cfg)


def take_rule(variant: str) -> str:
    return {"relaxed": "relaxed", "gumbel": "gumbel"}.get(variant, "stochastic")
