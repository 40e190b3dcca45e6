"""Generate the golden fixtures in this directory from the UNMODIFIED reference.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every array stored here is an output of the reference's own functions
(`sparse_sampler.pyramid`, `.density`, `.rng`, `.estimators`, `.banks`,
`.images`, `.tonemap`, `.losses`, and scipy's gaussian_filter exactly as
optimize.py calls it) on
seeded inputs that are stored alongside.  The oracle is pinned against these
files (tests/test_oracle_golden.py) and the GPU parity tests reuse them.
Level counts other than the reference's default 5 are produced by setting
`sparse_sampler.pyramid.LEVELS`, which every pyramid function reads at call
time (discrepancy 1).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import sparse_sampler.pyramid as P  # noqa: E402
from sparse_sampler import density as D  # noqa: E402
from sparse_sampler import estimators as E  # noqa: E402
from sparse_sampler import rng as R  # noqa: E402
from sparse_sampler import images as I  # noqa: E402
from sparse_sampler import losses as LS  # noqa: E402
from sparse_sampler import tonemap as TM  # noqa: E402
from sparse_sampler.banks import SampleBank  # noqa: E402
from scipy.ndimage import gaussian_filter  # noqa: E402  (the reference's own blur, optimize.py:20)

PYRAMID_CASES = [
    # name, H, W, levels, demod, prev, want_param_grads, logit scale
    ("p_8x8_L5_full", 8, 8, 5, True, True, True, 0.7),
    ("p_13x11_L3_demod", 13, 11, 3, True, False, True, 1.0),
    ("p_12x10_L4_plain", 12, 10, 4, False, False, True, 1.0),
    ("p_7x9_L4_demod_prev", 7, 9, 4, True, True, True, 1.2),
    ("p_16x16_L3_nograd", 16, 16, 3, True, False, False, 1.0),
    ("p_5x3_L2_demod", 5, 3, 2, True, False, True, 1.0),
    ("p_20x18_L3_demod", 20, 18, 3, True, False, True, 1.5),
    ("p_9x6_L2_prev", 9, 6, 2, False, True, True, 0.8),
]


def pyramid_case(name, h, w, levels, use_demod, use_prev, want, scale, seed):
    rng = np.random.default_rng(seed)
    old = P.LEVELS
    P.LEVELS = levels
    try:
        kf = P.zero_kernel_field(w, h)
        for arr in kf.logits:
            arr += rng.normal(0.0, scale, arr.shape)
        noisy = rng.uniform(0.01, 3.0, (h, w, 3)) * np.where(rng.uniform(size=(h, w, 1)) < 0.05, 20.0, 1.0)
        demod = rng.uniform(0.0005, 1.0, (h, w, 3)) if use_demod else None
        prev = rng.uniform(0.01, 2.0, (h, w, 3)) if use_prev else None
        up = rng.normal(0.0, 1.0, (h, w, 3))
        out, tape = P.reconstruct_core(noisy, kf, prev, demod)
        g = P.reconstruct_backward(tape, up, want_param_grads=want)
    finally:
        P.LEVELS = old
    d = {"H": h, "W": w, "levels": levels, "k": 5, "want": int(want),
         "noisy": noisy, "upstream": up, "out": out, "g_input": g.input}
    for l, arr in enumerate(kf.logits):
        d[f"logits{l}"] = arr
        if want:
            d[f"g_logits{l}"] = g.logits[l]
    if use_demod:
        d["demod"] = demod
        if want:
            d["g_demod"] = g.demod
    if use_prev:
        d["prev"] = prev
        d["g_prev"] = g.prev
    return d


def primitives(seed):
    rng = np.random.default_rng(seed)
    d = {}
    img = rng.uniform(0, 4, (9, 7, 3))
    wts = rng.dirichlet(np.ones(25), size=(9, 7))
    d["gather_img"], d["gather_w"], d["gather_out"] = img, wts, P.gather5(img, wts)
    coarse = rng.uniform(0, 5, (5, 4, 3))
    uw = rng.dirichlet(np.ones(4), size=(9, 7))
    d["up_coarse"], d["up_w"], d["up_out"] = coarse, uw, P.upsample2(coarse, uw)
    pyr_in = rng.uniform(0, 2, (11, 13, 3))
    d["pyr_in"] = pyr_in
    for l, lv in enumerate(P.build_pyramid(pyr_in).levels):
        d[f"pyr_level{l}"] = lv
    kf = P.zero_kernel_field(6, 5)
    for arr in kf.logits:
        arr += rng.normal(0, 2.0, arr.shape)
    for l, arr in enumerate(kf.logits):
        d[f"nk_logits{l}"] = arr
    for l, wl in enumerate(P.normalize_kernels(kf, include_temporal=True)):
        d[f"nk_wt{l}"] = wl
    for l, wl in enumerate(P.normalize_kernels(kf, include_temporal=False)):
        d[f"nk_wf{l}"] = wl
    return d


def placement(seed):
    rng = np.random.default_rng(seed)
    d = {}
    # rng: key-hash variates
    keys = [(0, 0, 0), (42, 7, 2), (9, 3, 1), (2**40 + 17, 123456, 0), (5, 2**31 + 3, 16)]
    for i, (s, f, st) in enumerate(keys):
        d[f"ug{i}_key"] = np.array([s, f, st], dtype=np.uint64)
        d[f"ug{i}"] = R.uniform_grid(s, f, 23, 17, st)
    d["ugb_frames"] = np.array([0, 5, 17, 1000003])
    d["ugb"] = R.uniform_grid_batch(2, d["ugb_frames"], 19, 11, 3)
    # normalize_density
    for i, (h, w, budget, sc) in enumerate([(17, 23, 0.25, 1.0), (8, 8, 1.0, 3.0), (31, 5, 0.5, 0.3)]):
        scores = rng.normal(0, sc, (h, w))
        d[f"nd{i}_scores"], d[f"nd{i}_budget"] = scores, np.float64(budget)
        d[f"nd{i}_spp"] = D.normalize_density(scores, budget).spp
    # allocate (stochastic mode) for all rules
    spp = D.normalize_density(rng.normal(0, 1.5, (21, 29)), 0.7).spp
    d["al_spp"] = spp
    dm = D.DensityMap(spp, 0.7)
    for rule in ("stochastic", "relaxed", "gumbel"):
        a = D.allocate(dm, "stochastic", frame=11, seed=5, rule=rule, gumbel_temp=0.7)
        d[f"al_{rule}_base"], d[f"al_{rule}_frac"] = a.base, a.frac
        d[f"al_{rule}_u"], d[f"al_{rule}_taken"] = a.u, a.taken
    mask = D.void_cluster_mask(16, seed=3)
    d["dm_rank"] = mask.rank
    a = D.allocate(dm, "dithered", mask=mask, frame=5)
    d["dm_u"], d["dm_taken"] = a.u, a.taken
    # estimators: stochastic_core per variant + estimate through a bank
    h, w, s_cap = 13, 15, 4
    samples = rng.lognormal(-1.0, 1.5, (h, w, s_cap, 3))
    samples *= np.where(rng.uniform(size=(h, w, s_cap, 1)) < 0.01, 100.0, 1.0)
    spp2 = D.normalize_density(rng.normal(0, 1.2, (h, w)), 1.3).spp
    d["es_samples"], d["es_spp"] = samples, spp2
    bank = SampleBank(samples, seed=0)
    dm2 = D.DensityMap(spp2, 1.3)
    for variant in ("stochastic", "relaxed", "straight-through", "gumbel"):
        cfg = E.EstimatorConfig(variant=variant, lam=7.0, gumbel_temp=0.8)
        alloc = D.allocate(dm2, "stochastic", frame=3, seed=9, rule=E.take_rule(variant),
                           gumbel_temp=0.8)
        res = E.estimate(variant, dm2, alloc, bank, cfg)
        key = variant.replace("-", "_")
        d[f"es_{key}_u"] = alloc.u
        d[f"es_{key}_noisy"] = res.noisy.data
        d[f"es_{key}_grad"] = res.grad_density
        d[f"es_{key}_contrib"] = res.holdout_contrib
        d[f"es_{key}_used"] = res.samples_used
        base = np.minimum(alloc.base, s_cap - 1)
        bs, ho = bank.prefix_sum(base), bank.sample_at(base)
        n2, g2, c2, dr2 = E.stochastic_core(variant, spp2, alloc.frac, alloc.u, bs, ho, cfg)
        d[f"es_{key}_drawn"] = dr2
        d[f"es_{key}_rawnoisy"] = n2
    return d


WARP_CASES = [
    # name, H, W, C, motion kind
    ("subpixel", 11, 13, 3, "uniform3"),
    ("integer", 9, 7, 3, "integer"),
    ("zero", 6, 8, 3, "zero"),
    ("large", 10, 12, 2, "uniform9"),
    ("single_channel", 5, 16, 1, "uniform2"),
]


def temporal(seed):
    """images.warp_array / warp_backward (images.py:88-147) on seeded inputs."""
    rng = np.random.default_rng(seed)
    d = {}
    for name, h, w, c, kind in WARP_CASES:
        if kind == "zero":
            motion = np.zeros((h, w, 2))
        elif kind == "integer":
            motion = rng.integers(-2, 3, (h, w, 2)).astype(np.float64)
        else:
            a = float(kind[len("uniform"):])
            motion = rng.uniform(-a, a, (h, w, 2))
        prev = rng.lognormal(-1.0, 1.5, (h, w, c))
        gout = rng.normal(0.0, 1.0, (h, w, c))
        out, valid = I.warp_array(prev, motion)
        d[f"{name}_motion"], d[f"{name}_prev"], d[f"{name}_gout"] = motion, prev, gout
        d[f"{name}_out"], d[f"{name}_validity"] = out, valid
        d[f"{name}_gprev"] = I.warp_backward(gout, motion)
    d["names"] = np.array([c[0] for c in WARP_CASES])
    return d


SCORE_CASES = [
    # name, H, W, frames, channels, budget, sigma
    ("blur", 12, 10, 2, 3, 0.25, 1.5),
    ("noblur", 9, 14, 2, 3, 0.5, 0.0),
    ("wide", 16, 16, 1, 3, 1.0, 2.5),
]


def scores(seed):
    """The sampler half of optimize.evaluate_step (optimize.py:244-251) written
    with the reference's own functions: density.softmax / softmax_backward and
    scipy's gaussian_filter(mode="nearest")."""
    rng = np.random.default_rng(seed)
    d = {}
    for name, h, w, f, c, budget, sigma in SCORE_CASES:
        sc = rng.normal(0.0, 1.0, (h, w))
        gi = rng.normal(0.0, 1.0, (f, h, w, c))
        gd = rng.normal(0.0, 1.0, (f, h, w, c)) * rng.uniform(0.1, 2.0, (f, h, w, 1))
        g_spp = None
        for k in range(f):
            t = (gi[k] * gd[k]).sum(axis=-1)
            g_spp = t if g_spp is None else g_spp + t
        if sigma > 0:
            g_spp = gaussian_filter(g_spp, sigma, mode="nearest")
        wts = D.softmax(sc)
        total = (7.0 / 8.0) * budget * wts.size
        d[f"{name}_scores"], d[f"{name}_gin"], d[f"{name}_gd"] = sc, gi, gd
        d[f"{name}_budget"], d[f"{name}_sigma"] = np.float64(budget), np.float64(sigma)
        d[f"{name}_gspp"] = g_spp
        d[f"{name}_gscores"] = total * D.softmax_backward(wts, g_spp)
    d["names"] = np.array([c[0] for c in SCORE_CASES])
    return d


def tonemap_losses(seed):
    """tonemap.tonemap_array / tonemap_backward, losses.spatial_loss /
    temporal_loss / combined_loss / make_mask("gradmag"), and the loss
    gradients as optimize.evaluate_step forms them (optimize.py:219-231, inline
    code there: restated here on the reference's own maps)."""
    rng = np.random.default_rng(seed)
    h, w = 13, 17
    d = {}
    tmos = [TM.TmoParams(), TM.sample_tmo(3), TM.sample_tmo(7)]
    rad = rng.lognormal(-1.0, 2.0, (h, w, 3))
    rad[0, :3] = [0.0, 1e-9, 5e-9]  # below the log floor (zero gradient)
    rad[1, 0] = 1e-12
    up = rng.normal(0.0, 1.0, (h, w, 3))
    d["rad"], d["up"] = rad, up
    for i, p in enumerate(tmos):
        d[f"tmo{i}"] = np.array([p.exposure, p.contrast, p.saturation, p.toe, p.shoulder])
        d[f"tm_ldr{i}"] = TM.tonemap_array(rad, p)
        d[f"gtm{i}"] = TM.tonemap_backward(rad, p, up)
    ldr1, ref, ldr0w, refw = (rng.uniform(0, 1, (h, w, 3)) for _ in range(4))
    ldr1[2, 2] = ref[2, 2]  # a sign(0) pixel
    validity = rng.choice([0.0, 0.5, 1.0], size=(h, w), p=[0.2, 0.1, 0.7])
    mask = LS.make_mask("gradmag", ref)
    d.update(ldr1=ldr1, ref=ref, ldr0w=ldr0w, refw=refw, validity=validity, mask=mask.weights)
    sp_map, sp = LS.spatial_loss(ldr1, ref, mask)
    tm_map, tm = LS.temporal_loss(ldr1, ldr0w, ref, refw, validity)
    cb_map, cb = LS.combined_loss(sp_map, tm_map)
    d.update(sp_map=sp_map, tm_map=tm_map, cb_map=cb_map, losses=np.array([sp, tm, cb]))
    n_pix = cb_map.size
    wins = (LS.TEMPORAL_WEIGHT * tm_map) > sp_map
    g_sp = (~wins).astype(np.float64) / n_pix
    g_tm = np.where(wins, LS.TEMPORAL_WEIGHT / n_pix, 0.0)
    d["g_ldr1"] = (np.sign(ldr1 - ref) * (g_sp * mask.weights)[..., None] / 3.0
                   + np.sign((ldr1 - ldr0w) - (ref - refw)) * g_tm[..., None] / 3.0)
    d["g_ldr0w"] = -np.sign((ldr1 - ldr0w) - (ref - refw)) * g_tm[..., None] / 3.0
    return d


def main(which=None):
    which = set(which or ["pyramid", "primitives", "placement", "temporal", "scores", "tonemap"])
    n = 0
    if "pyramid" in which:
        for i, case in enumerate(PYRAMID_CASES):
            d = pyramid_case(*case, seed=1000 + i)
            np.savez_compressed(os.path.join(HERE, f"{case[0]}.npz"), **d)
            n += 1
    for name, fn, seed in (("primitives", primitives, 77), ("placement", placement, 88),
                           ("temporal", temporal, 99), ("scores", scores, 111),
                           ("tonemap", tonemap_losses, 123)):
        if name in which:
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **fn(seed))
            n += 1
    print("wrote", n, "fixtures to", HERE)


if __name__ == "__main__":
    main(sys.argv[1:])  # e.g. `make_golden.py temporal scores` regenerates only those
