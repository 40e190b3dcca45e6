"""GPU parity of sample placement vs the reference: counter-based uniforms,
density normalisation, allocation (counts + masks bit-exact given the same
uniforms), estimator core and the fused inference path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import density as od  # noqa: E402
from oracle import estimators as oe  # noqa: E402
from oracle import rng as orng  # noqa: E402
from tests._golden import load  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08642_b200 import ops as _ops
    return _ops


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def test_uniform_grid_bit_exact(ops):
    d = load("placement")
    for i in range(5):
        s, f, st = (int(v) for v in d[f"ug{i}_key"])
        u = ops.uniform_grid(s, 17, 23, frame0=f, stream_id=st)[0].cpu().numpy()
        np.testing.assert_array_equal(u, d[f"ug{i}"])
    ub = ops.uniform_grid(2, 11, 19, frames=d["ugb_frames"], stream_id=3).cpu().numpy()
    np.testing.assert_array_equal(ub, d["ugb"])


def test_uniform_grid_large_and_statistics(ops):
    u = ops.uniform_grid(1, 1080, 1920, frame0=4).cpu().numpy()[0]
    np.testing.assert_array_equal(u[::97, ::89], orng.uniform_grid(1, 4, 1920, 1080, 0)[::97, ::89])
    assert 0.0 <= u.min() and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.002


def test_normalize_density(ops):
    d = load("placement")
    for i in range(3):
        spp = ops.normalize_density(cu(d[f"nd{i}_scores"]), float(d[f"nd{i}_budget"]))
        np.testing.assert_allclose(spp[0].cpu().numpy(), d[f"nd{i}_spp"], rtol=1e-13)
    rng = np.random.default_rng(0)
    scores = rng.normal(0, 2, (2, 300, 500))
    spp = ops.normalize_density(cu(scores), 0.25).cpu().numpy()
    for b in range(2):
        ref = od.normalize_density(scores[b], 0.25)
        np.testing.assert_allclose(spp[b], ref, rtol=1e-12)
        assert abs(spp[b].sum() - 0.25 * spp[b].size) <= 1e-4 * 0.25 * spp[b].size
        assert spp[b].min() >= 0.25 / 8 * (1 - 1e-12)


@pytest.mark.parametrize("rule", ["stochastic", "relaxed", "gumbel"])
def test_allocate_bit_exact(ops, rule):
    d = load("placement")
    base, frac, u, taken = ops.allocate(cu(d["al_spp"]), frame0=11, seed=5, rule=rule,
                                        gumbel_temp=0.7)
    np.testing.assert_array_equal(base[0].cpu().numpy(), d[f"al_{rule}_base"])
    np.testing.assert_array_equal(frac[0].cpu().numpy(), d[f"al_{rule}_frac"])
    np.testing.assert_array_equal(u[0].cpu().numpy(), d[f"al_{rule}_u"])
    np.testing.assert_array_equal(taken[0].cpu().numpy(), d[f"al_{rule}_taken"])


def test_allocate_dithered_bit_exact(ops):
    d = load("placement")
    _, _, u, taken = ops.allocate(cu(d["al_spp"]), mode="dithered", rank=d["dm_rank"], frame0=5)
    np.testing.assert_array_equal(u[0].cpu().numpy(), d["dm_u"])
    np.testing.assert_array_equal(taken[0].cpu().numpy(), d["dm_taken"])


def test_allocate_1080p_counts_and_masks(ops):
    """BASELINE density at 1080p, 0.25 spp: the fp32-rounded spp fed to both
    sides; counts/masks bit-exact over a full frame batch."""
    rng = np.random.default_rng(1)
    from scipy.ndimage import gaussian_filter
    h, w = 1080, 1920
    g = gaussian_filter(rng.normal(size=(h, w)), 8, mode="wrap")
    g = (g - g.mean()) / g.std()
    scores = np.log(np.log1p(np.exp(g)))
    spp = od.normalize_density(scores, 0.25).astype(np.float32).astype(np.float64)
    spp_b = np.stack([spp, spp])
    base, frac, u, taken = ops.allocate(cu(spp_b), frame0=3, seed=9)
    for b in range(2):
        rb, rf, ru, rt = od.allocate(spp, frame=3 + b, seed=9)
        np.testing.assert_array_equal(base[b].cpu().numpy(), rb)
        np.testing.assert_array_equal(frac[b].cpu().numpy(), rf)
        np.testing.assert_array_equal(u[b].cpu().numpy(), ru)
        np.testing.assert_array_equal(taken[b].cpu().numpy(), rt)
    assert abs(taken.float().mean().item() - 0.25) < 0.01


@pytest.mark.parametrize("variant", ["stochastic", "relaxed", "straight-through", "gumbel"])
def test_estimate_matches_reference(ops, variant):
    d = load("placement")
    key = variant.replace("-", "_")
    spp = d["es_spp"]
    base = np.floor(spp).astype(np.int64)
    frac = spp - base
    noisy, grad, contrib, used, _ = ops.estimate(variant, cu(spp), cu(base), cu(frac),
                                                 cu(d[f"es_{key}_u"]), cu(d["es_samples"]),
                                                 lam=7.0, gumbel_temp=0.8)
    if variant == "gumbel":  # log/exp: tolerance-only
        cmp = lambda a, b: np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-300)  # noqa: E731
    else:
        cmp = np.testing.assert_array_equal
    cmp(noisy[0].cpu().numpy(), d[f"es_{key}_noisy"])
    cmp(grad[0].cpu().numpy(), d[f"es_{key}_grad"])
    cmp(contrib[0].cpu().numpy(), d[f"es_{key}_contrib"])
    np.testing.assert_array_equal(used[0].cpu().numpy(), d[f"es_{key}_used"])


@pytest.mark.parametrize("variant", ["stochastic", "relaxed", "straight-through", "gumbel"])
def test_stochastic_core_kat_and_random(ops, variant):
    rng = np.random.default_rng(2)
    n = 5000
    spp = rng.uniform(0.0, 3.0, n)
    spp[:7] = [0.0, 1.0, 2.0, 0.3, 0.25, 1.7, 1e-9]
    frac = spp - np.floor(spp)
    u = rng.uniform(size=n)
    u[:7] = [0.5, 0.99, 0.5, 0.715, 0.8, 0.5, 0.1]
    bs = rng.uniform(0, 2, (n, 3))
    ho = rng.lognormal(-1, 1.5, (n, 3))
    ref = oe.stochastic_core(variant, spp, frac, u, bs, ho, lam=10.0, gumbel_temp=1.0)
    got = ops.stochastic_core(variant, cu(spp), cu(frac), cu(u), cu(bs), cu(ho), lam=10.0)
    for a, b in zip(got, ref):
        a = a.cpu().numpy()
        if variant == "gumbel" and a.dtype != bool:
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-300)
        else:
            np.testing.assert_array_equal(a, b)


def test_place_fused_matches_oracle_pipeline(ops):
    rng = np.random.default_rng(4)
    B, h, w, S = 2, 240, 320, 2
    scores = rng.normal(0, 1, (B, h, w)).astype(np.float32)
    bank = rng.lognormal(-1.0, 1.5, (B, S, 3, h, w)).astype(np.float32)
    noisy, spp, taken = ops.place_fused(cu(scores), cu(bank), 0.25, seed=3, frame0=10,
                                        want_spp=True, want_taken=True)
    for b in range(B):
        spp_r = od.normalize_density(scores[b].astype(np.float64), 0.25)
        np.testing.assert_allclose(spp[b].cpu().numpy(), spp_r.astype(np.float32), rtol=1e-6)
        base, frac, u, tk = od.allocate(spp_r, frame=10 + b, seed=3)
        np.testing.assert_array_equal(taken[b].cpu().numpy().astype(bool), tk)
        samples = bank[b].transpose(2, 3, 0, 1).astype(np.float64)  # (H, W, S, 3)
        nr, _, _, _ = oe.estimate("stochastic", spp_r, base, frac, u, samples)
        np.testing.assert_allclose(noisy[b].permute(1, 2, 0).cpu().numpy(), nr, rtol=1e-6,
                                   atol=1e-7)


def _oracle_place(scores_b, bank_b, budget, variant, frame, seed, lam, temp):
    """The reference pipeline on one frame: normalize_density -> allocate with
    take_rule(variant) -> estimate over the materialised bank."""
    spp_r = od.normalize_density(scores_b.astype(np.float64), budget)
    rule = {"relaxed": "relaxed", "gumbel": "gumbel"}.get(variant, "stochastic")
    base, frac, u, tk = od.allocate(spp_r, frame=frame, seed=seed, rule=rule, gumbel_temp=temp)
    samples = bank_b.transpose(2, 3, 0, 1).astype(np.float64)  # (H, W, S, 3)
    nr, gr, _, used = oe.estimate(variant, spp_r, base, frac, u, samples, lam=lam, gumbel_temp=temp)
    drawn = used - np.minimum(base, samples.shape[2] - 1)
    return spp_r, tk, drawn.astype(bool), nr, gr


@pytest.mark.parametrize("variant", ["stochastic", "relaxed", "straight-through", "gumbel"])
@pytest.mark.parametrize("h,w,S,budget", [(96, 128, 2, 0.25), (45, 70, 2, 0.5), (64, 64, 4, 1.7),
                                          (33, 37, 3, 0.9)])
def test_place_all_variants_vs_oracle(ops, variant, h, w, S, budget):
    """ssb_place for every stochastic variant (the fused training path):
    taken (take_rule(variant)) and drawn bit-exact; noisy and the density
    gradient within fp32 rounding of the float64 reference pipeline.  Covers
    the float4 (W % 4 == 0) and scalar paths, S = 2 specialised and general S,
    budgets with base counts >= 1 (1.7 spp)."""
    rng = np.random.default_rng(h * w + S)
    B, lam, temp = 2, 7.0, 0.8
    scores = rng.normal(0, 1, (B, h, w)).astype(np.float32)
    bank = rng.lognormal(-1.0, 1.5, (B, S, 3, h, w)).astype(np.float32)
    r = ops.place(cu(scores), cu(bank), budget, variant, seed=11, frame0=5, lam=lam, gumbel_temp=temp,
                  want_grad=True, want_spp=True, want_taken=True, want_drawn=True)
    for b in range(B):
        spp_r, tk, dr, nr, gr = _oracle_place(scores[b], bank[b], budget, variant, 5 + b, 11, lam, temp)
        np.testing.assert_allclose(r["spp"][b].cpu().numpy(), spp_r.astype(np.float32), rtol=1e-6)
        np.testing.assert_array_equal(r["taken"][b].cpu().numpy().astype(bool), tk)
        np.testing.assert_array_equal(r["drawn"][b].cpu().numpy().astype(bool), dr)
        np.testing.assert_allclose(r["noisy"][b].permute(1, 2, 0).cpu().numpy(), np.maximum(nr, 0.0),
                                   rtol=2e-6, atol=1e-30)
        np.testing.assert_allclose(r["grad"][b].permute(1, 2, 0).cpu().numpy(), gr, rtol=2e-6,
                                   atol=2e-6 * np.abs(gr).max())


def test_place_1080p_baseline_frame_counts_exact(ops):
    """A full BASELINE-distribution 1080p frame (GRF density, 0.25 spp): every
    pixel's holdout decision equals the reference allocation's."""
    import scipy.ndimage as ndi
    rng = np.random.default_rng(21)
    h, w = 1080, 1920
    z = ndi.gaussian_filter(rng.normal(size=(h, w)), 8, mode="wrap")
    z = (z - z.mean()) / z.std()
    scores = np.log(np.log1p(np.exp(z))).astype(np.float32)[None]
    bank = rng.lognormal(-1.0, 1.5, (1, 2, 3, h, w)).astype(np.float32)
    r = ops.place(cu(scores), cu(bank), 0.25, "stochastic", seed=1234, frame0=3, want_taken=True)
    spp_r, tk, _, nr, _ = _oracle_place(scores[0], bank[0], 0.25, "stochastic", 3, 1234, 10.0, 1.0)
    got = r["taken"][0].cpu().numpy().astype(bool)
    assert got.mean() > 0.2
    np.testing.assert_array_equal(got, tk)
    np.testing.assert_allclose(r["noisy"][0].permute(1, 2, 0).cpu().numpy(), nr, rtol=2e-6, atol=1e-30)
