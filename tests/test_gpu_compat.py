"""The reference-signature compat layer (the drop-in boundary) on the GPU.

Restates the kinds of checks the reference's own suite makes for these
functions (closed-form values, invariants, finite-difference gradchecks,
golden outputs) against `paper_2602_08642_b200.compat`, in its default float64
mode (exact drop-in) and in float32 mode.  Reference tests these mirror:
pkg/tests/test_pyramid.py, test_density.py, test_rng.py, test_estimators.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from tests._golden import case_logits, load, pyramid_cases  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08642_b200 import compat
    compat.set_precision("f64")
    return compat


def field(P, w, h, seed, scale=0.7):
    rng = np.random.default_rng(seed)
    kf = P.zero_kernel_field(w, h)
    for a in kf.logits:
        a += rng.normal(0, scale, a.shape)
    return kf


# ---------------------------------------------------------------- pyramid
def test_layout_and_dims(cp):
    P = cp.pyramid
    assert P.level_dims(10, 7) == [(7, 10), (4, 5), (2, 3), (1, 2), (1, 1)]
    assert [P.kernel_channels(l) for l in (0, 2, 4)] == [54, 29, 25]
    with pytest.raises(ValueError):
        P.KernelField([np.zeros((4, 4, 54))])


def test_build_pyramid_properties(cp):
    P = cp.pyramid
    for lv in P.build_pyramid(np.full((16, 16, 3), 2.5)).levels:
        np.testing.assert_allclose(lv, 2.5)
    img = np.array([[[1.0], [2.0]], [[3.0], [4.0]]]) * np.ones(3)
    np.testing.assert_allclose(P.build_pyramid(img).levels[1][0, 0], 2.5)
    for lv in P.build_pyramid(np.ones((5, 7, 3))).levels:
        np.testing.assert_allclose(lv, 1.0)


def test_normalize_kernels(cp):
    P = cp.pyramid
    w = P.normalize_kernels(P.zero_kernel_field(8, 8))
    np.testing.assert_allclose(w[0], 1 / 54)
    np.testing.assert_allclose(w[1], 1 / 29)
    np.testing.assert_allclose(w[4], 1 / 25)
    kf = field(P, 8, 8, 3)
    w = P.normalize_kernels(kf, include_temporal=False)
    np.testing.assert_array_equal(w[0][:, :, 29:], 0.0)
    np.testing.assert_allclose(w[0].sum(-1), 1.0, atol=1e-12)


def test_gather_and_upsample_exact(cp):
    P = cp.pyramid
    rng = np.random.default_rng(4)
    img = rng.uniform(0, 3, (6, 6, 3))
    w = np.zeros((6, 6, 25))
    w[:, :, 12] = 1.0
    np.testing.assert_array_equal(P.gather5(img, w), img)
    coarse = rng.uniform(0, 2, (3, 3, 3))
    uw = np.zeros((6, 6, 4))
    uw[:, :, 0] = 1.0
    out = P.upsample2(coarse, uw)
    for y in range(6):
        for x in range(6):
            np.testing.assert_array_equal(out[y, x], coarse[y // 2, x // 2])


def test_reconstruct_properties(cp):
    P = cp.pyramid
    rng = np.random.default_rng(8)
    img = rng.uniform(0.1, 4.0, (16, 16, 3))
    kf = P.zero_kernel_field(16, 16)
    kf.logits[0][:, :, 12] = 60.0
    out, _ = P.reconstruct_core(img, kf, None, None)
    np.testing.assert_allclose(out, img, rtol=1e-6)
    demod = rng.uniform(0.05, 3.0, (16, 16, 3))
    out, _ = P.reconstruct_core(img, kf, None, demod)
    np.testing.assert_allclose(out, img, rtol=1e-6)
    kf = field(P, 12, 12, 9)
    out, _ = P.reconstruct_core(np.full((12, 12, 3), 0.8), kf, np.full((12, 12, 3), 0.8), None)
    np.testing.assert_allclose(out, 0.8, rtol=1e-9)
    for trial in range(5):
        kf = field(P, 8, 8, 100 + trial, 1.5)
        a, b = rng.uniform(0, 6, (8, 8, 3)), rng.uniform(0, 6, (8, 8, 3))
        out, _ = P.reconstruct_core(a, kf, b, None)
        lo, hi = min(a.min(), b.min()), max(a.max(), b.max())
        assert (out >= lo - 1e-9).all() and (out <= hi + 1e-9).all()
    res = P.reconstruct(P.build_pyramid(rng.uniform(0, 2, (8, 8, 3))), field(P, 8, 8, 14))
    assert res.data.shape == (8, 8, 3) and (res.data >= 0).all()


def test_backward_zero_and_footprint(cp):
    P = cp.pyramid
    rng = np.random.default_rng(16)
    kf = field(P, 8, 8, 15)
    img = rng.uniform(0, 2, (8, 8, 3))
    out, tape = P.reconstruct_core(img, kf, img.copy(), np.ones((8, 8, 3)))
    g = P.reconstruct_backward(tape, np.zeros_like(out))
    for gl in g.logits:
        np.testing.assert_array_equal(gl, 0.0)
    np.testing.assert_array_equal(g.demod, 0.0)
    np.testing.assert_array_equal(g.input, 0.0)
    kf = field(P, 16, 16, 17)
    img = rng.uniform(0.1, 2, (16, 16, 3))
    out, tape = P.reconstruct_core(img, kf, None, None)
    up = np.zeros_like(out)
    up[2, 2] = 1.0
    g = P.reconstruct_backward(tape, up)
    nz = np.nonzero(np.abs(g.logits[0]).sum(-1))
    assert set(zip(*nz)) == {(2, 2)}
    nz1 = np.abs(g.logits[1]).sum(-1)
    assert nz1[1, 1] != 0 and nz1[6:, 6:].max() == 0


def test_backward_gradcheck_every_group(cp):
    """Central differences through the compat API itself (float64)."""
    P = cp.pyramid
    rng = np.random.default_rng(19)
    noisy = rng.uniform(0.01, 3.0, (8, 8, 3))
    prev = rng.uniform(0.01, 3.0, (8, 8, 3))
    demod = rng.uniform(0.2, 2.0, (8, 8, 3))
    kf = field(P, 8, 8, 20)
    up = rng.normal(size=(8, 8, 3))
    out, tape = P.reconstruct_core(noisy, kf, prev, demod)
    g = P.reconstruct_backward(tape, up)

    def loss():
        return float((up * P.reconstruct_core(noisy, kf, prev, demod)[0]).sum())

    gscale = max(np.abs(gl).max() for gl in g.logits)
    eps = 1e-5
    groups = [(kf.logits[l], g.logits[l]) for l in range(5)] + [(demod, g.demod), (noisy, g.input),
                                                              (prev, g.prev)]
    for arr, grad in groups:
        for _ in range(5):
            idx = tuple(int(rng.integers(0, s)) for s in arr.shape)
            old = arr[idx]
            arr[idx] = old + eps
            lp = loss()
            arr[idx] = old - eps
            lm = loss()
            arr[idx] = old
            fd = (lp - lm) / (2 * eps)
            assert abs(grad[idx] - fd) <= 1e-3 * max(abs(fd), abs(grad[idx]), 1e-3 * gscale)


@pytest.mark.parametrize("name", pyramid_cases())
@pytest.mark.parametrize("precision,rtol", [("f64", 1e-10), ("f32", 2e-5)])
def test_golden_through_compat(cp, name, precision, rtol):
    d = load(name)
    levels = int(d["levels"])
    P = cp.pyramid
    cp.set_precision(precision)
    try:
        class KF:  # any object with .logits works, like the reference's KernelField
            logits = case_logits(d)
        out, tape = P.reconstruct_core(d["noisy"], KF, d.get("prev"), d.get("demod"))
        g = P.reconstruct_backward(tape, d["upstream"], want_param_grads=bool(d["want"]))
    finally:
        cp.set_precision("f64")
    scale = lambda a: rtol * np.abs(a).max()  # noqa: E731
    np.testing.assert_allclose(out, d["out"], rtol=rtol, atol=scale(d["out"]))
    np.testing.assert_allclose(g.input, d["g_input"], rtol=rtol, atol=scale(d["g_input"]))
    if bool(d["want"]):
        gs = max(np.abs(d[f"g_logits{l}"]).max() for l in range(levels))
        for l in range(levels):
            np.testing.assert_allclose(g.logits[l], d[f"g_logits{l}"], rtol=rtol, atol=rtol * gs)
        if "g_demod" in d:
            np.testing.assert_allclose(g.demod, d["g_demod"], rtol=rtol, atol=scale(d["g_demod"]))
    if "g_prev" in d:
        np.testing.assert_allclose(g.prev, d["g_prev"], rtol=rtol, atol=scale(d["g_prev"]))


# ---------------------------------------------------------------- density / rng
def test_normalize_density_kats(cp):
    D = cp.density
    np.testing.assert_allclose(D.normalize_density(np.zeros((4, 6)), 1.0).spp, 1.0)
    d = D.normalize_density(np.array([[1e4, 0.0], [0.0, 0.0]]), 1.0)
    assert d.spp[0, 0] == pytest.approx(0.125 + 0.875 * 4, rel=1e-9)
    assert d.spp[0, 1] == pytest.approx(0.125, rel=1e-9)
    rng = np.random.default_rng(1)
    for _ in range(5):
        b = float(rng.uniform(0.2, 4.0))
        sp = D.normalize_density(rng.normal(0, 3, (7, 5)), b).spp
        assert abs(sp.sum() - b * 35) <= 1e-4 * b * 35 and sp.min() >= b / 8 * (1 - 1e-12)
    with pytest.raises(ValueError):
        D.normalize_density(np.array([[np.inf, 0.0]]), 1.0)
    with pytest.raises(ValueError):
        D.normalize_density(np.zeros((2, 2)), 0.0)


def test_allocation_kats(cp):
    D = cp.density
    a = D.allocate(D.uniform_density(6, 6, 2.0), "stochastic", frame=0, seed=0)
    np.testing.assert_array_equal(a.base, 2)
    np.testing.assert_array_equal(a.frac, 0.0)
    assert not a.taken.any()
    a = D.allocate(D.uniform_density(400, 250, 0.5), "stochastic", frame=0, seed=0)
    assert abs(a.taken.mean() - 0.5) < 0.005
    u = np.array([[0.1, 0.6, 0.95]])
    f = np.array([[0.5, 0.5, 0.5]])
    np.testing.assert_array_equal(D.holdout_taken("stochastic", u, f), [[True, False, False]])
    np.testing.assert_array_equal(D.holdout_taken("relaxed", u, f), [[False, True, True]])
    with pytest.raises(ValueError):
        D.allocate(D.uniform_density(4, 4, 0.5), "dithered")
    with pytest.raises(ValueError):
        D.holdout_taken("nope", u, f)


def test_dithered_allocation(cp):
    D = cp.density
    g = load("placement")

    class Mask:
        rank = g["dm_rank"]
        size = rank.shape[0]

    t = Mask.size
    a = D.allocate(D.uniform_density(t, t, 0.5), "dithered", mask=Mask, frame=0)
    assert a.taken.sum() == t * t // 2
    a0 = D.allocate(D.uniform_density(t, t, 0.5), "dithered", mask=Mask, frame=0)
    a1 = D.allocate(D.uniform_density(t, t, 0.5), "dithered", mask=Mask, frame=1)
    assert not np.array_equal(a0.taken, a1.taken) and a0.taken.sum() == a1.taken.sum()


def test_rng(cp):
    R = cp.rng
    g = R.uniform_grid(9, 3, 5, 4, 1)
    for y in range(4):
        for x in range(5):
            assert g[y, x] == R.pixel_uniform(R.PixelRngKey(9, 3, x, y, 1))
    frames = np.array([0, 5, 17])
    b = R.uniform_grid_batch(2, frames, 6, 4, 3)
    for i, f in enumerate(frames):
        np.testing.assert_array_equal(b[i], R.uniform_grid(2, int(f), 6, 4, 3))
    assert R.pixel_uniform(R.PixelRngKey(1, 2, 3, 4, 5)) != R.pixel_uniform(R.PixelRngKey(1, 2, 3, 4, 6))


# ---------------------------------------------------------------- estimators
class Bank:
    """SampleBank-shaped bank: .samples (H, W, S, 3) and .capacity."""

    def __init__(self, samples):
        self.samples = samples
        self.capacity = samples.shape[2]


def _alloc(cp, spp, u_value, rule="stochastic"):
    base = np.floor(spp).astype(np.int64)
    frac = spp - base
    u = np.full(spp.shape, u_value)
    return cp._types.SampleAllocation(base, frac, u, cp.density.holdout_taken(rule, u, frac))


def test_estimator_kats(cp):
    E = cp.estimators
    rng = np.random.default_rng(0)
    bank = Bank(rng.uniform(0.5, 1.5, (4, 4, 16, 3)))
    d = cp._types.DensityMap(np.full((4, 4), 1.7), 1.7)
    res = E.estimate_stochastic(d, _alloc(cp, d.spp, 0.5), bank)
    np.testing.assert_allclose(res.noisy.data, (bank.samples[:, :, 0] + bank.samples[:, :, 1]) / 1.7)
    np.testing.assert_array_equal(res.samples_used, 2)
    np.testing.assert_allclose(res.grad_density, -res.noisy.data / 1.7)
    d = cp._types.DensityMap(np.full((4, 4), 0.25), 0.25)
    res = E.estimate_stochastic(d, _alloc(cp, d.spp, 0.8), bank)
    np.testing.assert_array_equal(res.noisy.data, 0.0)
    np.testing.assert_array_equal(res.samples_used, 0)
    d = cp._types.DensityMap(np.full((4, 4), 0.3), 0.3)
    res = E.estimate_relaxed(d, _alloc(cp, d.spp, 0.715, "relaxed"), bank,
                             cp._types.EstimatorConfig("relaxed", lam=10))
    np.testing.assert_allclose(res.holdout_contrib, bank.samples[:, :, 0] * (20.0 / 19.0) * 0.5)
    d = cp._types.DensityMap(np.full((4, 4), 0.5), 0.5)
    res = E.estimate_straight_through(d, _alloc(cp, d.spp, 0.9), bank)
    np.testing.assert_allclose(res.grad_density, bank.samples[:, :, 0] / 0.5)
    d = cp._types.DensityMap(np.full((4, 4), 1.0), 1.0)
    res = E.estimate_gumbel(d, _alloc(cp, d.spp, 0.5), bank, cp._types.EstimatorConfig("gumbel"))
    assert np.isfinite(res.grad_density).all()
    with pytest.raises(ValueError):
        E.estimate("stochastic", d, None, bank, cp._types.EstimatorConfig("stochastic"))


def test_stochastic_core_broadcasts_leading_axis(cp):
    """spp/frac (H, W) with u/base_sum/holdout over a leading K axis
    (ref estimators.py:95-97, optimize.py:430)."""
    from oracle import estimators as oe
    rng = np.random.default_rng(3)
    K, h, w = 6, 5, 7
    spp = rng.uniform(0.05, 2.5, (h, w))
    frac = spp - np.floor(spp)
    u = rng.uniform(size=(K, h, w))
    bs, ho = rng.uniform(0, 2, (K, h, w, 3)), rng.uniform(0, 2, (K, h, w, 3))
    cfg = cp._types.EstimatorConfig("relaxed", lam=10.0)
    got = cp.estimators.stochastic_core("relaxed", spp, frac, u, bs, ho, cfg)
    ref = oe.stochastic_core("relaxed", spp, frac, u, bs, ho, lam=10.0)
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- temporal warp
# mirrors pkg/tests/test_images.py::TestWarp on the drop-in (f64 and f32)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_warp_kats(cp, precision):
    cp.set_precision(precision)
    try:
        rng = np.random.default_rng(0)
        img = rng.uniform(0, 5, (6, 8, 3))
        out, validity = cp.images.warp_array(img, np.zeros((6, 8, 2)))
        np.testing.assert_allclose(out, img, rtol=1e-6)
        np.testing.assert_allclose(validity, 1.0)
        img = rng.uniform(0, 5, (6, 10, 3))
        out, _ = cp.images.warp_array(img, np.tile([3.0, 0.0], (6, 10, 1)))
        np.testing.assert_allclose(out[:, :7], img[:, 3:], rtol=1e-6)
        out, validity = cp.images.warp_array(np.ones((4, 4, 3)), np.tile([100.0, 0.0], (4, 4, 1)))
        np.testing.assert_array_equal(out, 0.0)
        np.testing.assert_array_equal(validity, 0.0)
        a, b = rng.uniform(0, 3, (5, 5, 3)), rng.uniform(0, 3, (5, 5, 3))
        m = rng.uniform(-1.5, 1.5, (5, 5, 2))
        wab, _ = cp.images.warp_array(2.0 * a + 3.0 * b, m)
        np.testing.assert_allclose(wab, 2.0 * cp.images.warp_array(a, m)[0] + 3.0 * cp.images.warp_array(b, m)[0],
                                   rtol=1e-5)
        img = rng.uniform(0, 2, (6, 7, 3))
        m = rng.uniform(-2, 2, (6, 7, 2))
        g = rng.normal(0, 1, (6, 7, 3))
        out, _ = cp.images.warp_array(img, m)
        gin = cp.images.warp_backward(g, m)
        assert np.isclose((out * g).sum(), (img * gin).sum(), rtol=1e-5)
        with pytest.raises(ValueError):
            cp.images.warp_array(img, np.zeros((5, 7, 2)))
    finally:
        cp.set_precision("f64")


def test_warp_golden_through_compat(cp):
    d = load("temporal")
    for n in d["names"]:
        out, val = cp.images.warp_array(d[f"{n}_prev"], d[f"{n}_motion"])
        np.testing.assert_array_equal(out, d[f"{n}_out"])
        np.testing.assert_array_equal(val, d[f"{n}_validity"])
        np.testing.assert_array_equal(cp.images.warp_backward(d[f"{n}_gout"], d[f"{n}_motion"]), d[f"{n}_gprev"])


def test_score_gradient_golden_through_compat(cp):
    d = load("scores")
    for n in d["names"]:
        r = cp.density.score_gradient(d[f"{n}_scores"], float(d[f"{n}_budget"]), list(d[f"{n}_gin"]),
                                      list(d[f"{n}_gd"]), float(d[f"{n}_sigma"]))
        ref = d[f"{n}_gscores"]
        np.testing.assert_allclose(r, ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())


# ---------------------------------------------------------------- tonemap + losses
# mirrors pkg/tests/test_tonemap.py / test_losses.py kinds of checks


def test_tonemap_losses_through_compat(cp):
    import types
    d = load("tonemap")
    t = d["tmo1"]
    p = types.SimpleNamespace(exposure=t[0], contrast=t[1], saturation=t[2], toe=t[3], shoulder=t[4])
    np.testing.assert_allclose(cp.tonemap.tonemap_array(d["rad"], p), d["tm_ldr1"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(cp.tonemap.tonemap_backward(d["rad"], p, d["up"]), d["gtm1"], rtol=1e-12,
                               atol=1e-13 * np.abs(d["gtm1"]).max())
    mask = types.SimpleNamespace(weights=d["mask"])
    sp_map, sp = cp.losses.spatial_loss(d["ldr1"], d["ref"], mask)
    np.testing.assert_array_equal(sp_map, d["sp_map"])
    assert abs(sp - d["losses"][0]) <= 1e-13 * abs(d["losses"][0])
    tm_map, tm = cp.losses.temporal_loss(d["ldr1"], d["ldr0w"], d["ref"], d["refw"], d["validity"])
    np.testing.assert_array_equal(tm_map, d["tm_map"])
    assert abs(tm - d["losses"][1]) <= 1e-13 * abs(d["losses"][1])
    g1, g0 = cp.losses.loss_gradients(d["ldr1"], d["ref"], d["ldr0w"], d["refw"], d["validity"], mask)
    np.testing.assert_array_equal(g1, d["g_ldr1"])
    np.testing.assert_array_equal(g0, d["g_ldr0w"])
    with pytest.raises(ValueError):
        cp.losses.spatial_loss(d["ldr1"], d["ref"][:-1], mask)
