"""GPU parity of the temporal warp (images.py:88-147) and of the estimator
backward to the density scores (optimize.py:244-251) -- SURVEY.md 8(f) rows 2
and 3 -- through the C ABI, against the reference's golden outputs and the
oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import scores as osc  # noqa: E402
from oracle import temporal as ot  # noqa: E402
from tests._golden import load  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08642_b200 import ops as _ops
    return _ops


def planar(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).transpose(2, 0, 1))[None]).cuda().to(dtype)


def hwc(t):
    return t[0].permute(1, 2, 0).double().cpu().numpy()


def test_warp_f64_bit_exact_vs_reference(ops):
    d = load("temporal")
    for n in d["names"]:
        out, val = ops.warp(planar(d[f"{n}_prev"], torch.float64), planar(d[f"{n}_motion"], torch.float64))
        np.testing.assert_array_equal(hwc(out), d[f"{n}_out"], err_msg=str(n))
        np.testing.assert_array_equal(val[0].cpu().numpy(), d[f"{n}_validity"], err_msg=str(n))
        gp = ops.warp_backward(planar(d[f"{n}_gout"], torch.float64), planar(d[f"{n}_motion"], torch.float64))
        np.testing.assert_array_equal(hwc(gp), d[f"{n}_gprev"], err_msg=str(n))


def test_warp_f32_vs_oracle(ops):
    rng = np.random.default_rng(3)
    h, w = 67, 131
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    prev = f32(rng.lognormal(-1, 1.5, (h, w, 3)))
    g = f32(rng.normal(size=(h, w, 3)))
    m = f32(rng.uniform(-5, 5, (h, w, 2)))
    out_r, val_r = ot.warp_array(prev, m)
    gp_r = ot.warp_backward(g, m)
    out, val = ops.warp(planar(prev, torch.float32), planar(m, torch.float32))
    gp = ops.warp_backward(planar(g, torch.float32), planar(m, torch.float32))
    np.testing.assert_allclose(hwc(out), out_r, rtol=1e-5, atol=1e-5 * np.abs(out_r).max())
    np.testing.assert_allclose(val[0].double().cpu().numpy(), val_r, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(hwc(gp), gp_r, rtol=1e-5, atol=1e-5 * np.abs(gp_r).max())


@pytest.mark.parametrize("amp,c,h,w", [(0.4, 3, 45, 77), (2.0, 3, 67, 131), (3.0, 3, 40, 33),
                                       (2.0, 4, 37, 70), (1.5, 1, 19, 200), (3.0, 3, 1, 9)])
def test_warp_f32_small_motion_vs_oracle(ops, amp, c, h, w):
    """max|motion| <= 3: the staged forward gather and the landing-mask
    transpose (temporal.cu), incl. channel counts other than 3 and borders."""
    rng = np.random.default_rng(int(amp * 10) + c + h)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    prev = f32(rng.lognormal(-1, 1.5, (h, w, c)))
    g = f32(rng.normal(size=(h, w, c)))
    m = f32(rng.uniform(-amp, amp, (h, w, 2)))
    m[0, 0] = (amp, -amp)  # the extreme offsets
    out_r, val_r = ot.warp_array(prev, m)
    gp_r = ot.warp_backward(g, m)
    out, val = ops.warp(planar(prev, torch.float32), planar(m, torch.float32))
    gp = ops.warp_backward(planar(g, torch.float32), planar(m, torch.float32))
    np.testing.assert_allclose(hwc(out), out_r, rtol=1e-5, atol=1e-5 * np.abs(out_r).max())
    np.testing.assert_allclose(val[0].double().cpu().numpy(), val_r, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(hwc(gp), gp_r, rtol=1e-5, atol=1e-5 * np.abs(gp_r).max())


def test_warp_f32_integer_motion_vs_oracle(ops):
    """Integer-valued motion (fractions 0: one tap weight 1, three 0) through
    the staged warp and the landing-mask transpose, incl. the |o| = 2 and
    |o| = 3 mask layouts."""
    rng = np.random.default_rng(5)
    h, w = 41, 72
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    for amp in (2, 3):
        prev = f32(rng.lognormal(-1, 1.0, (h, w, 3)))
        g = f32(rng.normal(size=(h, w, 3)))
        m = rng.integers(-amp, amp + 1, (h, w, 2)).astype(np.float64)
        out_r, val_r = ot.warp_array(prev, m)
        gp_r = ot.warp_backward(g, m)
        out, val = ops.warp(planar(prev, torch.float32), planar(m, torch.float32))
        gp = ops.warp_backward(planar(g, torch.float32), planar(m, torch.float32))
        np.testing.assert_allclose(hwc(out), out_r, rtol=1e-5, atol=1e-5 * np.abs(out_r).max())
        np.testing.assert_allclose(val[0].double().cpu().numpy(), val_r, rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(hwc(gp), gp_r, rtol=1e-5, atol=1e-5 * np.abs(gp_r).max())


def test_warp_f32_deterministic_and_adjoint_1080p(ops):
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((2, 3, 1080, 1920), device="cuda", generator=gen)
    g = torch.randn((2, 3, 1080, 1920), device="cuda", generator=gen)
    m = (torch.rand((2, 2, 1080, 1920), device="cuda", generator=gen) - 0.5) * 4
    y, _ = ops.warp(x, m)
    gt1 = ops.warp_backward(g, m)
    gt2 = ops.warp_backward(g, m)
    assert torch.equal(gt1, gt2)
    lhs, rhs = (y.double() * g.double()).sum().item(), (x.double() * gt1.double()).sum().item()
    assert abs(lhs - rhs) <= 1e-5 * (y.double().abs() * g.double().abs()).sum().item()


def test_warp_backward_deterministic_and_adjoint_1080p(ops):
    """Size-independent properties at 1080p: bitwise run-to-run determinism of
    the gather-transpose and <warp(x), g> = <x, warp^T(g)>."""
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((1, 3, 1080, 1920), device="cuda", dtype=torch.float64, generator=gen)
    g = torch.randn((1, 3, 1080, 1920), device="cuda", dtype=torch.float64, generator=gen)
    m = (torch.rand((1, 2, 1080, 1920), device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 6
    y, _ = ops.warp(x, m)
    gt1 = ops.warp_backward(g, m)
    gt2 = ops.warp_backward(g, m)
    assert torch.equal(gt1, gt2)
    lhs, rhs = (y * g).sum().item(), (x * gt1).sum().item()
    assert abs(lhs - rhs) <= 1e-9 * abs(lhs) + 1e-6


def test_warp_rejects_bad_shapes(ops):
    x = torch.zeros((1, 3, 8, 8), device="cuda")
    with pytest.raises(ValueError):
        ops.warp(x, torch.zeros((1, 2, 8, 9), device="cuda"))
    with pytest.raises(ValueError):
        ops.warp(x, torch.zeros((1, 3, 8, 8), device="cuda"))


def _score_inputs(d, n, dtype):
    gi = torch.from_numpy(np.ascontiguousarray(d[f"{n}_gin"].transpose(0, 3, 1, 2))[None]).cuda().to(dtype)
    gd = torch.from_numpy(np.ascontiguousarray(d[f"{n}_gd"].transpose(0, 3, 1, 2))[None]).cuda().to(dtype)
    sc = torch.from_numpy(d[f"{n}_scores"][None]).cuda().to(dtype)
    return sc, gi, gd


def test_score_grad_f64_vs_reference(ops):
    d = load("scores")
    for n in d["names"]:
        sc, gi, gd = _score_inputs(d, n, torch.float64)
        r = ops.score_grad(sc, gi, gd, float(d[f"{n}_budget"]), float(d[f"{n}_sigma"]))[0].cpu().numpy()
        ref = d[f"{n}_gscores"]
        np.testing.assert_allclose(r, ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max(), err_msg=str(n))


def test_score_grad_f32_vs_oracle(ops):
    rng = np.random.default_rng(11)
    h, w = 135, 240
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    sc = f32(rng.normal(size=(h, w)))
    gi = f32(rng.normal(size=(2, h, w, 3)))
    gd = f32(rng.normal(size=(2, h, w, 3)))
    ref = osc.score_grad(sc, 0.25, list(gi), list(gd), 1.5)
    d = {"x_gin": gi, "x_gd": gd, "x_scores": sc}
    s_t, gi_t, gd_t = _score_inputs(d, "x", torch.float32)
    r = ops.score_grad(s_t, gi_t, gd_t, 0.25, 1.5)[0].double().cpu().numpy()
    np.testing.assert_allclose(r, ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())


@pytest.mark.parametrize("sigma,h,w,f,c", [(0.0, 64, 96, 1, 3), (0.6, 37, 53, 2, 3), (1.5, 64, 100, 3, 1),
                                           (3.9, 70, 44, 2, 3), (1.5, 1, 257, 2, 3)])
def test_score_grad_f32_configs_vs_oracle(ops, sigma, h, w, f, c):
    """float32 estimator backward across blur radii 0..16 (the radius-templated
    tiles), frame / channel counts, quad-vector and scalar shapes, B = 2."""
    rng = np.random.default_rng(int(sigma * 10) + h + w)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    cases = [(f32(rng.normal(size=(h, w))), f32(rng.normal(size=(f, h, w, c))), f32(rng.normal(size=(f, h, w, c))))
             for _ in range(2)]
    refs = [osc.score_grad(sc, 0.25, list(gi), list(gd), sigma) for sc, gi, gd in cases]
    ins = [_score_inputs({"x_gin": gi, "x_gd": gd, "x_scores": sc}, "x", torch.float32) for sc, gi, gd in cases]
    r = ops.score_grad(torch.cat([i[0] for i in ins]), torch.cat([i[1] for i in ins]),
                       torch.cat([i[2] for i in ins]), 0.25, sigma).double().cpu().numpy()
    for k in range(2):
        np.testing.assert_allclose(r[k], refs[k], rtol=1e-5, atol=1e-5 * np.abs(refs[k]).max())


def test_score_grad_sums_to_zero(ops):
    """softmax backward: sum(g_scores) = 0 per frame (any g_spp)."""
    gen = torch.Generator(device="cuda").manual_seed(1)
    sc = torch.randn((2, 540, 960), device="cuda", dtype=torch.float64, generator=gen)
    gi = torch.randn((2, 2, 3, 540, 960), device="cuda", dtype=torch.float64, generator=gen)
    gd = torch.randn((2, 2, 3, 540, 960), device="cuda", dtype=torch.float64, generator=gen)
    g = ops.score_grad(sc, gi, gd, 0.25, 1.5)
    tot = g.abs().sum(dim=(1, 2))
    assert torch.all(g.sum(dim=(1, 2)).abs() <= 1e-9 * tot)


@pytest.mark.parametrize("case", ["outlier", "pan", "nonfinite", "chaos"])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_warp_backward_large_motion(ops, case, precision):
    """max |motion| + 1 > 16 takes the O(HW) segment-candidate path (ADVICE
    r01: one 64-px vector, or an inf, used to turn every pixel's source scan
    frame-wide): float64 bit-exact to the reference's np.add.at order, float32
    within 1e-5; infinite motion lands nowhere, as in the reference."""
    rng = np.random.default_rng(len(case))
    h, w = 70, 150
    m = rng.uniform(-2, 2, (h, w, 2))
    if case == "outlier":
        m[33, 71] = (64.3, -20.7)
        m[5, 140] = (-139.5, 60.25)
    elif case == "pan":
        m += np.array([37.25, -19.5])
    elif case == "nonfinite":
        m[10, 10] = (np.inf, 0.5)  # (NaN motion makes the reference itself raise: not an input)
        m[40, 100] = (3.0, -np.inf)
        m[1, 2] = (25.0, 3.0)
    else:
        m = rng.uniform(-80, 80, (h, w, 2))
    g = rng.normal(size=(h, w, 3))
    if precision == "f32":
        m = m.astype(np.float32).astype(np.float64)
        g = g.astype(np.float32).astype(np.float64)
    ref = ot.warp_backward(g, m)
    dt = torch.float64 if precision == "f64" else torch.float32
    gp = hwc(ops.warp_backward(planar(g, dt), planar(m, dt)))
    if precision == "f64":
        np.testing.assert_array_equal(gp, ref)
    else:
        np.testing.assert_allclose(gp, ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())
