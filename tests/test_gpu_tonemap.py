"""GPU parity of the tonemap + loss epilogue through
the C ABI: tonemap.py:87-118, losses.py:58-91 and the loss gradient of
optimize.py:219-231, against the reference's golden outputs (float64) and the
oracle (float32)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import tonemap as otm  # noqa: E402
from tests._golden import load  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08642_b200 import ops as _ops
    return _ops


def planar(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).transpose(2, 0, 1))[None]).cuda().to(dtype)


def hwc(t):
    return t[0].permute(1, 2, 0).double().cpu().numpy()


def test_tonemap_f64_vs_reference(ops):
    d = load("tonemap")
    for i in range(3):
        t = tuple(d[f"tmo{i}"])
        ldr = hwc(ops.tonemap(planar(d["rad"]), t))
        np.testing.assert_allclose(ldr, d[f"tm_ldr{i}"], rtol=1e-13, atol=1e-15)
        g = hwc(ops.tonemap_backward(planar(d["rad"]), t, planar(d["up"])))
        ref = d[f"gtm{i}"]
        np.testing.assert_allclose(g, ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max())
        assert np.all(g[0, 0] == 0.0) and np.all(g[1, 0][ref[1, 0] == 0] == 0.0)  # below the log floor


def test_losses_f64_vs_reference(ops):
    d = load("tonemap")
    cu = lambda a: torch.from_numpy(np.asarray(a)[None]).cuda()  # noqa: E731
    r = ops.losses(planar(d["ldr1"]), planar(d["ref"]), planar(d["ldr0w"]), planar(d["refw"]),
                   validity=cu(d["validity"]), mask=cu(d["mask"]), want_grads=True)
    np.testing.assert_array_equal(r["spatial_map"][0].cpu().numpy(), d["sp_map"])
    np.testing.assert_array_equal(r["temporal_map"][0].cpu().numpy(), d["tm_map"])
    np.testing.assert_array_equal(r["combined_map"][0].cpu().numpy(), d["cb_map"])
    np.testing.assert_allclose(r["losses"][0].cpu().numpy(), d["losses"], rtol=1e-13)
    np.testing.assert_array_equal(hwc(r["g_ldr1"]), d["g_ldr1"])
    np.testing.assert_array_equal(hwc(r["g_ldr0_w"]), d["g_ldr0w"])


def test_tonemap_and_losses_f32_vs_oracle(ops):
    rng = np.random.default_rng(4)
    h, w = 135, 240
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    rad = f32(rng.lognormal(-1.0, 2.0, (h, w, 3)))
    up = f32(rng.normal(size=(h, w, 3)))
    t = (0.3, 1.1, 0.9, 0.4, 0.6)
    ldr = hwc(ops.tonemap(planar(rad, torch.float32), t))
    np.testing.assert_allclose(ldr, otm.tonemap(rad, t), rtol=1e-5, atol=1e-6)
    g = hwc(ops.tonemap_backward(planar(rad, torch.float32), t, planar(up, torch.float32)))
    gr = otm.tonemap_backward(rad, t, up)
    np.testing.assert_allclose(g, gr, rtol=1e-4, atol=1e-5 * np.abs(gr).max())
    a, b = f32(rng.uniform(0, 1, (h, w, 3))), f32(rng.uniform(0, 1, (h, w, 3)))
    r = ops.losses(planar(a, torch.float32), planar(b, torch.float32), want_grads=True)
    sp, _, _, vals = otm.losses(a, b)
    np.testing.assert_allclose(r["spatial_map"][0].double().cpu().numpy(), sp, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(r["losses"][0, 0].item(), vals[0], rtol=1e-6)
    g1, _ = otm.loss_grads(a, b)
    np.testing.assert_allclose(hwc(r["g_ldr1"]), g1, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("h,w", [(64, 96), (33, 51)])  # quad-vector kernels / scalar fallback
def test_tonemap_and_full_losses_f32_vs_oracle(ops, h, w):
    """float32: tonemap (all three filmic pieces), tonemap backward, and the
    single-pass loss kernel with the warped history, validity and a mask:
    maps, per-frame losses and both gradients."""
    rng = np.random.default_rng(h + w)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    B = 2
    t = (0.2, 1.3, 0.8, 0.35, 0.45)
    rad = [f32(rng.lognormal(-0.5, 2.5, (h, w, 3))) for _ in range(B)]
    up = [f32(rng.normal(size=(h, w, 3))) for _ in range(B)]
    stack = lambda xs: torch.cat([planar(x, torch.float32) for x in xs])  # noqa: E731
    ldr = ops.tonemap(stack(rad), t)
    g = ops.tonemap_backward(stack(rad), t, stack(up))
    for i in range(B):
        np.testing.assert_allclose(ldr[i].permute(1, 2, 0).double().cpu().numpy(), otm.tonemap(rad[i], t),
                                   rtol=1e-5, atol=1e-6)
        gr = otm.tonemap_backward(rad[i], t, up[i])
        np.testing.assert_allclose(g[i].permute(1, 2, 0).double().cpu().numpy(), gr, rtol=1e-4,
                                   atol=1e-5 * np.abs(gr).max())
    img = lambda: [f32(rng.uniform(0, 1, (h, w, 3))) for _ in range(B)]  # noqa: E731
    a1, rf, a0, rw = img(), img(), img(), img()
    val = [(rng.uniform(size=(h, w)) > 0.2).astype(np.float64) for _ in range(B)]
    msk = [f32(rng.uniform(0, 1, (h, w))) for _ in range(B)]
    tm = lambda xs: torch.from_numpy(np.stack(xs)).cuda().float()  # noqa: E731
    r = ops.losses(stack(a1), stack(rf), stack(a0), stack(rw), validity=tm(val), mask=tm(msk), want_grads=True)
    for i in range(B):
        sp, tmm, cb, vals = otm.losses(a1[i], rf[i], a0[i], rw[i], val[i], msk[i])
        for key, ref in (("spatial_map", sp), ("temporal_map", tmm), ("combined_map", cb)):
            np.testing.assert_allclose(r[key][i].double().cpu().numpy(), ref, rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(r["losses"][i].cpu().numpy(), vals, rtol=1e-6)
        g1, g0 = otm.loss_grads(a1[i], rf[i], a0[i], rw[i], val[i], msk[i])
        # the branch choice (temporal vs spatial) may flip on float32 near-ties
        agree = np.isclose(r["g_ldr1"][i].permute(1, 2, 0).double().cpu().numpy(), g1, rtol=1e-6, atol=1e-12)
        assert agree.mean() > 0.999
        agree0 = np.isclose(r["g_ldr0_w"][i].permute(1, 2, 0).double().cpu().numpy(), g0, rtol=1e-6, atol=1e-12)
        assert agree0.mean() > 0.999


@pytest.mark.parametrize("dtype,h,w,hist", [(torch.float64, 37, 53, True), (torch.float64, 16, 24, False),
                                             (torch.float32, 64, 96, True), (torch.float32, 33, 51, True),
                                             (torch.float32, 48, 64, False)])
def test_fused_epilogue_matches_composition(ops, dtype, h, w, hist):
    """ssb_epilogue == tonemap -> losses(want_grads) -> tonemap_backward:
    bit-identical in float64, within float32 rounding (and the same
    temporal/spatial branch on all but near-tie pixels) in float32."""
    gen = torch.Generator(device="cuda").manual_seed(h * w)
    B = 2
    rnd = lambda *s: torch.rand(s, device="cuda", dtype=dtype, generator=gen)  # noqa: E731
    rad = torch.exp(torch.randn((B, 3, h, w), device="cuda", dtype=dtype, generator=gen) * 2.0 - 0.5)
    ref = rnd(B, 3, h, w)
    l0w, rw = (rnd(B, 3, h, w), rnd(B, 3, h, w)) if hist else (None, None)
    val = (rnd(B, h, w) > 0.2).to(dtype) if hist else None
    msk = rnd(B, h, w)
    t = (0.2, 1.3, 0.8, 0.35, 0.45)
    f = ops.loss_epilogue(rad, ref, t, l0w, rw, validity=val, mask=msk, want_ldr=True)
    ldr = ops.tonemap(rad, t)
    r = ops.losses(ldr, ref, l0w, rw, validity=val, mask=msk, want_maps=False, want_grads=True)
    g = ops.tonemap_backward(rad, t, r["g_ldr1"])
    if dtype == torch.float64:
        assert torch.equal(f["ldr"], ldr)
        assert torch.equal(f["grad_radiance"], g)
        assert torch.equal(f["losses"], r["losses"])
        if hist:
            assert torch.equal(f["g_ldr0_w"], r["g_ldr0_w"])
    else:
        torch.testing.assert_close(f["ldr"], ldr, rtol=1e-5, atol=1e-6)
        torch.testing.assert_close(f["losses"], r["losses"], rtol=1e-5, atol=1e-9)
        close = torch.isclose(f["grad_radiance"], g, rtol=1e-4, atol=1e-5 * g.abs().max().item())
        assert close.float().mean().item() > 0.999
        if hist:
            assert torch.isclose(f["g_ldr0_w"], r["g_ldr0_w"]).float().mean().item() > 0.999


def test_losses_reject_bad_inputs(ops):
    x = torch.zeros((1, 3, 8, 8), device="cuda", dtype=torch.float64)
    with pytest.raises(ValueError):
        ops.losses(x, torch.zeros((1, 3, 8, 9), device="cuda", dtype=torch.float64))
    with pytest.raises(ValueError):
        ops.losses(x, x, ldr0_w=x)
    with pytest.raises(ValueError):
        ops.tonemap(x, (0.0, 1.0, 1.0, 1.5, 0.5))  # toe outside (0, 1)
