"""GPU parity of the gather-pyramid filter (forward + backward) vs the reference.

Golden fixtures are outputs of the unmodified reference; larger and k != 5
cases compare against the oracle restatement (itself pinned to the fixtures).
Tolerances (north star): float64 path ~1e-10; float32 path rtol 1e-5 with an
atol floor of 1e-5 * max|ref| (softmax-backward cancellation); bf16 logits
rtol 2e-2 with a 2e-2 * max|ref| floor.  Every floor is taken per tensor and,
for the logit gradients, per LEVEL (`assert_levels_close`), and every tensor
also meets a relative-L2 bound of rtol.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import pyramid as op  # noqa: E402
from tests._conv import (assert_close, assert_levels_close, device_glogits_to_ref,  # noqa: E402
                         hwc_to_planar, planar_to_hwc, ref_logits_to_device)
from tests._golden import case_logits, load, pyramid_cases  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08642_b200 import ops as _ops
    return _ops


def run_case(ops, noisy, logits_ref, demod, prev, up, k, dtype, logit_dtype=None, want=True,
             blend="native"):
    temporal = prev is not None
    ldt = logit_dtype or dtype
    n = hwc_to_planar(noisy, dtype)
    lg = ref_logits_to_device(logits_ref, k, temporal, ldt)
    dm = hwc_to_planar(demod, dtype) if demod is not None else None
    pv = hwc_to_planar(prev, dtype) if prev is not None else None
    out, tape = ops.pyramid_forward(n, lg, dm, pv, ksize=k, blend=blend)
    g = ops.pyramid_backward(tape, hwc_to_planar(up, dtype), want_param_grads=want)
    torch.cuda.synchronize()
    res = {"out": planar_to_hwc(out), "g_input": planar_to_hwc(g.input)}
    if want:
        res["g_logits"] = device_glogits_to_ref(g.logits, logits_ref, k, temporal)
        if g.demod is not None:
            res["g_demod"] = planar_to_hwc(g.demod)
    if g.prev is not None:
        res["g_prev"] = planar_to_hwc(g.prev)
    return res


def compare(res, ref, rtol, levels, want):
    assert_close(res["out"], ref["out"], rtol, "out")
    assert_close(res["g_input"], ref["g_input"], rtol, "g_input")
    if want:
        assert len(res["g_logits"]) == levels
        assert_levels_close(res["g_logits"], ref["g_logits"], rtol, scales=ref.get("scales"))
        if "g_demod" in ref:
            assert_close(res["g_demod"], ref["g_demod"], rtol, "g_demod")
    if "g_prev" in ref:
        assert_close(res["g_prev"], ref["g_prev"], rtol, "g_prev")


@pytest.mark.parametrize("name", pyramid_cases())
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_golden_cases(ops, name, precision):
    d = load(name)
    want = bool(d["want"])
    dtype = torch.float64 if precision == "f64" else torch.float32
    if precision == "f32":
        # feed the fp32-rounded inputs to the reference arithmetic (oracle)
        rnd = lambda a: None if a is None else a.astype(np.float32).astype(np.float64)  # noqa: E731
        inputs = dict(noisy=rnd(d["noisy"]), demod=rnd(d.get("demod")), prev=rnd(d.get("prev")),
                      up=rnd(d["upstream"]))
        logits = [rnd(z) for z in case_logits(d)]
        out, tape = op.forward(inputs["noisy"], logits, inputs["prev"], inputs["demod"])
        g = op.backward(tape, inputs["up"], want_param_grads=want)
        ref = {"out": out, "g_input": g.input, "g_logits": g.logits, "g_demod": g.demod,
               "g_prev": g.prev, "scales": g.operand_scale}
        ref = {k: v for k, v in ref.items() if v is not None}
        rtol = 1e-5
    else:
        inputs = dict(noisy=d["noisy"], demod=d.get("demod"), prev=d.get("prev"), up=d["upstream"])
        logits = case_logits(d)
        ref = {"out": d["out"], "g_input": d["g_input"]}
        if want:
            ref["g_logits"] = [d[f"g_logits{l}"] for l in range(int(d["levels"]))]
            # operand scales of the same inputs (the oracle is bit-exact to the goldens)
            _, tp = op.forward(inputs["noisy"], logits, inputs["prev"], inputs["demod"])
            ref["scales"] = op.backward(tp, inputs["up"]).operand_scale
            if "g_demod" in d:
                ref["g_demod"] = d["g_demod"]
        if "g_prev" in d:
            ref["g_prev"] = d["g_prev"]
        rtol = 1e-10
    res = run_case(ops, inputs["noisy"], logits, inputs["demod"], inputs["prev"], inputs["up"], 5,
                   dtype, want=want)
    compare(res, ref, rtol, int(d["levels"]), want)


def oracle_case(h, w, L, k, seed, demod=True, prev=False, blend="native", scale=1.0):
    rng = np.random.default_rng(seed)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    logits = [f32(z) for z in op.random_logits(h, w, L, k, rng, temporal=prev, blend=blend,
                                               scale=scale)]
    noisy = f32(rng.lognormal(-1.0, 1.5, (h, w, 3)))
    dm = f32(rng.uniform(0.05, 1.0, (h, w, 3))) if demod else None
    pv = f32(rng.uniform(0.01, 2.0, (h, w, 3))) if prev else None
    up = f32(rng.normal(size=(h, w, 3)))
    out, tape = op.forward(noisy, logits, pv, dm, k=k, blend=blend)
    g = op.backward(tape, up)
    ref = {"out": out, "g_input": g.input, "g_logits": g.logits, "scales": g.operand_scale}
    if dm is not None:
        ref["g_demod"] = g.demod
    if pv is not None:
        ref["g_prev"] = g.prev
    return noisy, logits, dm, pv, up, ref


@pytest.mark.parametrize("h,w,L,k,prev,blend", [
    (64, 80, 3, 5, False, "native"),
    (67, 45, 4, 5, False, "native"),
    (130, 70, 3, 7, False, "native"),
    (41, 77, 4, 3, False, "native"),
    (33, 29, 3, 7, True, "native"),
    (50, 61, 3, 5, True, "native"),
    (48, 40, 3, 5, False, "tied"),
    (37, 52, 4, 7, False, "tied"),
    (3, 2, 2, 7, False, "native"),
    (1, 9, 2, 5, False, "native"),
    (200, 1, 3, 5, True, "native"),
    (256, 256, 4, 5, False, "native"),
    # history on the TMA path (W % 4 == 0): level 0 by the log-sum-exp
    # weights + the temporal pass, in the level-0-last order
    (64, 80, 3, 5, True, "native"),
    (72, 128, 4, 7, True, "native"),
    (45, 96, 3, 3, True, "native"),
    (48, 40, 3, 5, True, "tied"),
    (37, 52, 4, 7, True, "tied"),
])
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_oracle_cases(ops, h, w, L, k, prev, blend, precision):
    noisy, logits, dm, pv, up, ref = oracle_case(h, w, L, k, seed=h * 1000 + w + k, prev=prev,
                                                 blend=blend)
    dtype = torch.float32 if precision == "f32" else torch.float64
    temporal = prev
    n = hwc_to_planar(noisy, dtype)
    lg = [hwc_to_planar(z, dtype) for z in logits]
    d = hwc_to_planar(dm, dtype) if dm is not None else None
    p = hwc_to_planar(pv, dtype) if pv is not None else None
    out, tape = ops.pyramid_forward(n, lg, d, p, ksize=k, blend=blend)
    g = ops.pyramid_backward(tape, hwc_to_planar(up, dtype))
    rtol = 1e-5 if precision == "f32" else 1e-10
    assert_close(planar_to_hwc(out), ref["out"], rtol, "out")
    assert_close(planar_to_hwc(g.input), ref["g_input"], rtol, "g_input")
    assert_levels_close([planar_to_hwc(z) for z in g.logits], ref["g_logits"], rtol, scales=ref["scales"])
    if dm is not None:
        assert_close(planar_to_hwc(g.demod), ref["g_demod"], rtol, "g_demod")
    if temporal:
        assert_close(planar_to_hwc(g.prev), ref["g_prev"], rtol, "g_prev")


@pytest.mark.parametrize("k,L,h,w", [(5, 3, 90, 132), (7, 4, 90, 132), (7, 4, 72, 128), (5, 3, 64, 96),
                                     (3, 3, 72, 128), (3, 4, 64, 112)])
def test_bf16_logits(ops, k, L, h, w):
    """bf16 logits, fp32 radiance and accumulation: within 2e-2 of the oracle
    fed the bf16-rounded logits.  W % 8 == 0 at every level (72 x 128, 64 x
    96) runs the TMA level kernels (bf16 rows must be 16-B multiples; k = 7:
    the pixel-pair forward), the other sizes the generic kernels."""
    rng = np.random.default_rng(7)
    lg32 = [torch.from_numpy(z.astype(np.float32)) for z in
            op.random_logits(h, w, L, k, rng, temporal=False)]
    lgb = [z.to(torch.bfloat16) for z in lg32]
    logits = [z.double().numpy() for z in lgb]
    noisy = rng.lognormal(-1.0, 1.5, (h, w, 3)).astype(np.float32).astype(np.float64)
    dm = rng.uniform(0.05, 1.0, (h, w, 3)).astype(np.float32).astype(np.float64)
    up = rng.normal(size=(h, w, 3)).astype(np.float32).astype(np.float64)
    out_r, tape = op.forward(noisy, logits, None, dm, k=k)
    g_r = op.backward(tape, up)
    dev_lg = [hwc_to_planar(z, torch.bfloat16) for z in logits]  # exact: values are bf16
    out, t = ops.pyramid_forward(hwc_to_planar(noisy, torch.float32), dev_lg,
                                 hwc_to_planar(dm, torch.float32), ksize=k)
    g = ops.pyramid_backward(t, hwc_to_planar(up, torch.float32))
    assert g.logits[0].dtype == torch.bfloat16
    assert_close(planar_to_hwc(out), out_r, 2e-2)
    assert_close(planar_to_hwc(g.input), g_r.input, 2e-2)
    assert_close(planar_to_hwc(g.demod), g_r.demod, 2e-2)
    assert_levels_close([planar_to_hwc(z) for z in g.logits], g_r.logits, 2e-2, scales=g_r.operand_scale)


def test_many_channels_batched_draws(ops):
    """C = 3K channels share one weight set (the batched-draws convention,
    ref optimize.py:433-437): parity incl. g_logits summed over all channels."""
    rng = np.random.default_rng(3)
    h, w, L, k, K = 40, 36, 3, 5, 5
    logits = op.random_logits(h, w, L, k, rng, temporal=False)
    noisy = rng.uniform(0.01, 2, (h, w, 3 * K))
    dm = np.tile(rng.uniform(0.1, 1, (h, w, 3)), (1, 1, K))
    up = rng.normal(size=(h, w, 3 * K))
    out_r, tape = op.forward(noisy, logits, None, dm, k=k)
    g_r = op.backward(tape, up)
    out, t = ops.pyramid_forward(hwc_to_planar(noisy), [hwc_to_planar(z) for z in logits],
                                 hwc_to_planar(dm), ksize=k)
    g = ops.pyramid_backward(t, hwc_to_planar(up))
    assert_close(planar_to_hwc(out), out_r, 1e-10)
    assert_close(planar_to_hwc(g.input), g_r.input, 1e-10)
    assert_close(planar_to_hwc(g.demod), g_r.demod, 1e-10)
    for l in range(L):
        assert_close(planar_to_hwc(g.logits[l]), g_r.logits[l], 1e-10)


def test_batch_equals_single_frames_bitwise(ops):
    rng = np.random.default_rng(11)
    B, h, w, L, k = 3, 70, 90, 3, 5
    dev = "cuda"
    noisy = torch.rand(B, 3, h, w, device=dev) + 0.01
    dm = torch.rand(B, 3, h, w, device=dev) * 0.9 + 0.05
    lg = [torch.randn(B, ops.logit_channels(l, L, k), hh, ww, device=dev)
          for l, (hh, ww) in enumerate(ops.level_shapes(h, w, L))]
    up = torch.randn(B, 3, h, w, device=dev)
    out, t = ops.pyramid_forward(noisy, lg, dm, ksize=k)
    g = ops.pyramid_backward(t, up)
    for b in range(B):
        o1, t1 = ops.pyramid_forward(noisy[b:b + 1].contiguous(), [z[b:b + 1].contiguous() for z in lg],
                                     dm[b:b + 1].contiguous(), ksize=k)
        g1 = ops.pyramid_backward(t1, up[b:b + 1].contiguous())
        assert torch.equal(o1[0], out[b])
        assert torch.equal(g1.input[0], g.input[b])
        assert torch.equal(g1.demod[0], g.demod[b])
        for l in range(L):
            assert torch.equal(g1.logits[l][0], g.logits[l][b])
    del rng


@pytest.mark.parametrize("h,w,L,k,ldt", [(1080, 1920, 3, 5, torch.float32),
                                         (2160, 3840, 4, 7, torch.bfloat16)])
def test_full_size_properties(ops, h, w, L, k, ldt):
    """Size-independent checks at the BASELINE sizes: adjointness
    <up, out> = <g_noisy, noisy> (out is linear in noisy for fixed logits),
    per-pixel sum of logit gradients = 0 (softmax), constant-input
    preservation, and run-to-run determinism."""
    torch.manual_seed(0)
    dev = "cuda"
    noisy = torch.rand(1, 3, h, w, device=dev) * 2
    dm = torch.rand(1, 3, h, w, device=dev) * 0.95 + 0.05
    lg = [torch.randn(1, ops.logit_channels(l, L, k), hh, ww, device=dev).to(ldt)
          for l, (hh, ww) in enumerate(ops.level_shapes(h, w, L))]
    up = torch.randn(1, 3, h, w, device=dev)
    out, t = ops.pyramid_forward(noisy, lg, dm, ksize=k)
    g = ops.pyramid_backward(t, up)
    lhs = (up.double() * out.double()).sum().item()
    rhs = (g.input.double() * noisy.double()).sum().item()
    assert abs(lhs - rhs) <= 1e-4 * abs(lhs)
    for l in range(L):
        s = g.logits[l].float().sum(dim=1)
        scale = g.logits[l].float().abs().amax(dim=1) + 1e-30
        tol = 1e-4 if ldt == torch.float32 else 5e-2
        assert (s.abs() / scale).max().item() < tol
    out2, t2 = ops.pyramid_forward(noisy, lg, dm, ksize=k)
    g2 = ops.pyramid_backward(t2, up)
    assert torch.equal(out, out2) and torch.equal(g.input, g2.input)
    assert all(torch.equal(a, b) for a, b in zip(g.logits, g2.logits))
    c = torch.full_like(noisy, 0.7)
    oc, _ = ops.pyramid_forward(c, lg, None, ksize=k)
    assert (oc - 0.7).abs().max().item() < 1e-5


def test_autograd_function(ops):
    rng = np.random.default_rng(5)
    h, w, L, k = 24, 30, 3, 5
    noisy, logits, dm, _, up, ref = oracle_case(h, w, L, k, seed=5)
    n = hwc_to_planar(noisy).requires_grad_()
    d = hwc_to_planar(dm).requires_grad_()
    lg = [hwc_to_planar(z).requires_grad_() for z in logits]
    out = ops.pyramid_filter(n, lg, d, ksize=k)
    (out * hwc_to_planar(up)).sum().backward()
    assert_close(planar_to_hwc(n.grad), ref["g_input"], 1e-10)
    assert_close(planar_to_hwc(d.grad), ref["g_demod"], 1e-10)
    for l in range(L):
        assert_close(planar_to_hwc(lg[l].grad), ref["g_logits"][l], 1e-10)
    del rng


def test_primitives_match_reference(ops):
    d = load("primitives")
    img = hwc_to_planar(d["gather_img"])
    wts = hwc_to_planar(d["gather_w"])
    np.testing.assert_allclose(planar_to_hwc(ops.gather(img, wts, 5)), d["gather_out"], rtol=1e-13)
    up = ops.upsample2(hwc_to_planar(d["up_coarse"]), hwc_to_planar(d["up_w"]))
    np.testing.assert_allclose(planar_to_hwc(up), d["up_out"], rtol=1e-13)
    lv = ops.build_pyramid(hwc_to_planar(d["pyr_in"]), 5)
    for l in range(5):
        np.testing.assert_allclose(planar_to_hwc(lv[l]), d[f"pyr_level{l}"], rtol=1e-13)
    z = hwc_to_planar(d["nk_logits0"])
    np.testing.assert_allclose(planar_to_hwc(ops.softmax_channels(z)), d["nk_wt0"], rtol=1e-13)
    np.testing.assert_allclose(planar_to_hwc(ops.softmax_channels(z, active=29)), d["nk_wf0"],
                               rtol=1e-13, atol=0)


TMA_CASES = [  # TMA-eligible shapes (fp32, W % 4 == 0 at every level) incl. edge sizes
    (8, 16, 2, 5, 3), (1, 32, 2, 5, 3), (3, 8, 2, 3, 3), (70, 64, 3, 5, 3), (130, 128, 4, 7, 3),
    (64, 96, 3, 5, 6), (37, 256, 3, 5, 3), (96, 64, 3, 3, 5),
]


@pytest.mark.parametrize("h,w,L,k,C", TMA_CASES)
@pytest.mark.parametrize("want", [True, False])
def test_tma_path_vs_oracle(ops, h, w, L, k, C, want):
    """The TMA-pipelined backward (fp32, demod) against the oracle, incl.
    image smaller than the kernel, single-row frames, two channel groups."""
    rng = np.random.default_rng(h * 7 + w + C)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    logits = [f32(z) for z in op.random_logits(h, w, L, k, rng, temporal=False)]
    noisy = f32(rng.lognormal(-1.0, 1.5, (h, w, C)))
    dm = f32(rng.uniform(0.0005, 1.0, (h, w, C)))
    up = f32(rng.normal(size=(h, w, C)))
    out_r, tape = op.forward(noisy, logits, None, dm, k=k)
    g_r = op.backward(tape, up, want_param_grads=want)
    out, t = ops.pyramid_forward(hwc_to_planar(noisy, torch.float32),
                                 [hwc_to_planar(z, torch.float32) for z in logits],
                                 hwc_to_planar(dm, torch.float32), ksize=k)
    g = ops.pyramid_backward(t, hwc_to_planar(up, torch.float32), want_param_grads=want)
    assert_close(planar_to_hwc(out), out_r, 1e-5)
    assert_close(planar_to_hwc(g.input), g_r.input, 1e-5)
    if want:
        assert_close(planar_to_hwc(g.demod), g_r.demod, 1e-5)
        assert_levels_close([planar_to_hwc(z) for z in g.logits], g_r.logits, 1e-5, scales=g_r.operand_scale)


def test_tma_and_generic_paths_agree(ops, monkeypatch):
    """SSB_NO_TMA=1 forces the generic strip walker: both backward kernels
    agree to fp32 rounding on a 1080p-shaped batch."""
    torch.manual_seed(3)
    H, W, L, k = 270, 480, 3, 5
    noisy = torch.rand(2, 3, H, W, device="cuda")
    dm = torch.rand(2, 3, H, W, device="cuda") * 0.9 + 0.05
    lg = [torch.randn(2, ops.logit_channels(l, L, k), h, w, device="cuda")
          for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    up = torch.randn(2, 3, H, W, device="cuda")
    _, t = ops.pyramid_forward(noisy, lg, dm, ksize=k)
    g1 = ops.pyramid_backward(t, up)
    monkeypatch.setenv("SSB_NO_TMA", "1")
    g2 = ops.pyramid_backward(t, up)
    for a_, b_ in [(g1.input, g2.input), (g1.demod, g2.demod)] + list(zip(g1.logits, g2.logits)):
        scale = b_.abs().max().item()
        assert (a_ - b_).abs().max().item() <= 2e-5 * scale


@pytest.mark.parametrize("H,W,L,k,ldt,hist", [(67, 132, 3, 5, "f32", False), (66, 136, 2, 5, "f32", False),
                                              (45, 96, 4, 7, "bf16", False), (33, 64, 5, 3, "f32", False),
                                              (67, 132, 3, 5, "f32", True), (45, 96, 4, 7, "bf16", True),
                                              (33, 64, 5, 3, "f32", True)])
def test_level0_last_order_matches_general_order(H, W, L, k, ldt, hist, monkeypatch):
    """The level-0-last backward (up-transpose pre-pass, pool chain, level 0
    writing final outputs; csrc/pyr_chain.cuh; with history: level 0 by the
    log-sum-exp weights plus the temporal pass) against the general order
    (fine -> coarse + the coarse -> fine sweep kernel) on the same inputs."""
    from paper_2602_08642_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(H * W + L)
    dev = torch.device("cuda")
    noisy = torch.rand((2, 3, H, W), device=dev, generator=g) * 2
    demod = torch.rand((2, 3, H, W), device=dev, generator=g) * 0.99 + 0.0005
    prev = torch.rand((2, 3, H, W), device=dev, generator=g) * 2 if hist else None
    shapes = ops.level_shapes(H, W, L)
    logits = [torch.randn((2, ops.logit_channels(l, L, k, has_prev=hist and l == 0), h, w), device=dev, generator=g)
              for l, (h, w) in enumerate(shapes)]
    if ldt == "bf16":
        logits = [z.to(torch.bfloat16) for z in logits]
    up = torch.randn((2, 3, H, W), device=dev, generator=g)
    res = {}
    for mode in ("chain", "general"):
        if mode == "general":
            monkeypatch.setenv("SSB_NO_CHAIN", "1")
        out, tape = ops.pyramid_forward(noisy, logits, demod, prev, ksize=k)
        gr = ops.pyramid_backward(tape, up)
        res[mode] = (out, gr)
        monkeypatch.delenv("SSB_NO_CHAIN", raising=False)
    (o1, g1), (o2, g2) = res["chain"], res["general"]
    assert torch.equal(o1, o2)
    pairs = [(g1.input, g2.input), (g1.demod, g2.demod)] + list(zip(g1.logits, g2.logits))
    if hist:
        pairs.append((g1.prev, g2.prev))
    for a, b in pairs:
        a, b = a.double(), b.double()
        tol = 2e-2 if ldt == "bf16" else 1e-5
        assert torch.allclose(a, b, rtol=tol, atol=tol * b.abs().max().item()), (a - b).abs().max().item()


@pytest.mark.parametrize("k,ldt,blend,C", [(7, torch.bfloat16, "native", 3), (7, torch.bfloat16, "tied", 6),
                                           (7, torch.bfloat16, "native", 4), (5, torch.float32, "tied", 6),
                                           (5, torch.float32, "native", 4), (3, torch.float32, "native", 3)])
def test_tma_and_generic_forward_backward_agree(ops, monkeypatch, k, ldt, blend, C):
    """The TMA level kernels (incl. the bf16 k = 7 pixel-pair forward and the
    level-0-last backward) against the generic kernels (SSB_NO_TMA=1) on the
    same inputs: forward outputs and every gradient to fp32 rounding; tied
    blend and C = 6 (two channel groups) included."""
    g = torch.Generator(device="cuda").manual_seed(k * 10 + C)
    H, W, L = 72, 128, 4
    noisy = torch.rand((2, C, H, W), device="cuda", generator=g) * 2
    dm = torch.rand((2, C, H, W), device="cuda", generator=g) * 0.9 + 0.05
    lg = [torch.randn((2, ops.logit_channels(l, L, k, blend=blend), h, w), device="cuda", generator=g).to(ldt)
          for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    up = torch.randn((2, C, H, W), device="cuda", generator=g)
    res = []
    for mode in ("tma", "generic"):
        if mode == "generic":
            monkeypatch.setenv("SSB_NO_TMA", "1")
        out, t = ops.pyramid_forward(noisy, lg, dm, ksize=k, blend=blend)
        res.append((out, ops.pyramid_backward(t, up)))
        monkeypatch.delenv("SSB_NO_TMA", raising=False)
    (o1, g1), (o2, g2) = res
    assert (o1 - o2).abs().max().item() <= 2e-5 * o2.abs().max().item()
    tol = 2e-2 if ldt == torch.bfloat16 else 2e-5  # bf16 logit gradients round differently
    for a_, b_ in [(g1.input, g2.input), (g1.demod, g2.demod)]:
        assert (a_ - b_).abs().max().item() <= 2e-5 * b_.abs().max().item()
    for a_, b_ in zip(g1.logits, g2.logits):
        a_, b_ = a_.float(), b_.float()
        assert (a_ - b_).abs().max().item() <= tol * b_.abs().max().item()



@pytest.mark.parametrize("H,W", [(67, 132), (130, 256)])
def test_s8_level0_backward_matches_s4(ops, monkeypatch, H, W):
    """SSB_BWD_S8=1 (the 8-row-step, 512-thread level-0 backward, k5 fp32)
    against the default 4-row-step kernel on the same tape: every gradient
    to fp32 rounding."""
    g = torch.Generator(device="cuda").manual_seed(H + W)
    L, k = 3, 5
    noisy = torch.rand((2, 3, H, W), device="cuda", generator=g) * 2
    dm = torch.rand((2, 3, H, W), device="cuda", generator=g) * 0.9 + 0.05
    lg = [torch.randn((2, ops.logit_channels(l, L, k), h, w), device="cuda", generator=g)
          for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    up = torch.randn((2, 3, H, W), device="cuda", generator=g)
    _, t = ops.pyramid_forward(noisy, lg, dm, ksize=k)
    g4 = ops.pyramid_backward(t, up)
    monkeypatch.setenv("SSB_BWD_S8", "1")
    g8 = ops.pyramid_backward(t, up)
    monkeypatch.delenv("SSB_BWD_S8")
    for a_, b_ in [(g8.input, g4.input), (g8.demod, g4.demod)] + list(zip(g8.logits, g4.logits)):
        assert (a_ - b_).abs().max().item() <= 1e-5 * b_.abs().max().item()


@pytest.mark.parametrize("h,w,L,k,ldt", [(96, 128, 3, 5, torch.float32), (72, 128, 4, 7, torch.bfloat16),
                                         (45, 70, 3, 5, torch.float32)])
def test_no_demod_identity_path(ops, monkeypatch, h, w, L, k, ldt):
    """demod=None (reconstruct_core's default) runs the fused demodulating
    kernels with an identity demod: against the oracle without demod, and
    against the generic no-demod kernels (SSB_NO_IDENTITY_DEMOD=1)."""
    rng = np.random.default_rng(h + w)
    logits32 = op.random_logits(h, w, L, k, rng, temporal=False)
    lg = [hwc_to_planar(z, torch.float32).to(ldt) for z in logits32]
    logits = [planar_to_hwc(z) for z in lg]  # the device values (bf16-rounded)
    noisy = rng.lognormal(-1.0, 1.5, (h, w, 3)).astype(np.float32).astype(np.float64)
    up = rng.normal(size=(h, w, 3)).astype(np.float32).astype(np.float64)
    out_r, tape = op.forward(noisy, logits, None, None, k=k)
    g_r = op.backward(tape, up)
    rtol = 1e-5 if ldt == torch.float32 else 2e-2
    res = []
    for generic in (False, True):
        if generic:
            monkeypatch.setenv("SSB_NO_IDENTITY_DEMOD", "1")
        out, t = ops.pyramid_forward(hwc_to_planar(noisy, torch.float32), lg, None, ksize=k)
        g = ops.pyramid_backward(t, hwc_to_planar(up, torch.float32))
        monkeypatch.delenv("SSB_NO_IDENTITY_DEMOD", raising=False)
        assert g.demod is None
        assert_close(planar_to_hwc(out), out_r, rtol, "out")
        assert_close(planar_to_hwc(g.input), g_r.input, rtol, "g_input")
        assert_levels_close([planar_to_hwc(z) for z in g.logits], g_r.logits, rtol, scales=g_r.operand_scale)
        res.append((out, g))
    (o1, g1), (o2, g2) = res
    assert (o1 - o2).abs().max().item() <= 2e-5 * o2.abs().max().item()


@pytest.mark.parametrize("k,ldt", [(5, "f32"), (7, "bf16")])
def test_history_without_param_grads_matches_general_order(k, ldt, monkeypatch):
    """History on the TMA path without parameter gradients (no g_demod, no
    logit gradients: the temporal pass without its g_demod box) against the
    general order -- g_noisy and g_prev."""
    from paper_2602_08642_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(31 + k)
    dev = torch.device("cuda")
    H, W, L = 52, 96, 3
    noisy = torch.rand((2, 3, H, W), device=dev, generator=g) * 2
    demod = torch.rand((2, 3, H, W), device=dev, generator=g) * 0.99 + 0.0005
    prev = torch.rand((2, 3, H, W), device=dev, generator=g) * 2
    logits = [torch.randn((2, ops.logit_channels(l, L, k, has_prev=l == 0), h, w), device=dev, generator=g)
              for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    if ldt == "bf16":
        logits = [z.to(torch.bfloat16) for z in logits]
    up = torch.randn((2, 3, H, W), device=dev, generator=g)
    res = {}
    for mode in ("chain", "general"):
        if mode == "general":
            monkeypatch.setenv("SSB_NO_CHAIN", "1")
        _, tape = ops.pyramid_forward(noisy, logits, demod, prev, ksize=k)
        res[mode] = ops.pyramid_backward(tape, up, want_param_grads=False)
        monkeypatch.delenv("SSB_NO_CHAIN", raising=False)
    a, b = res["chain"], res["general"]
    assert a.demod is None and a.logits is None
    tol = 2e-2 if ldt == "bf16" else 1e-5
    for x, y in ((a.input, b.input), (a.prev, b.prev)):
        x, y = x.double(), y.double()
        assert torch.allclose(x, y, rtol=tol, atol=tol * y.abs().max().item()), (x - y).abs().max().item()


def test_history_accumulate_into_tma_path():
    """accumulate_into with history on the TMA path (the temporal pass adds
    into the temporal channels, level 0 into the others): two accumulated
    backward passes equal twice one pass."""
    from paper_2602_08642_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(77)
    dev = torch.device("cuda")
    H, W, L, k = 40, 64, 3, 5
    noisy = torch.rand((1, 3, H, W), device=dev, generator=g) * 2
    demod = torch.rand((1, 3, H, W), device=dev, generator=g) * 0.99 + 0.01
    prev = torch.rand((1, 3, H, W), device=dev, generator=g) * 2
    logits = [torch.randn((1, ops.logit_channels(l, L, k, has_prev=l == 0), h, w), device=dev, generator=g)
              for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    up = torch.randn((1, 3, H, W), device=dev, generator=g)
    _, tape = ops.pyramid_forward(noisy, logits, demod, prev, ksize=k)
    one = ops.pyramid_backward(tape, up)
    acc = [torch.zeros_like(z) for z in logits]
    ops.pyramid_backward(tape, up, accumulate_into=acc)
    ops.pyramid_backward(tape, up, accumulate_into=acc)
    for a, b in zip(acc, one.logits):
        assert torch.allclose(a, 2 * b, rtol=1e-6, atol=1e-6 * b.abs().max().item())


@pytest.mark.parametrize("h,w,L,k", [(48, 64, 3, 5), (37, 56, 4, 7), (30, 40, 3, 3)])
def test_history_without_demod_vs_oracle(ops, h, w, L, k):
    """reconstruct_core with a history and demod=None (the identity
    demodulation on the fused kernels: level 0 by the log-sum-exp weights +
    the temporal pass) against the float64 oracle, float32, every level."""
    noisy, logits, dm, pv, up, ref = oracle_case(h, w, L, k, seed=h + w + k, demod=False, prev=True)
    assert dm is None
    dt = torch.float32
    out, tape = ops.pyramid_forward(hwc_to_planar(noisy, dt), [hwc_to_planar(z, dt) for z in logits], None,
                                    hwc_to_planar(pv, dt), ksize=k)
    g = ops.pyramid_backward(tape, hwc_to_planar(up, dt))
    assert g.demod is None
    assert_close(planar_to_hwc(out), ref["out"], 1e-5, "out")
    assert_close(planar_to_hwc(g.input), ref["g_input"], 1e-5, "g_input")
    assert_close(planar_to_hwc(g.prev), ref["g_prev"], 1e-5, "g_prev")
    assert_levels_close([planar_to_hwc(z) for z in g.logits], ref["g_logits"], 1e-5, scales=ref["scales"])


@pytest.mark.parametrize("h,w,L,k,prev", [(40, 64, 3, 7, False), (48, 64, 3, 5, True), (36, 56, 4, 7, True)])
def test_peaky_logits_log_sum_exp_path(ops, h, w, L, k, prev):
    """Large-magnitude logits (scale 8: near one-hot softmaxes, exponents far
    below the max) on the paths that evaluate the weights from the forward's
    log-sum-exp (k = 7, history): float32 within 1e-5 of the oracle."""
    noisy, logits, dm, pv, up, ref = oracle_case(h, w, L, k, seed=7 * h + w, prev=prev, scale=8.0)
    dt = torch.float32
    out, tape = ops.pyramid_forward(hwc_to_planar(noisy, dt), [hwc_to_planar(z, dt) for z in logits],
                                    hwc_to_planar(dm, dt), hwc_to_planar(pv, dt) if prev else None, ksize=k)
    g = ops.pyramid_backward(tape, hwc_to_planar(up, dt))
    assert_close(planar_to_hwc(out), ref["out"], 1e-5, "out")
    assert_close(planar_to_hwc(g.input), ref["g_input"], 1e-5, "g_input")
    assert_close(planar_to_hwc(g.demod), ref["g_demod"], 1e-5, "g_demod")
    if prev:
        assert_close(planar_to_hwc(g.prev), ref["g_prev"], 1e-5, "g_prev")
    assert_levels_close([planar_to_hwc(z) for z in g.logits], ref["g_logits"], 1e-5, scales=ref["scales"])
