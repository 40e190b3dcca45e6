"""Pin the CPU oracle against fixtures produced by the unmodified reference.

The oracle restates the reference with k and L as parameters; at k = 5 it
must reproduce the reference bit-for-bit (float64).  No GPU needed.
"""
import numpy as np
import pytest

from oracle import density as od
from oracle import estimators as oe
from oracle import pyramid as op
from oracle import rng as orng
from tests._golden import case_logits, load, pyramid_cases


@pytest.mark.parametrize("name", pyramid_cases())
def test_pyramid_forward_backward_bit_exact(name):
    d = load(name)
    out, tape = op.forward(d["noisy"], case_logits(d), d.get("prev"), d.get("demod"))
    np.testing.assert_array_equal(out, d["out"])
    g = op.backward(tape, d["upstream"], want_param_grads=bool(d["want"]))
    np.testing.assert_array_equal(g.input, d["g_input"])
    if bool(d["want"]):
        for l in range(int(d["levels"])):
            np.testing.assert_array_equal(g.logits[l], d[f"g_logits{l}"])
        if "g_demod" in d:
            np.testing.assert_array_equal(g.demod, d["g_demod"])
    if "g_prev" in d:
        np.testing.assert_array_equal(g.prev, d["g_prev"])


def test_primitives_bit_exact():
    d = load("primitives")
    np.testing.assert_array_equal(op.gather(d["gather_img"], d["gather_w"], 5), d["gather_out"])
    np.testing.assert_array_equal(op.upsample(d["up_coarse"], d["up_w"]), d["up_out"])
    lv, _ = op.pyramid_levels(d["pyr_in"], 5)
    for l in range(5):
        np.testing.assert_array_equal(lv[l], d[f"pyr_level{l}"])
    logits = [d[f"nk_logits{l}"] for l in range(5)]
    for temporal, key in ((True, "nk_wt"), (False, "nk_wf")):
        ws = op.kernel_weights(logits, 5, temporal)
        for l in range(5):
            np.testing.assert_array_equal(ws[l], d[f"{key}{l}"])


def test_rng_bit_exact():
    d = load("placement")
    for i in range(5):
        s, f, st = (int(v) for v in d[f"ug{i}_key"])
        np.testing.assert_array_equal(orng.uniform_grid(s, f, 23, 17, st), d[f"ug{i}"])
    np.testing.assert_array_equal(orng.uniform_grid_batch(2, d["ugb_frames"], 19, 11, 3), d["ugb"])


def test_density_and_allocation_bit_exact():
    d = load("placement")
    for i in range(3):
        np.testing.assert_array_equal(od.normalize_density(d[f"nd{i}_scores"], float(d[f"nd{i}_budget"])),
                                      d[f"nd{i}_spp"])
    for rule in ("stochastic", "relaxed", "gumbel"):
        base, frac, u, taken = od.allocate(d["al_spp"], "stochastic", frame=11, seed=5, rule=rule,
                                           gumbel_temp=0.7)
        np.testing.assert_array_equal(base, d[f"al_{rule}_base"])
        np.testing.assert_array_equal(frac, d[f"al_{rule}_frac"])
        np.testing.assert_array_equal(u, d[f"al_{rule}_u"])
        np.testing.assert_array_equal(taken, d[f"al_{rule}_taken"])
    _, _, u, taken = od.allocate(d["al_spp"], "dithered", rank=d["dm_rank"], frame=5)
    np.testing.assert_array_equal(u, d["dm_u"])
    np.testing.assert_array_equal(taken, d["dm_taken"])


@pytest.mark.parametrize("variant", ["stochastic", "relaxed", "straight-through", "gumbel"])
def test_estimators_bit_exact(variant):
    d = load("placement")
    key = variant.replace("-", "_")
    spp = d["es_spp"]
    base = np.floor(spp).astype(np.int64)
    frac = spp - base
    noisy, grad, contrib, used = oe.estimate(variant, spp, base, frac, d[f"es_{key}_u"],
                                             d["es_samples"], lam=7.0, gumbel_temp=0.8)
    np.testing.assert_array_equal(noisy, d[f"es_{key}_noisy"])
    np.testing.assert_array_equal(grad, d[f"es_{key}_grad"])
    np.testing.assert_array_equal(contrib, d[f"es_{key}_contrib"])
    np.testing.assert_array_equal(used, d[f"es_{key}_used"])


def test_tied_blend_equals_broadcast_native():
    rng = np.random.default_rng(3)
    tied = op.random_logits(9, 11, 3, 5, rng, temporal=False, blend="tied")
    native = op.expand_blend(tied, 5)
    noisy = rng.uniform(0.1, 2, (9, 11, 3))
    up = rng.normal(size=(9, 11, 3))
    o1, t1 = op.forward(noisy, tied, k=5, blend="tied")
    o2, t2 = op.forward(noisy, native, k=5)
    np.testing.assert_array_equal(o1, o2)
    g1 = op.backward(t1, up)
    g2 = op.backward(t2, up)
    for a, b in zip(g1.logits, op.collapse_blend_grads(g2.logits, 5)):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("k", [3, 7])
def test_radius_generalised_gradcheck(k):
    """The k != 5 restatement has no reference counterpart: check it by
    central differences on every parameter group."""
    rng = np.random.default_rng(10 + k)
    h, w, L = 9, 8, 3
    logits = op.random_logits(h, w, L, k, rng, temporal=True)
    noisy = rng.uniform(0.05, 2.0, (h, w, 3))
    prev = rng.uniform(0.05, 2.0, (h, w, 3))
    demod = rng.uniform(0.2, 2.0, (h, w, 3))
    up = rng.normal(size=(h, w, 3))
    out, tape = op.forward(noisy, logits, prev, demod, k=k)
    g = op.backward(tape, up)

    def loss():
        return float((up * op.forward(noisy, logits, prev, demod, k=k)[0]).sum())

    eps = 1e-6
    checks = [(logits[l], g.logits[l]) for l in range(L)] + [(noisy, g.input), (demod, g.demod),
                                                            (prev, g.prev)]
    for arr, grad in checks:
        for _ in range(6):
            idx = tuple(int(rng.integers(0, s)) for s in arr.shape)
            old = arr[idx]
            arr[idx] = old + eps
            lp = loss()
            arr[idx] = old - eps
            lm = loss()
            arr[idx] = old
            fd = (lp - lm) / (2 * eps)
            assert abs(grad[idx] - fd) <= 1e-5 * max(1.0, abs(fd))


def test_temporal_warp_bit_exact():
    """oracle/temporal.py vs images.warp_array / warp_backward (8(f) row 2)."""
    from oracle import temporal as ot
    d = load("temporal")
    for n in d["names"]:
        out, val = ot.warp_array(d[f"{n}_prev"], d[f"{n}_motion"])
        np.testing.assert_array_equal(out, d[f"{n}_out"])
        np.testing.assert_array_equal(val, d[f"{n}_validity"])
        np.testing.assert_array_equal(ot.warp_backward(d[f"{n}_gout"], d[f"{n}_motion"]), d[f"{n}_gprev"])


def test_temporal_warp_adjoint():
    from oracle import temporal as ot
    rng = np.random.default_rng(5)
    x = rng.normal(size=(9, 11, 3))
    g = rng.normal(size=(9, 11, 3))
    m = rng.uniform(-4, 4, (9, 11, 2))
    lhs = (ot.warp_array(x, m)[0] * g).sum()
    rhs = (x * ot.warp_backward(g, m)).sum()
    assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs))


def test_score_grad_bit_exact():
    """oracle/scores.py vs the reference's softmax_backward chain with scipy's
    gaussian_filter (optimize.py:244-251; 8(f) row 3)."""
    from oracle import scores as osc
    d = load("scores")
    for n in d["names"]:
        r = osc.score_grad(d[f"{n}_scores"], float(d[f"{n}_budget"]), list(d[f"{n}_gin"]),
                           list(d[f"{n}_gd"]), float(d[f"{n}_sigma"]))
        np.testing.assert_array_equal(r, d[f"{n}_gscores"])


def test_tonemap_and_losses_bit_exact():
    """oracle/tonemap.py vs tonemap.py / losses.py and the loss gradient of
    optimize.py:219-231 (8(f) row 4)."""
    from oracle import tonemap as otm
    d = load("tonemap")
    for i in range(3):
        t = tuple(d[f"tmo{i}"])
        np.testing.assert_array_equal(otm.tonemap(d["rad"], t), d[f"tm_ldr{i}"])
        np.testing.assert_array_equal(otm.tonemap_backward(d["rad"], t, d["up"]), d[f"gtm{i}"])
    sp, tm, cb, vals = otm.losses(d["ldr1"], d["ref"], d["ldr0w"], d["refw"], d["validity"], d["mask"])
    np.testing.assert_array_equal(sp, d["sp_map"])
    np.testing.assert_array_equal(tm, d["tm_map"])
    np.testing.assert_array_equal(cb, d["cb_map"])
    np.testing.assert_array_equal(np.array(vals), d["losses"])
    g1, g0 = otm.loss_grads(d["ldr1"], d["ref"], d["ldr0w"], d["refw"], d["validity"], d["mask"])
    np.testing.assert_array_equal(g1, d["g_ldr1"])
    np.testing.assert_array_equal(g0, d["g_ldr0w"])
