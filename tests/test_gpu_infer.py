"""The small-frame inference path (``ops.infer`` -> ``ssb_infer_small``: the
stochastic fused placement + reconstruct_core in one cooperative kernel,
BASELINE c0) against the two-call path it replaces (``place_fused`` +
``pyramid_forward``) and the float64 oracle.

* noisy: bit-identical to ``place_fused`` (same partial pairs, fold and
  per-pixel placement);
* out: within float32 rounding of ``pyramid_forward`` on that noisy (rtol
  1e-5 with the per-tensor floor of SURVEY.md 8(c)) and of the oracle's
  forward (pyramid.py:292-345);
* frames beyond the small-frame limit take the two-call path (bitwise equal).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import pyramid as op  # noqa: E402
from tests._conv import assert_close  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08642_b200 import ops as o
    return o


def _inputs(ops, B, H, W, L, k, seed):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    scores = torch.randn(B, H, W, generator=g, device=dev)
    bank = torch.exp(-1.0 + 1.5 * torch.randn(B, 2, 3, H, W, generator=g, device=dev))
    demod = torch.rand(B, 3, H, W, generator=g, device=dev) * 0.95 + 0.0005
    logits = [torch.randn(B, ops.logit_channels(l, L, k), h, w, generator=g, device=dev)
              for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    return scores, bank, demod, logits


@pytest.mark.parametrize("B,H,W,L,k", [(1, 256, 256, 3, 5), (3, 64, 96, 4, 3), (2, 45, 80, 2, 7),
                                       (1, 33, 52, 5, 5), (8, 128, 128, 3, 5)])
def test_infer_small_matches_two_call_path(ops, B, H, W, L, k):
    from paper_2602_08642_b200 import _lib
    scores, bank, demod, logits = _inputs(ops, B, H, W, L, k, seed=H * W + L)
    lib = _lib.load()
    n0 = lib.ssb_launch_count()
    out, noisy = ops.infer(scores, bank, demod, logits, 0.4, ksize=k, seed=9, frame0=2)
    torch.cuda.synchronize()
    assert lib.ssb_launch_count() - n0 == 1, "the small-frame path is one launch"
    ref_noisy, _, _ = ops.place_fused(scores, bank, 0.4, seed=9, frame0=2)
    assert torch.equal(noisy, ref_noisy)
    ref_out, _ = ops.pyramid_forward(ref_noisy, logits, demod, ksize=k)
    for b in range(B):
        assert_close(out[b].double().cpu().numpy(), ref_out[b].double().cpu().numpy(), 1e-5, f"out[{b}]")


def test_infer_small_vs_oracle(ops):
    B, H, W, L, k = 1, 72, 96, 3, 5
    scores, bank, demod, logits = _inputs(ops, B, H, W, L, k, seed=5)
    out, noisy = ops.infer(scores, bank, demod, logits, 0.25, ksize=k, seed=1)
    host = lambda t: t[0].permute(1, 2, 0).double().cpu().numpy()  # noqa: E731
    ref, _ = op.forward(host(noisy), [host(z) for z in logits], None, host(demod), k=k)
    assert_close(host(out), ref, 1e-5, "out")
    assert np.count_nonzero(host(noisy)) > 0


def test_infer_large_frame_takes_two_call_path(ops):
    B, H, W, L, k = 1, 1080, 1000, 3, 5  # > 2^20 pixels
    scores, bank, demod, logits = _inputs(ops, B, H, W, L, k, seed=3)
    out, noisy = ops.infer(scores, bank, demod, logits, 0.25, ksize=k, seed=4)
    ref_noisy, _, _ = ops.place_fused(scores, bank, 0.25, seed=4)
    ref_out, _ = ops.pyramid_forward(ref_noisy, logits, demod, ksize=k)
    assert torch.equal(noisy, ref_noisy) and torch.equal(out, ref_out)
