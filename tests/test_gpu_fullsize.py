"""Oracle parity at the BASELINE sizes themselves.

The CUDA filter (through the C ABI, `ops`) against the float64 oracle
restatement of the reference (pinned bit-for-bit to the reference's golden
outputs in tests/test_oracle_golden.py) on FULL frames with the BASELINE
input distributions (bench.synthetic_inputs: GRF density, 0.25 spp fused
placement over a log-normal bank with 1% x100 fireflies, albedo demod, N(0,1)
logits and upstream):

* c0: one 256x256 frame, L3 k5, fp32;
* c1 / c4a: one 1920x1080 frame, L3 k5, fp32 (c4a is 64 of these);
* c3: one 3840x2160 frame, L4 k7, bf16 logits (the oracle gets the
  bf16-rounded logits, upcast exactly), fp32 radiance and accumulation.

Comparator (tests/_conv.py): per tensor and, for the logit
gradients, per LEVEL -- elementwise rtol with an atol floor of
rtol * max|ref_l| of that tensor, plus relative-L2 <= rtol; rtol = 1e-5
(fp32) / 2e-2 (bf16 logits), the north-star tolerances.  The c3 oracle run
takes ~2 min and ~22 GB of host memory.
"""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import pyramid as op  # noqa: E402
from tests._conv import assert_close, assert_levels_close  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _host(t):
    return t[0].permute(1, 2, 0).double().cpu().numpy()


@pytest.mark.parametrize("name,H,W,L,k,ldt,rtol", [
    ("c0", 256, 256, 3, 5, "f32", 1e-5),
    ("c1", 1080, 1920, 3, 5, "f32", 1e-5),
    ("c3", 2160, 3840, 4, 7, "bf16", 2e-2),
])
def test_full_frame_vs_oracle(name, H, W, L, k, ldt, rtol):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    import bench
    from paper_2602_08642_b200 import ops
    dev = torch.device("cuda:0")
    noisy, demod, logits, up = bench.synthetic_inputs(1, H, W, L, k, ldt, dev, seed=17 + L * k)
    out, tape = ops.pyramid_forward(noisy, logits, demod, ksize=k)
    g = ops.pyramid_backward(tape, up)
    torch.cuda.synchronize()
    if ldt == "bf16":
        assert g.logits[0].dtype == torch.bfloat16
    gpu = {"out": _host(out), "g_input": _host(g.input), "g_demod": _host(g.demod),
           "g_logits": [_host(z) for z in g.logits]}
    ins = {"noisy": _host(noisy), "demod": _host(demod), "up": _host(up),
           "logits": [_host(z) for z in logits]}  # exact upcasts of the device values
    del out, tape, g, noisy, demod, logits, up
    torch.cuda.empty_cache()
    assert np.count_nonzero(ins["noisy"]) > 0
    ref_out, ref_tape = op.forward(ins["noisy"], ins["logits"], None, ins["demod"], k=k)
    ref_g = op.backward(ref_tape, ins["up"])
    del ref_tape
    assert_close(gpu["out"], ref_out, rtol, f"{name} out")
    assert_close(gpu["g_input"], ref_g.input, rtol, f"{name} g_noisy")
    assert_close(gpu["g_demod"], ref_g.demod, rtol, f"{name} g_demod")
    assert_levels_close(gpu["g_logits"], ref_g.logits, rtol, f"{name} g_logits", scales=ref_g.operand_scale)
    for l, (z, s) in enumerate(zip(ref_g.logits, ref_g.operand_scale)):
        print(f"{name} level {l}: max|ref| {np.abs(z).max():.3e}, operand scale {s:.3e}")


def test_full_frame_history_vs_oracle():
    """evaluate_step's frame-1 call shape at a full 1080p frame: L3 k5 fp32
    with the 25-tap temporal group over a warped history (the TMA path:
    log-sum-exp level-0 weights + the temporal pass), against the float64
    oracle -- every tensor and level within 1e-5."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    import bench
    from paper_2602_08642_b200 import ops
    dev = torch.device("cuda:0")
    H, W, L, k = 1080, 1920, 3, 5
    noisy, demod, logits, up = bench.synthetic_inputs(1, H, W, L, k, "f32", dev, seed=29)
    g = torch.Generator(device=dev).manual_seed(30)
    prev = torch.exp(-1.0 + 1.0 * torch.randn(1, 3, H, W, generator=g, device=dev))
    logits[0] = torch.cat([logits[0], torch.randn(1, k * k, H, W, generator=g, device=dev)], dim=1).contiguous()
    out, tape = ops.pyramid_forward(noisy, logits, demod, prev, ksize=k)
    gr = ops.pyramid_backward(tape, up)
    torch.cuda.synchronize()
    gpu = {"out": _host(out), "g_input": _host(gr.input), "g_demod": _host(gr.demod), "g_prev": _host(gr.prev),
           "g_logits": [_host(z) for z in gr.logits]}
    ins = {"noisy": _host(noisy), "demod": _host(demod), "up": _host(up), "prev": _host(prev),
           "logits": [_host(z) for z in logits]}
    del out, tape, gr, noisy, demod, logits, up, prev
    torch.cuda.empty_cache()
    ref_out, ref_tape = op.forward(ins["noisy"], ins["logits"], ins["prev"], ins["demod"], k=k)
    ref_g = op.backward(ref_tape, ins["up"])
    del ref_tape
    assert_close(gpu["out"], ref_out, 1e-5, "c1h out")
    assert_close(gpu["g_input"], ref_g.input, 1e-5, "c1h g_noisy")
    assert_close(gpu["g_demod"], ref_g.demod, 1e-5, "c1h g_demod")
    assert_close(gpu["g_prev"], ref_g.prev, 1e-5, "c1h g_prev")
    assert_levels_close(gpu["g_logits"], ref_g.logits, 1e-5, "c1h g_logits", scales=ref_g.operand_scale)
