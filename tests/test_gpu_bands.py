"""Row bands: stitched band outputs equal the single-GPU
full-frame forward bit for bit (bands emulated on one GPU; the distributed
exchange itself is covered on CPU by tests/test_bands_dist.py)."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("H,W,L,k,G,ldt", [
    (720, 300, 3, 5, 3, torch.float32),
    (1100, 256, 4, 7, 4, torch.float32),
    (1088, 200, 4, 7, 3, torch.bfloat16),
    (4320, 512, 4, 7, 8, torch.float32),   # 8K height, narrow strip
])
def test_bands_bitwise_equal_full_frame(H, W, L, k, G, ldt):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08642_b200 import bands, ops
    torch.manual_seed(H + W)
    noisy = torch.rand(1, 3, H, W, device="cuda") * 2
    demod = torch.rand(1, 3, H, W, device="cuda") * 0.9 + 0.05
    logits = [torch.randn(1, ops.logit_channels(l, L, k), h, w, device="cuda").to(ldt)
              for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    full, _ = ops.pyramid_forward(noisy, logits, demod, ksize=k)
    banded = bands.forward_emulated(noisy, logits, demod, ksize=k, bands=G)
    assert torch.equal(full, banded)
