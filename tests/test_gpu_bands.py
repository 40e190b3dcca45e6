"""Row bands on the GPU: the band protocol of
paper_2602_08642_b200/bands.py (halo rows of each pooled level + one Lhat row
per level; no logits exchanged) with the library's level kernels
(ssb_pyr_forward_level, ssb_pool2_strided): the stitched band outputs equal
the single-GPU full-frame ssb_pyr_forward bit for bit.  Bands are emulated in
one process (LocalTransport, lockstep); the distributed exchange protocol is
covered on CPU (tests/test_bands_dist.py), and the peer-memory transport's
kernels (P2P-store copy + generation flag, stream wait) here on one device."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08642_b200 import ops as _ops
    return _ops


@pytest.mark.parametrize("H,W,L,k,G,ldt", [
    (720, 300, 3, 5, 3, torch.float32),
    (1100, 256, 4, 7, 4, torch.float32),
    (1088, 200, 4, 7, 3, torch.bfloat16),
    (4320, 512, 4, 7, 8, torch.float32),   # 8K height, narrow strip
    (333, 96, 3, 3, 2, torch.float32),     # odd frame height (last band odd at every level)
    (200, 64, 3, 5, 2, torch.float64),
])
def test_bands_bitwise_equal_full_frame(ops, H, W, L, k, G, ldt):
    from paper_2602_08642_b200 import bands
    torch.manual_seed(H + W)
    idt = torch.float64 if ldt == torch.float64 else torch.float32
    noisy = (torch.rand(1, 3, H, W, device="cuda") * 2).to(idt)
    demod = (torch.rand(1, 3, H, W, device="cuda") * 0.9 + 0.05).to(idt)
    logits = [torch.randn(1, ops.logit_channels(l, L, k), h, w, device="cuda").to(ldt)
              for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    full, _ = ops.pyramid_forward(noisy, logits, demod, ksize=k)
    banded = bands.forward_emulated(noisy, logits, demod, ksize=k, bands=G)
    assert torch.equal(full, banded)


def test_forward_level_matches_pyramid_forward(ops):
    """Level by level through ssb_pyr_forward_level (+ strided pooling) on
    plain full-frame buffers == ssb_pyr_forward."""
    H, W, L, k = 130, 96, 3, 5
    g = torch.Generator(device="cuda").manual_seed(1)
    noisy = torch.rand(2, 3, H, W, device="cuda", generator=g)
    demod = torch.rand(2, 3, H, W, device="cuda", generator=g) * 0.9 + 0.05
    shapes = ops.level_shapes(H, W, L)
    logits = [torch.randn(2, ops.logit_channels(l, L, k), h, w, device="cuda", generator=g)
              for l, (h, w) in enumerate(shapes)]
    full, _ = ops.pyramid_forward(noisy, logits, demod, ksize=k)
    lv = [None] * L
    for l in range(1, L):
        lv[l] = torch.empty(2, 3, *shapes[l], device="cuda")
        ops.pool2_into(noisy if l == 1 else lv[l - 1], lv[l], demod if l == 1 else None)
    lhat = [None] * L
    for l in range(L - 1, -1, -1):
        img = noisy if l == 0 else lv[l]
        lhat[l] = ops.pyramid_forward_level(img, logits[l], ksize=k, demod=demod if l == 0 else None,
                                            coarse=lhat[l + 1] if l < L - 1 else None)
    assert torch.equal(lhat[0], full)


def test_halo_put_and_flag_wait(ops):
    """The peer transport's kernels on one device (no cross-rank waiting):
    the row-block copy lands exactly, the generation flag is published after
    it, and a wait on an already-published generation passes."""
    src = torch.randn(2, 3, 40, 64, device="cuda")
    dst = torch.zeros(2, 3, 50, 64, device="cuda")
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    ops.halo_put(dst[:, :, 10:14], src[:, :, 3:7], flags[1], 5)
    ops.flag_wait(flags[1], 5)
    ops.flag_release(flags[2], 7, torch.device("cuda"))
    ops.flag_wait(flags[2], 7)
    torch.cuda.synchronize()
    assert torch.equal(dst[:, :, 10:14], src[:, :, 3:7])
    assert dst[:, :, :10].abs().sum().item() == 0 and dst[:, :, 14:].abs().sum().item() == 0
    assert flags.tolist() == [0, 5, 7, 0]
