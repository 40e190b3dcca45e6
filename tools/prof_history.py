"""One fwd+bwd of the history call shape (evaluate_step frame 1: the 25-tap
temporal group over a warped history), 4 x 1080p L3 k5 fp32, for an ncu
launch list (per-kernel times of the shape)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_08642_b200 import ops  # noqa: E402


def main():
    frames, H, W, L, k = int(os.environ.get("FRAMES", 4)), 1080, 1920, 3, 5
    C = int(os.environ.get("CH", 3))
    hist = os.environ.get("HIST", "1") == "1"
    want = os.environ.get("WANT", "1") == "1"
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(11)
    shapes = bench.level_shapes(H, W, L)
    noisy = torch.rand(frames, C, H, W, generator=g, device=dev)
    demod = torch.rand(frames, C, H, W, generator=g, device=dev) * 0.95 + 0.05
    prev = torch.rand(frames, C, H, W, generator=g, device=dev) if hist else None
    logits = [torch.randn(frames, ops.logit_channels(l, L, k, has_prev=hist and l == 0), h, w, generator=g,
                          device=dev) for l, (h, w) in enumerate(shapes)]
    up = torch.randn(frames, C, H, W, generator=g, device=dev)
    for _ in range(2):
        o, t = ops.pyramid_forward(noisy, logits, demod, prev, ksize=k)
        ops.pyramid_backward(t, up, want_param_grads=want)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
