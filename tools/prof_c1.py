"""c1-shaped inference (one 1080p frame: fused placement + L3 k5 forward) for
an ncu launch list: python tools/prof_c1.py [H W]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_08642_b200 import ops  # noqa: E402

H, W = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1080, 1920)
L, k = 3, 5
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
scores = torch.randn(1, H, W, generator=g, device=dev)
bank = torch.exp(torch.randn(1, 2, 3, H, W, generator=g, device=dev))
demod = torch.rand(1, 3, H, W, generator=g, device=dev) * 0.9 + 0.1
logits = [torch.randn(1, ops.logit_channels(l, L, k), h, w, generator=g, device=dev)
          for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
noisy = torch.empty(1, 3, H, W, device=dev)
out = torch.empty_like(noisy)
for _ in range(3):
    ops.place_fused(scores[0:1], bank, 0.25, noisy=noisy)
    ops.pyramid_forward(noisy, logits, demod, ksize=k, out=out)
torch.cuda.synchronize()
print("ok")
