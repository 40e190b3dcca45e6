"""Small fixed workload for ncu: the 8(f) rows (temporal warp + transpose,
score gradient, tonemap + loss epilogue) at 8 x 1080p fp32."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_08642_b200 import ops  # noqa: E402

B, H, W = 8, 1080, 1920
gen = torch.Generator(device="cuda").manual_seed(5)
prev = torch.rand((B, 3, H, W), device="cuda", generator=gen)
motion = (torch.rand((B, 2, H, W), device="cuda", generator=gen) - 0.5) * 4
g = torch.randn((B, 3, H, W), device="cuda", generator=gen)
sc = torch.randn((B, H, W), device="cuda", generator=gen)
gi = torch.randn((B, 2, 3, H, W), device="cuda", generator=gen)
gd = torch.randn((B, 2, 3, H, W), device="cuda", generator=gen)
rad = torch.rand((B, 3, H, W), device="cuda", generator=gen) * 4
ref = torch.rand((B, 3, H, W), device="cuda", generator=gen)
l0w = torch.rand((B, 3, H, W), device="cuda", generator=gen)
rw = torch.rand((B, 3, H, W), device="cuda", generator=gen)
val = (torch.rand((B, H, W), device="cuda", generator=gen) > 0.1).float()
msk = torch.ones((B, H, W), device="cuda")
tmo = (0.0, 1.0, 1.0, 0.5, 0.5)
for _ in range(2):
    ops.warp(prev, motion)
    ops.warp_backward(g, motion)
    ops.score_grad(sc, gi, gd, 0.25, 1.5)
    ldr = ops.tonemap(rad, tmo)
    r = ops.losses(ldr, ref, l0w, rw, validity=val, mask=msk, want_maps=False, want_grads=True)
    ops.tonemap_backward(rad, tmo, r["g_ldr1"])
    ops.loss_epilogue(rad, ref, tmo, l0w, rw, validity=val, mask=msk)
torch.cuda.synchronize()
print("ok")
