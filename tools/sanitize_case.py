"""Small, odd-sized invocations of the round-1 kernels, synchronously (an
illegal address surfaces at the launch that caused it):

    CUDA_LAUNCH_BLOCKING=1 python tools/sanitize_case.py   (compute-sanitizer is unavailable on the pool)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_08642_b200 import ops  # noqa: E402

dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)


def rnd(*s, dtype=torch.float32):
    return torch.rand(s, device=dev, generator=g).to(dtype)


# pyramid: TMA level kernels (k5 fp32 level-0-last, k7 bf16 pair forward), generic shapes
for (H, W, L, k, ldt) in [(72, 128, 4, 7, torch.bfloat16), (66, 136, 3, 5, torch.float32),
                          (45, 97, 3, 5, torch.float32), (33, 64, 5, 3, torch.float32)]:
    noisy, dm, up = rnd(2, 3, H, W) * 2, rnd(2, 3, H, W) * 0.9 + 0.05, rnd(2, 3, H, W) - 0.5
    lg = [(rnd(2, ops.logit_channels(l, L, k), h, w) * 4 - 2).to(ldt)
          for l, (h, w) in enumerate(ops.level_shapes(H, W, L))]
    out, t = ops.pyramid_forward(noisy, lg, dm, ksize=k)
    ops.pyramid_backward(t, up)
# temporal warp + transpose (staged / landing-mask paths and the general scan)
for (H, W, amp) in [(37, 70, 2.0), (19, 33, 3.0), (23, 41, 6.0)]:
    x, gr = rnd(1, 3, H, W), rnd(1, 3, H, W)
    m = (rnd(1, 2, H, W) - 0.5) * 2 * amp
    ops.warp(x, m)
    ops.warp_backward(gr, m)
# score gradient (radius-templated blur), tonemap / losses / fused epilogue
sc = rnd(2, 35, 61)
gi, gd = rnd(2, 2, 3, 35, 61), rnd(2, 2, 3, 35, 61)
for sigma in (0.0, 1.5, 3.9):
    ops.score_grad(sc, gi, gd, 0.25, sigma)
for (H, W) in [(33, 51), (32, 64)]:
    rad, ref, l0, rw = rnd(2, 3, H, W) * 4, rnd(2, 3, H, W), rnd(2, 3, H, W), rnd(2, 3, H, W)
    val, msk = (rnd(2, H, W) > 0.2).float(), rnd(2, H, W)
    t = (0.2, 1.3, 0.8, 0.35, 0.45)
    ldr = ops.tonemap(rad, t)
    r = ops.losses(ldr, ref, l0, rw, validity=val, mask=msk, want_grads=True)
    ops.tonemap_backward(rad, t, r["g_ldr1"])
    ops.loss_epilogue(rad, ref, t, l0, rw, validity=val, mask=msk, want_ldr=True)
torch.cuda.synchronize()
print("sanitize case ok")
