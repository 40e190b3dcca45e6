"""Where the drop-in caller's time goes (compat reconstruct_core +
reconstruct_backward at 1080p L3 k5, f32 kernels): cProfile top entries."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_08642_b200 import compat  # noqa: E402

H, W, L, k = 1080, 1920, 3, 5
rng = np.random.default_rng(5)
shapes = [(1080, 1920), (540, 960), (270, 480)]
chans = [54, 29, 25]


class KF:
    def __init__(self, lg):
        self.logits = lg


kf = KF([rng.normal(0, 1, (h, w, c)) for (h, w), c in zip(shapes, chans)])
noisy = rng.lognormal(-1.0, 1.5, (H, W, 3))
demod = rng.uniform(0.05, 1.0, (H, W, 3))
up = rng.normal(size=(H, W, 3))
compat.set_precision("f32")


def frame():
    out, tape = compat.pyramid.reconstruct_core(noisy, kf, None, demod)
    return compat.pyramid.reconstruct_backward(tape, up)


frame()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(2):
    frame()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
