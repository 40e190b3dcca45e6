"""Small fixed workload for ncu / compute-sanitizer runs (one GPU).

    python tools/prof_case.py [--frames 4] [--h 1080 --w 1920 --levels 3 --k 5 --ldt f32] [--iters 3]

Runs `iters` forward+backward passes of the pyramid filter through the C ABI
on synthetic BASELINE-distributed inputs.  Launch order per iteration:
pool(L-1), fwd(L levels, coarse->fine), bwd(L levels, fine->coarse), final.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--h", type=int, default=1080)
    ap.add_argument("--w", type=int, default=1920)
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--ldt", default="f32")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    noisy, demod, logits, up = bench.synthetic_inputs(a.frames, a.h, a.w, a.levels, a.k, a.ldt, dev, 7)
    r = bench.Runner(noisy, demod, logits, up, a.k)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(a.iters):
        r.step(s)
    torch.cuda.synchronize()
    print("ok", a)


if __name__ == "__main__":
    main()
