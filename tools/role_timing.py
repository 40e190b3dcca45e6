"""Per-role cycle split of the TMA backward level kernels (experiment build:
SSB_NVCC_FLAGS=-DSSB_ROLE_TIMING, see build.py): for warps 0-3 (B1 logit
gradients) and 4-7 (B2 gather-transpose) the share of cycles spent waiting
for the step's TMA, in phase A (incl. its barrier), in the role's B work, and
at the end-of-step barrier.  Counters cover every k_pyr_bwd_tma launch of the
k's translation unit (all levels; level 0 dominates).

    python tools/role_timing.py [--k 5 --ldt f32 --frames 4 | --k 7 --ldt bf16 --h 2160 --w 3840 --levels 4 --frames 1]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_08642_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--h", type=int, default=1080)
    ap.add_argument("--w", type=int, default=1920)
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--ldt", default="f32")
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    lib = _lib.load()
    fns = [getattr(lib, f"ssb_debug_role_cycles{t}") for t in ("0", "3", "5", "7", "5b", "7b")]
    buf = (C.c_ulonglong * 8)()

    def read():
        tot = [0] * 8
        for f in fns:
            assert f(buf) == 0
            for i in range(8):
                tot[i] += buf[i]
        return tot
    noisy, demod, logits, up = bench.synthetic_inputs(a.frames, a.h, a.w, a.levels, a.k, a.ldt,
                                                      torch.device("cuda"), 7)
    r = bench.Runner(noisy, demod, logits, up, a.k)
    s = torch.cuda.current_stream().cuda_stream
    r.step(s)
    torch.cuda.synchronize()
    read()  # reset
    for _ in range(a.iters):
        r.step(s)
    torch.cuda.synchronize()
    buf = read()
    names = ["TMA wait", "phase A (+barrier)", "B work", "end-of-step barrier"]
    for role, label in ((0, "warps 0-3 (B1)"), (1, "warps 4-7 (B2)")):
        v = [buf[4 * role + k] for k in range(4)]
        tot = sum(v) or 1
        print(f"{label}: " + ", ".join(f"{n} {100 * x / tot:.1f}%" for n, x in zip(names, v)))


if __name__ == "__main__":
    main()
