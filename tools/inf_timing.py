"""Stage times of the small-frame cooperative inference kernel (experiment
build SSB_NVCC_FLAGS=-DSSB_INF_TIMING, loaded through SSB_LIB_PATH)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_08642_b200 import _lib, ops  # noqa: E402
from tests.test_gpu_infer import _inputs  # noqa: E402

s, b, d, l = _inputs(ops, 1, 256, 256, 3, 5, 1)
lib = _lib.load()
for _ in range(5):
    ops.infer(s, b, d, l, 0.25, ksize=5)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
if hasattr(lib, "ssb_debug_inf_times"):
    lib.ssb_debug_inf_times(buf)
t = list(buf)
if not any(t):
    print("no stage times (library built without -DSSB_INF_TIMING)")
    sys.exit(0)
names = {1: "partials", 2: "fold+place", 3: "pools", 4: "fwd top", 5: "fwd l1", 12: "end"}
prev = t[0]
for k in (1, 2, 3, 4, 5, 12):
    if t[k]:
        print(f"{names[k]:>12s} {(t[k] - prev) / 1000:.2f} us")
        prev = t[k]
print("total", (t[12] - t[0]) / 1000, "us")
