import sys, os
sys.path.insert(0, "/root/repo")
import torch, ctypes as C
from paper_2602_08642_b200 import ops
B, H, W = 8, 1080, 1920
g = torch.Generator(device="cuda").manual_seed(5)
scores = torch.randn(B, H, W, generator=g, device="cuda") * 0.5
bank = torch.exp(-1.0 + 1.5 * torch.randn(B, 2, 3, H, W, generator=g, device="cuda"))
noisy = torch.empty(B, 3, H, W, device="cuda")
wsb = C.c_size_t(); ops._lib.load().ssb_density_workspace_bytes(B, H, W, C.byref(wsb))
ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ops.place(scores, bank, 0.25, "relaxed", noisy=noisy, want_grad=True, workspace=ws)
torch.cuda.synchronize(); print("ok")
