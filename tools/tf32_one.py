"""Run the C3 layer-2 fp32 conv passes (fwd, bwd-data) on the 3xTF32 kernel a few times (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import functional as F  # noqa: E402

B, H, W = 256, 40, 40
which = sys.argv[1] if len(sys.argv) > 1 else "l2"
ci, co, n = {"l2": (16, 32, 2), "l4": (32, 64, 1)}[which]
if which == "l4":
    H = W = 20
x = torch.randn(B, ci, H, W, device="cuda")
w = torch.randn(co, ci, F.num_taps(n), device="cuda") * 0.05
dy = torch.randn(B, co, H, W, device="cuda")
y = torch.empty(B, co, H, W, device="cuda")
dx = torch.empty_like(x)
for _ in range(3):
    F.conv2d_fwd(x, w, None, n=n, out=y)
    F.conv2d_bwd_data(dy, w, (H, W), n=n, out=dx)
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record()
for _ in range(10):
    F.conv2d_fwd(x, w, None, n=n, out=y)
e1.record()
for _ in range(10):
    F.conv2d_bwd_data(dy, w, (H, W), n=n, out=dx)
e2.record()
torch.cuda.synchronize()
print(which, "fwd us", e0.elapsed_time(e1) * 100, "dgrad us", e1.elapsed_time(e2) * 100)
