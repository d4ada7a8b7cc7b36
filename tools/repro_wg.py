"""Run the weight gradient of one layer shape once and synchronise (development repro)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import functional as F  # noqa: E402

B, Ci, Co, H, W, n = (int(v) for v in sys.argv[1:7])
x = torch.randn(B, H, W, Ci, device="cuda").to(torch.bfloat16)
g = torch.randn(B, H, W, Co, device="cuda").to(torch.bfloat16)
dw, db = F.conv2d_bwd_weight(x, g, n=n, layout="NHWC")
torch.cuda.synchronize()
ref = torch.einsum("bhwc->c", g.float())
print("ok", (db - ref).abs().max().item(), ref.abs().max().item())
