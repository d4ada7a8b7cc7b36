"""Run one hex-conv / pool op a few times (target for ncu captures).

usage: python tools/one_op.py {fwd|dgrad|wgrad|poolf|poolb} B Cin Cout H W n [iters]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import functional as F  # noqa: E402


def main():
    op = sys.argv[1]
    B, Ci, Co, H, W, n = (int(v) for v in sys.argv[2:8])
    iters = int(sys.argv[8]) if len(sys.argv) > 8 else 3
    T = F.num_taps(n)
    x = torch.randn(B, H, W, Ci, device="cuda").to(torch.bfloat16)
    g = torch.randn(B, H, W, Co, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Co, Ci, T, device="cuda") / (Ci * T) ** 0.5).to(torch.bfloat16)
    for _ in range(iters):
        if op == "fwd":
            F.conv2d_fwd(x, w, None, n=n, layout="NHWC")
        elif op == "dgrad":
            F.conv2d_bwd_data(g, w, (H, W), n=n, layout="NHWC")
        elif op == "wgrad":
            F.conv2d_bwd_weight(x, g, n=n, layout="NHWC")
        elif op == "convpool":
            F.conv2d_fwd_maxpool(x, w, None, n=n)
        elif op == "poolf":
            F.pool2d_fwd(x, 1, 2, 0, "max", "NHWC")
        elif op == "l1fwd":
            x1 = torch.randn(B, H, W, 1, device="cuda").to(torch.bfloat16)
            w1 = (torch.randn(Co, 1, T, device="cuda") / T ** 0.5).to(torch.bfloat16)
            F.conv2d_fwd(x1, w1, None, n=n, layout="NHWC")
        elif op == "l1wgrad":
            x1 = torch.randn(B, H, W, 1, device="cuda").to(torch.bfloat16)
            F.conv2d_bwd_weight(x1, g, n=n, layout="NHWC")
        elif op == "poolb":
            y, am = F.pool2d_fwd(x, 1, 2, 0, "max", "NHWC")
            F.pool2d_bwd(torch.randn_like(y), am, (H, W), 1, 2, 0, "max", "NHWC")
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
