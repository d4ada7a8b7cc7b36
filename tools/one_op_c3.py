"""Run the config-3 (fp32 NCHW, 256 x 40x40) ops a few times: ncu target.

usage: python tools/one_op_c3.py {l1fwd|l1wgrad|l2fwd|l2dgrad|l2wgrad|avgf|avgb} [iters]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import functional as F  # noqa: E402


def main():
    op = sys.argv[1]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    B, H, W = 256, 40, 40
    x1 = torch.randn(B, 1, H, W, device="cuda")
    x16 = torch.randn(B, 16, H, W, device="cuda")
    g16 = torch.randn(B, 16, H, W, device="cuda")
    g32 = torch.randn(B, 32, H, W, device="cuda")
    w1 = torch.randn(16, 1, 7, device="cuda") * 0.3
    w2 = torch.randn(32, 16, 19, device="cuda") * 0.05
    p32 = torch.randn(B, 32, 20, 20, device="cuda")
    for _ in range(iters):
        if op == "l1fwd":
            F.conv2d_fwd(x1, w1, None, n=1, relu=True)
        elif op == "l1wgrad":
            F.conv2d_bwd_weight(x1, g16, n=1)
        elif op == "l2fwd":
            F.conv2d_fwd(x16, w2, None, n=2)
        elif op == "l2dgrad":
            F.conv2d_bwd_data(g32, w2, (H, W), n=2)
        elif op == "l2wgrad":
            F.conv2d_bwd_weight(x16, g32, n=2)
        elif op == "avgf":
            F.pool2d_fwd(g32, n=1, stride=2, mode="avg")
        elif op == "avgb":
            F.pool2d_bwd(p32, None, (H, W), n=1, stride=2, mode="avg")
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
