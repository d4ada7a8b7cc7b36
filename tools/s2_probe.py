"""Stride-2 bf16 NHWC forward: tcgen05 (default) vs CUDA-core (HEXCONV_NO_TC_STRIDE2=1), development timing."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import functional as F  # noqa: E402


def main():
    B, C, Co, H, W, n = 64, 128, 128, 96, 96, 1
    x = torch.randn(B, H, W, C, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Co, C, F.num_taps(n), device="cuda") / (C * 7) ** 0.5).to(torch.bfloat16)
    for _ in range(3):
        F.conv2d_fwd(x, w, None, n=n, stride=2, layout="NHWC")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        F.conv2d_fwd(x, w, None, n=n, stride=2, layout="NHWC")
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    Ho, Wo, _ = F.output_shape(H, W, 2)
    flops = 2.0 * B * Ho * Wo * 7 * C * Co
    print(f"stride-2 fwd {B}x{C}->{Co} {H}x{W} n{n}: {us:.1f} us  {flops / us / 1e6:.1f} TFLOP/s (nominal taps)"
          f"  algo={F.conv_algo(B, C, Co, H, W, n, 2, 0, torch.bfloat16, 'NHWC')}")


if __name__ == "__main__":
    main()
