"""Stride-2 bf16 NHWC forward: tcgen05 (default) vs CUDA-core (HEXCONV_NO_TC_STRIDE2=1), development timing."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import functional as F  # noqa: E402


def timed(fn, it=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


def main():
    B, C, Co, H, W, n = 64, 128, 128, 96, 96, 1
    x = torch.randn(B, H, W, C, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Co, C, F.num_taps(n), device="cuda") / (C * 7) ** 0.5).to(torch.bfloat16)
    Ho, Wo, _ = F.output_shape(H, W, 2)
    g = torch.randn(B, Ho, Wo, Co, device="cuda").to(torch.bfloat16)
    flops = 2.0 * B * Ho * Wo * 7 * C * Co
    for name, pid, fn in (("fwd", 0, lambda: F.conv2d_fwd(x, w, None, n=n, stride=2, layout="NHWC")),
                          ("dgrad", 1, lambda: F.conv2d_bwd_data(g, w, (H, W), n=n, stride=2, layout="NHWC")),
                          ("wgrad", 2, lambda: F.conv2d_bwd_weight(x, g, n=n, stride=2, layout="NHWC"))):
        us = timed(fn)
        print(f"stride-2 {name} {B}x{C}->{Co} {H}x{W} n{n}: {us:.1f} us  {flops / us / 1e6:.1f} TFLOP/s "
              f"(nominal taps)  algo={F.conv_algo(B, C, Co, H, W, n, 2, 0, torch.bfloat16, 'NHWC', pid)}")


if __name__ == "__main__":
    main()
