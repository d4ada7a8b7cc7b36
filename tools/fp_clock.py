"""Sustained-load clocks and power of one C5 op: loops the op for ~2 s while NVML is sampled every
50 ms; prints the per-call device time, median SM clock, median board power and the clock-event
reasons (0x4 = sw_power_cap).  Separates power-capped kernels from latency-bound ones.

usage: python tools/fp_clock.py {fused|l2dgrad|l2fwd|l6wgrad|l5fwd} [iters]
"""
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import functional as F  # noqa: E402


def make(op):
    bf = torch.bfloat16
    if op in ("fused", "l2fwd", "l2dgrad"):
        B, Ci, Co, H, W, n = 256, 64, 128, 96, 96, 1
    elif op == "l6wgrad":
        B, Ci, Co, H, W, n = 256, 256, 256, 24, 24, 1
    else:  # l5fwd
        B, Ci, Co, H, W, n = 256, 256, 256, 24, 24, 2
    T = F.num_taps(n)
    x = torch.randn(B, H, W, Ci, device="cuda").to(bf)
    w = (torch.randn(Co, Ci, T, device="cuda") / (Ci * T) ** 0.5).to(bf)
    g = torch.randn(B, H, W, Co, device="cuda").to(bf)
    b = torch.zeros(Co, device="cuda")
    if op == "fused":
        return lambda: F.conv2d_fwd_maxpool(x, w, b, n=n)
    if op == "l2dgrad":
        return lambda: F.conv2d_bwd_data(g, w, (H, W), n=n, layout="NHWC", relu_y=x)
    if op == "l6wgrad":
        return lambda: F.conv2d_bwd_weight(x, g, n=n, layout="NHWC")
    return lambda: F.conv2d_fwd(x, w, b, n=n, layout="NHWC")


def main():
    op = sys.argv[1] if len(sys.argv) > 1 else "fused"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6000
    fn = make(op)
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    clks, pw, stop = [], [], [False]

    def sample():
        while not stop[0]:
            clks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000)
            time.sleep(0.05)

    t = threading.Thread(target=sample)
    t.start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop[0] = True
    t.join()
    reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    clks.sort()
    pw.sort()
    label = op + (" " + os.environ["LABEL"] if "LABEL" in os.environ else "")
    print(f"{label:24s} {e0.elapsed_time(e1) / iters * 1e3:7.1f} us  sm_mhz med {clks[len(clks) // 2]}  "
          f"power med {pw[len(pw) // 2]:.0f} W  reasons 0x{reasons:x}", flush=True)


if __name__ == "__main__":
    main()
