"""Run the config-2 or config-3 fp32 fwd + bwd pass sequence (the same library calls bench.py times)
K times -- the target of the ncu launch list and full captures in profiles/r02.

    python tools/c23_step.py c3 [K]
    python tools/c23_step.py c2 [K]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1903_01814_b200 import functional as F  # noqa: E402


def c3_passes():
    c = synth.CONFIGS["c3"]
    B, H, W = c["B"], c["H"], c["W"]
    H2, W2, _ = F.output_shape(H, W, 2)
    x = torch.from_numpy(synth.shower_images(B, H, W, c["R"], 3).astype(np.float32)).cuda()
    convs = [(1, 16, 1), (16, 32, 2), (32, 64, 1)]
    ws = [torch.from_numpy(synth.kaiming_uniform((co, ci, F.num_taps(n)), 20 + i).astype(np.float32)).cuda()
          for i, (ci, co, n) in enumerate(convs)]
    bs = [torch.zeros(co, device="cuda") for _, co, _ in convs]
    t = {k: torch.empty(shape, device="cuda") for k, shape in (
        ("y1", (B, 16, H, W)), ("y2", (B, 32, H, W)), ("p", (B, 32, H2, W2)), ("y4", (B, 64, H2, W2)),
        ("dy4", (B, 64, H2, W2)), ("dp", (B, 32, H2, W2)), ("dy2", (B, 32, H, W)), ("dy1", (B, 16, H, W)))}
    g4 = torch.from_numpy(synth.normal((B, 64, H2, W2), 4).astype(np.float32)).cuda()

    def step():
        F.conv2d_fwd(x, ws[0], bs[0], n=1, relu=True, out=t["y1"])
        F.conv2d_fwd(t["y1"], ws[1], bs[1], n=2, relu=True, out=t["y2"])
        F.pool2d_fwd(t["y2"], n=1, stride=2, mode="avg", out=t["p"])
        F.conv2d_fwd(t["p"], ws[2], bs[2], n=1, relu=True, out=t["y4"])
        dy4 = F.relu_bwd(g4, t["y4"])
        F.conv2d_bwd_weight(t["p"], dy4, n=1)
        F.conv2d_bwd_data(dy4, ws[2], (H2, W2), n=1, out=t["dp"])
        F.pool2d_bwd(t["dp"], None, (H, W), n=1, stride=2, mode="avg", out=t["dy2"], relu_y=t["y2"])
        F.conv2d_bwd_weight(t["y1"], t["dy2"], n=2)
        F.conv2d_bwd_data(t["dy2"], ws[1], (H, W), n=2, relu_y=t["y1"], out=t["dy1"])
        F.conv2d_bwd_weight(x, t["dy1"], n=1)
    return step


def c2_passes():
    B, Ci, Co, H, W = 32, 16, 32, 48, 48
    x = torch.from_numpy(synth.normal((B, Ci, H, W), 0).astype(np.float32)).cuda()
    w = torch.from_numpy(synth.kaiming_uniform((Co, Ci, 19), 1).astype(np.float32)).cuda()
    y = F.conv2d_fwd(x, w, None, n=2, stride=2)
    p, am = F.pool2d_fwd(y, n=1, stride=2, mode="max")
    gp = torch.from_numpy(synth.normal(tuple(p.shape), 2).astype(np.float32)).cuda()

    def step():
        F.conv2d_fwd(x, w, None, n=2, stride=2, out=y)
        F.pool2d_fwd(y, n=1, stride=2, mode="max")
        gy = F.pool2d_bwd(gp, am, tuple(y.shape[-2:]), n=1, stride=2, mode="max")
        F.conv2d_bwd_data(gy, w, (H, W), n=2, stride=2)
        F.conv2d_bwd_weight(x, gy, n=2, stride=2)
    return step


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "c3"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    step = c3_passes() if which == "c3" else c2_passes()
    for _ in range(k):
        step()
    torch.cuda.synchronize()
    print(which, "ok")
