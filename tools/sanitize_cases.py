"""Small shapes of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Families exercised: the config-5 training step at batch 2 (Cin = 1 mma.sync stencils, fused conv + max pool,
view-pair bwd-data, tap-reuse fwd / wgrad incl. CTA pairs, one-box-per-tap fwd / 2-CTA wgrad, pool fwd / bwd
kernels, head, SGD), fp32 NCHW convs (plane, tiled, f32 wgrad, direct, strided) and pools, bf16 strided
tcgen05 fwd / upsampled bwd, conv3d (depth-in-K tcgen05 and unfold), the ReLU-backward kernel and the
gather map.  Exits 0 after a device synchronize; the sanitizer's own report is the result."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1903_01814_b200 import functional as F  # noqa: E402
from paper_1903_01814_b200.hexcnn import HexCNN  # noqa: E402


def main():
    dev = "cuda"
    torch.manual_seed(0)
    # config-5 step at batch 2 (96 x 96)
    x = torch.from_numpy(np.ascontiguousarray(synth.shower_images(2, 96, 96, 47, 1).transpose(0, 2, 3, 1))
                         ).to(dev).to(torch.bfloat16)
    y = torch.from_numpy(synth.labels(2, 2)).to(dev)
    m = HexCNN(batch=2, seed=0)
    m.step(x, y)
    torch.cuda.synchronize()
    print("c5 step ok", flush=True)

    # fp32 NCHW: plane (Cin = 1), tiled / f32-wgrad (s = 1), direct (s = 2, 3), pools
    for (B, Ci, Co, H, W, n, s) in [(2, 1, 16, 12, 13, 1, 1), (2, 4, 8, 11, 12, 2, 1), (2, 16, 32, 14, 14, 2, 2),
                                    (1, 3, 5, 9, 10, 1, 3)]:
        xx = torch.randn(B, Ci, H, W, device=dev)
        w = torch.randn(Co, Ci, F.num_taps(n), device=dev) * 0.1
        b = torch.randn(Co, device=dev)
        yy = F.conv2d_fwd(xx, w, b, n=n, stride=s, relu=True)
        g = torch.randn_like(yy)
        F.conv2d_bwd_data(g, w, (H, W), n=n, stride=s, relu_y=xx if Ci > 1 else None)
        F.conv2d_bwd_weight(xx, g, n=n, stride=s)
        F.relu_bwd(g, yy)
    for mode in ("max", "avg", "avg_pad"):
        for layout, dt, C in (("NCHW", torch.float32, 3), ("NHWC", torch.bfloat16, 64)):
            xx = torch.randn(2, 12, 13, C, device=dev).to(dt)
            if layout == "NCHW":
                xx = xx.permute(0, 3, 1, 2).contiguous()
            p, am = F.pool2d_fwd(xx, n=1, stride=2, mode=mode, layout=layout)
            F.pool2d_bwd(torch.randn_like(p.float()).to(dt), am, (12, 13), n=1, stride=2, mode=mode, layout=layout)
    torch.cuda.synchronize()
    print("fp32 convs / pools ok", flush=True)

    # bf16 NHWC tcgen05: stride 2 forward, upsampled strided backward, C4-like 256 channels
    xb = torch.randn(1, 20, 22, 64, device=dev).to(torch.bfloat16)
    wb = (torch.randn(128, 64, 7, device=dev) * 0.05).to(torch.bfloat16)
    yb = F.conv2d_fwd(xb, wb, None, n=1, stride=2, layout="NHWC")
    gb = torch.randn_like(yb.float()).to(torch.bfloat16)
    F.conv2d_bwd_data(gb, wb, (20, 22), n=1, stride=2, layout="NHWC")
    F.conv2d_bwd_weight(xb, gb, n=1, stride=2, layout="NHWC")
    x4 = torch.randn(1, 16, 16, 256, device=dev).to(torch.bfloat16)
    for n in (1, 2):
        w4 = (torch.randn(256, 256, F.num_taps(n), device=dev) * 0.02).to(torch.bfloat16)
        y4 = F.conv2d_fwd(x4, w4, None, n=n, layout="NHWC")
        F.conv2d_bwd_data(y4, w4, (16, 16), n=n, layout="NHWC")
        F.conv2d_bwd_weight(x4, y4, n=n, layout="NHWC")
    torch.cuda.synchronize()
    print("tcgen05 ok", flush=True)

    # conv3d: depth-in-K tcgen05 path and the unfold path (fp32 NCDHW)
    x3 = torch.randn(1, 5, 12, 12, 64, device=dev).to(torch.bfloat16)
    w3 = (torch.randn(64, 64, 3, 7, device=dev) * 0.05).to(torch.bfloat16)
    y3 = F.conv3d_fwd(x3, w3, None, n=1, layout="NDHWC")
    F.conv3d_bwd_data(y3, w3, (5, 12, 12), n=1, layout="NDHWC")
    F.conv3d_bwd_weight(x3, y3, 3, n=1, layout="NDHWC")
    x3f = torch.randn(1, 2, 4, 9, 9, device=dev)
    w3f = torch.randn(3, 2, 3, 7, device=dev) * 0.1
    y3f = F.conv3d_fwd(x3f, w3f, None, n=1)
    F.conv3d_bwd_data(y3f, w3f, (4, 9, 9), n=1)
    F.conv3d_bwd_weight(x3f, y3f, 3, n=1)
    F.gather_map(9, 10, 2, stride=2)
    torch.cuda.synchronize()
    print("conv3d / gather map ok", flush=True)


if __name__ == "__main__":
    main()
