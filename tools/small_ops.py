"""CUDA-graph timing (hot / L2-flushed, bench.py's GraphTimer) of the small config-3 / config-5 ops one at a
time -- the quick check used while tuning them.

    python tools/small_ops.py [op ...]     (default: all)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from bench import GraphTimer  # noqa: E402
from paper_1903_01814_b200 import functional as F  # noqa: E402


def c3_ops():
    B, H, W = 256, 40, 40
    H2, W2, _ = F.output_shape(H, W, 2)
    x = torch.from_numpy(synth.shower_images(B, H, W, 12, 3).astype(np.float32)).cuda()
    w1 = torch.from_numpy(synth.kaiming_uniform((16, 1, 7), 20).astype(np.float32)).cuda()
    b1 = torch.zeros(16, device="cuda")
    y1 = torch.empty(B, 16, H, W, device="cuda")
    g1 = torch.randn(B, 16, H, W, device="cuda")
    y2 = torch.randn(B, 32, H, W, device="cuda")
    p = torch.empty(B, 32, H2, W2, device="cuda")
    dp = torch.randn(B, 32, H2, W2, device="cuda")
    dy2 = torch.empty(B, 32, H, W, device="cuda")
    dw = torch.empty(16, 1, 7, device="cuda")
    x16 = torch.randn(B, 16, H, W, device="cuda")
    w2 = torch.randn(32, 16, 19, device="cuda") * 0.05
    g32 = torch.randn(B, 32, H, W, device="cuda")
    p32 = torch.randn(B, 32, H2, W2, device="cuda")
    w4 = torch.randn(64, 32, 7, device="cuda") * 0.05
    g64 = torch.randn(B, 64, H2, W2, device="cuda")
    o = {k: torch.empty(sh, device="cuda") for k, sh in (("y2", (B, 32, H, W)), ("dx16", (B, 16, H, W)),
                                                          ("y4", (B, 64, H2, W2)), ("dp", (B, 32, H2, W2)))}
    dw2 = torch.empty(32, 16, 19, device="cuda")
    dw4 = torch.empty(64, 32, 7, device="cuda")
    return {
        "c3_l2_fwd": lambda: F.conv2d_fwd(x16, w2, None, n=2, out=o["y2"]),
        "c3_l2_dgrad": lambda: F.conv2d_bwd_data(g32, w2, (H, W), n=2, out=o["dx16"]),
        "c3_l2_wgrad": lambda: F.conv2d_bwd_weight(x16, g32, n=2, dw=dw2),
        "c3_l4_fwd": lambda: F.conv2d_fwd(p32, w4, None, n=1, out=o["y4"]),
        "c3_l4_dgrad": lambda: F.conv2d_bwd_data(g64, w4, (H2, W2), n=1, out=o["dp"]),
        "c3_l4_wgrad": lambda: F.conv2d_bwd_weight(p32, g64, n=1, dw=dw4),
        "c3_l1_fwd": lambda: F.conv2d_fwd(x, w1, b1, n=1, relu=True, out=y1),
        "c3_l1_wgrad": lambda: F.conv2d_bwd_weight(x, g1, n=1, dw=dw),
        "c3_pool_fwd_avg": lambda: F.pool2d_fwd(y2, n=1, stride=2, mode="avg", out=p),
        "c3_pool_bwd_relu": lambda: F.pool2d_bwd(dp, None, (H, W), n=1, stride=2, mode="avg", out=dy2, relu_y=y2),
    }


def c2_ops():
    # config 2: 32 x 16 -> 32, 48 x 48, n = 2, stride 2 (fp32 NCHW)
    B, H, W = 32, 48, 48
    Ho, Wo, _ = F.output_shape(H, W, 2)
    x = torch.randn(B, 16, H, W, device="cuda")
    w = torch.randn(32, 16, 19, device="cuda") * 0.06
    g = torch.randn(B, 32, Ho, Wo, device="cuda")
    y = torch.empty(B, 32, Ho, Wo, device="cuda")
    dx = torch.empty(B, 16, H, W, device="cuda")
    dw = torch.empty(32, 16, 19, device="cuda")
    return {"c2_fwd": lambda: F.conv2d_fwd(x, w, None, n=2, stride=2, out=y),
            "c2_dgrad": lambda: F.conv2d_bwd_data(g, w, (H, W), n=2, stride=2, out=dx),
            "c2_wgrad": lambda: F.conv2d_bwd_weight(x, g, n=2, stride=2, dw=dw)}


def c5_ops():
    B, H, W, Ci, Co = 256, 96, 96, 64, 128
    g = torch.Generator().manual_seed(0)
    x = torch.randn(B, H, W, Ci, generator=g).to(torch.bfloat16).cuda()
    w = (torch.randn(Co, Ci, 7, generator=g) / 21.0).to(torch.bfloat16).cuda()
    b = torch.zeros(Co, device="cuda")
    y = torch.randn(B, H, W, Co, generator=g).to(torch.bfloat16).cuda()
    x2 = torch.empty_like(x)
    x1 = torch.randn(B, H, W, 1, generator=g).to(torch.bfloat16).cuda()  # layer 1: 1 -> 64, n = 2
    w1 = (torch.randn(Ci, 1, 19, generator=g) / 4.4).to(torch.bfloat16).cuda()
    b1 = torch.zeros(Ci, device="cuda")
    dw1 = torch.empty(Ci, 1, 19, device="cuda")
    return {
        "c5_l2_fwd_maxpool": lambda: F.conv2d_fwd_maxpool(x, w, b, n=1),
        "c5_l2_fwd_avgpool": lambda: F.conv2d_fwd_avgpool(x, w, b, n=1),
        "c5_l2_fwd_maxpool_nobias": lambda: F.conv2d_fwd_maxpool(x, w, None, n=1),
        "c5_l2_fwd_then_avgpool": lambda: (F.conv2d_fwd(x, w, b, n=1, relu=True, layout="NHWC", out=y),
                                           F.pool2d_fwd(y, 1, 2, 0, "avg", "NHWC")),
        "c5_l2_dgrad": lambda: F.conv2d_bwd_data(y, w, (H, W), n=1, layout="NHWC", relu_y=x, out=x2),
        "c5_l1_fwd": lambda: F.conv2d_fwd(x1, w1, b1, n=2, relu=True, layout="NHWC", out=x2),
        "c5_l1_wgrad": lambda: F.conv2d_bwd_weight(x1, x, n=2, layout="NHWC", dw=dw1, dbias=b1),
    }



def c5_wgrad_ops():
    # config-5 CTA-pair weight gradients: layer 4 (128 -> 256, n = 1, 48 x 48), 5 (256 -> 256, n = 2, 24 x 24),
    # 6 (256 -> 256, n = 1, 24 x 24)
    out = {}
    for name, (ci, co, hw, n) in {"c5_l2_wgrad": (64, 128, 96, 1), "c5_l3_wgrad": (128, 128, 48, 2),
                                  "c5_l4_wgrad": (128, 256, 48, 1), "c5_l5_wgrad": (256, 256, 24, 2),
                                  "c5_l6_wgrad": (256, 256, 24, 1)}.items():
        x = torch.randn(256, hw, hw, ci, device="cuda").to(torch.bfloat16)
        g = torch.randn(256, hw, hw, co, device="cuda").to(torch.bfloat16)
        dw = torch.empty(co, ci, F.num_taps(n), device="cuda")
        db = torch.empty(co, device="cuda")
        out[name] = (lambda x=x, g=g, dw=dw, db=db, n=n:
                     F.conv2d_bwd_weight(x, g, n=n, layout="NHWC", dw=dw, dbias=db))
        w = (torch.randn(co, ci, F.num_taps(n), device="cuda") / 40).to(torch.bfloat16)
        y = torch.empty(256, hw, hw, co, device="cuda", dtype=torch.bfloat16)
        out[name.replace("wgrad", "fwd")] = (lambda x=x, w=w, y=y, n=n:
                                             F.conv2d_fwd(x, w, None, n=n, layout="NHWC", out=y))
    return out


def c3d_ops():
    B, D, H, W, C, Co, kd, n = 16, 16, 64, 64, 64, 128, 3, 1
    x = torch.randn(B, D, H, W, C, device="cuda").to(torch.bfloat16)
    g3 = torch.randn(B, D, H, W, Co, device="cuda").to(torch.bfloat16)
    return {"c3d_wgrad": lambda: F.conv3d_bwd_weight(x, g3, kd, n=n, layout="NDHWC")}


def s2_ops(s=2):
    # strided bf16 layer (f4): 64 images 96x96, 128 -> 128 channels, stride s (ops "s2_*" / "s3_*")
    B, C, H, W = 64, 128, 96, 96
    Ho, Wo, _ = F.output_shape(H, W, s)
    out = {}
    for n in (1, 2):
        T = F.num_taps(n)
        w = (torch.randn(C, C, T, device="cuda") / (C * T) ** 0.5).to(torch.bfloat16)
        g = torch.randn(B, Ho, Wo, C, device="cuda").to(torch.bfloat16)
        dx = torch.empty(B, H, W, C, device="cuda", dtype=torch.bfloat16)
        out[f"s{s}_n{n}_dgrad"] = (lambda w=w, g=g, dx=dx, n=n:
                                 F.conv2d_bwd_data(g, w, (H, W), n=n, stride=s, layout="NHWC", out=dx))
        x = torch.randn(B, H, W, C, device="cuda").to(torch.bfloat16)
        y = torch.empty(B, Ho, Wo, C, device="cuda", dtype=torch.bfloat16)
        out[f"s{s}_n{n}_fwd"] = (lambda w=w, x=x, y=y, n=n:
                                 F.conv2d_fwd(x, w, None, n=n, stride=s, layout="NHWC", out=y))
        dw = torch.empty(C, C, T, device="cuda")
        out[f"s{s}_n{n}_wgrad"] = (lambda x=x, g=g, dw=dw, n=n:
                                 F.conv2d_bwd_weight(x, g, n=n, stride=s, layout="NHWC", dw=dw))
    return out


def nvls_ops():
    # NVLS gradient sum of the config-5 gradient vector, one multicast replica (one GPU): the protocol's cost
    from paper_1903_01814_b200 import nvls
    from paper_1903_01814_b200.hexcnn import HexCNN
    m = HexCNN(batch=2)
    buf = nvls.NvlsBuffer(4 * m.nparams, local=not nvls.supported())
    nvls_ops.keep = buf
    segs = [m._segment_range(l) for l in range(m.L + 1)]

    def run():
        for l, (off, n) in enumerate(segs):
            buf.allreduce(off, n, l)
    return {"nvls_c5_buckets": run, "nvls_c5_l5": lambda: buf.allreduce(*segs[4], 20)}


def main():
    ops = c3_ops()
    if any(a.startswith("c2") for a in sys.argv[1:]):
        ops.update(c2_ops())
    if any(a.startswith("nvls") for a in sys.argv[1:]):
        ops.update(nvls_ops())
    if any(a.startswith("s2") for a in sys.argv[1:]):
        ops.update(s2_ops(2))
    if any(a.startswith("s3") for a in sys.argv[1:]):
        ops.update(s2_ops(3))
    if any(a.startswith("c3d") for a in sys.argv[1:]):
        ops.update(c3d_ops())
    if any(a.startswith("c5") for a in sys.argv[1:]):
        ops.update(c5_ops())
        ops.update(c5_wgrad_ops())
    sel = sys.argv[1:] or list(ops)
    gt = GraphTimer("cuda")
    for name in sel:
        g = gt.capture(ops[name])
        hot, fl = gt.time(g, 50)
        print(f"{name:22s} hot {hot * 1e3:8.2f} us   flushed {fl * 1e3:8.2f} us")


if __name__ == "__main__":
    main()
