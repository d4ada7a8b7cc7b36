"""Development timing of the NCHW n = 1, stride 2 pool kernels (config-3 / config-2 shapes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import _abi as A  # noqa: E402
from paper_1903_01814_b200 import functional as F  # noqa: E402


def t(fn, it=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


for (B, C, H, W) in [(256, 32, 40, 40), (32, 32, 24, 24)]:
    x = torch.randn(B, C, H, W, device="cuda")
    for mode in ("avg", "max"):
        y, am = F.pool2d_fwd(x, n=1, stride=2, mode=mode)
        g = torch.randn_like(y)
        dx = torch.empty_like(x)
        r = {"fwd": t(lambda: F.pool2d_fwd(x, n=1, stride=2, mode=mode, out=y)),
             "bwd": t(lambda: F.pool2d_bwd(g, am, (H, W), n=1, stride=2, mode=mode, out=dx)),
             "bwd+relu": t(lambda: F.pool2d_bwd(g, am, (H, W), n=1, stride=2, mode=mode, out=dx, relu_y=x))}
        with A.switch("HEXCONV_POOL_GENERIC"):
            r["old fwd"] = t(lambda: F.pool2d_fwd(x, n=1, stride=2, mode=mode, out=y))
            r["old bwd"] = t(lambda: F.pool2d_bwd(g, am, (H, W), n=1, stride=2, mode=mode, out=dx))
        print((B, C, H, W), mode, {k: round(v, 1) for k, v in r.items()})
