"""Quick per-op timing probe (CUDA events on the launching stream, L2 flushed
between iterations).  Not the bench: a development tool.

usage: python tools/probe.py [c4|c5|c2|c3|all]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200 import functional as F  # noqa: E402

PEAK_TF = 1621.7
PEAK_GBS = 6538.3
flush_buf = None


def flush():
    """Evict L2 by READING a 256 MB buffer: a write-based flush leaves ~126 MB of
    dirty lines whose write-back would be charged to the next (timed) kernel."""
    global flush_buf
    if flush_buf is None:
        flush_buf = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    flush_buf.sum()


def _graph(body):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        body()
    torch.cuda.synchronize()
    return g


def _time_graph(g, iters):
    ts = []
    for _ in range(iters):
        s0, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(s0.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def timeit(fn, iters=5, warmup=3, reps=10):
    """Device time of one call with L2 flushed before it.  `reps` (flush, call)
    pairs are captured in one CUDA graph and the same number of flushes alone in
    another; the difference / reps is the call's time, free of host dispatch
    (tens of us per call through Python/ctypes) and of the flush itself."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()

    def pairs():
        for _ in range(reps):
            flush()
            fn()

    def flushes():
        for _ in range(reps):
            flush()

    gp, gf = _graph(pairs), _graph(flushes)
    return max(_time_graph(gp, iters) - _time_graph(gf, iters), 0.0) / reps


def valid_taps(H, W, n):
    m = F.gather_map(H, W, n)
    return int((m >= 0).sum().item())


def conv_layer(B, Ci, Co, H, W, n, dtype=torch.bfloat16, layout="NHWC", label=""):
    T = F.num_taps(n)
    if layout == "NHWC":
        x = torch.randn(B, H, W, Ci, device="cuda").to(dtype)
        g = torch.randn(B, H, W, Co, device="cuda").to(dtype)
    else:
        x = torch.randn(B, Ci, H, W, device="cuda").to(dtype)
        g = torch.randn(B, Co, H, W, device="cuda").to(dtype)
    w = (torch.randn(Co, Ci, T, device="cuda") / (Ci * T) ** 0.5).to(dtype)
    vt = valid_taps(H, W, n)
    flops = 2.0 * B * vt * Ci * Co
    res = {}
    for name, fn in [("fwd", lambda: F.conv2d_fwd(x, w, None, n=n, layout=layout)),
                     ("dgrad", lambda: F.conv2d_bwd_data(g, w, (H, W), n=n, layout=layout)),
                     ("wgrad", lambda: F.conv2d_bwd_weight(x, g, n=n, layout=layout))]:
        ms = timeit(fn)
        algo = F.conv_algo(B, Ci, Co, H, W, n, 1, 0, dtype, layout, {"fwd": 0, "dgrad": 1, "wgrad": 2}[name])
        tf = flops / ms / 1e9
        res[name] = ms
        print(f"{label:10s} {name:5s} B{B} {Ci}->{Co} {H}x{W} n{n} {algo:8s} {ms*1e3:9.1f} us  "
              f"{tf:8.1f} TFLOP/s  {tf/PEAK_TF*100:5.1f}% of {PEAK_TF}")
    return res


def fused_layer(B, Ci, Co, H, W, n, label=""):
    x = torch.randn(B, H, W, Ci, device="cuda").to(torch.bfloat16)
    w = (torch.randn(Co, Ci, F.num_taps(n), device="cuda") / (Ci * F.num_taps(n)) ** 0.5).to(torch.bfloat16)
    if not F.conv2d_fwd_maxpool_supported(B, Ci, Co, H, W, n):
        return
    ms = timeit(lambda: F.conv2d_fwd_maxpool(x, w, None, n=n))
    flops = 2.0 * B * valid_taps(H, W, n) * Ci * Co
    print(f"{label:10s} fused conv+relu+maxpool {ms*1e3:9.1f} us  {flops / ms / 1e9:8.1f} TFLOP/s (conv FLOPs)")


def pool_layer(B, C, H, W, n, s, mode, dtype=torch.bfloat16, layout="NHWC", label=""):
    x = torch.randn(B, H, W, C, device="cuda").to(dtype) if layout == "NHWC" else \
        torch.randn(B, C, H, W, device="cuda").to(dtype)
    Ho, Wo, _ = F.output_shape(H, W, s)
    y, am = F.pool2d_fwd(x, n, s, 0, mode, layout)
    g = torch.randn_like(y)
    es = x.element_size()
    fwd_bytes = x.numel() * es + y.numel() * es + (am.numel() if am is not None else 0)
    bwd_bytes = g.numel() * es + x.numel() * es + (am.numel() if am is not None else 0)
    for name, fn, nb in [("fwd", lambda: F.pool2d_fwd(x, n, s, 0, mode, layout), fwd_bytes),
                         ("bwd", lambda: F.pool2d_bwd(g, am, (H, W), n, s, 0, mode, layout), bwd_bytes)]:
        ms = timeit(fn)
        gbs = nb / ms / 1e6
        print(f"{label:10s} {mode}pool {name} B{B} C{C} {H}x{W} n{n} s{s} {ms*1e3:9.1f} us  {gbs:8.1f} GB/s "
              f" {gbs/PEAK_GBS*100:5.1f}% of {PEAK_GBS}")


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("c4", "all"):
        conv_layer(128, 256, 256, 64, 64, 1, label="C4 n1")
        conv_layer(128, 256, 256, 64, 64, 2, label="C4 n2")
    if which in ("c5", "all"):
        conv_layer(256, 1, 64, 96, 96, 2, label="C5 L1")
        conv_layer(256, 64, 128, 96, 96, 1, label="C5 L2")
        pool_layer(256, 128, 96, 96, 1, 2, "max", label="C5 P1")
        fused_layer(256, 64, 128, 96, 96, 1, label="C5 L2+P1")
        conv_layer(256, 128, 128, 48, 48, 2, label="C5 L3")
        conv_layer(256, 128, 256, 48, 48, 1, label="C5 L4")
        pool_layer(256, 256, 48, 48, 1, 2, "max", label="C5 P2")
        conv_layer(256, 256, 256, 24, 24, 2, label="C5 L5")
        conv_layer(256, 256, 256, 24, 24, 1, label="C5 L6")
    if which == "fused":
        fused_layer(256, 64, 128, 96, 96, 1, label="C5 L2+P1")
    if which in ("c3", "all"):
        conv_layer(256, 1, 16, 40, 40, 1, torch.float32, "NCHW", label="C3 L1")
        conv_layer(256, 16, 32, 40, 40, 2, torch.float32, "NCHW", label="C3 L2")
        pool_layer(256, 32, 40, 40, 1, 2, "avg", torch.float32, "NCHW", label="C3 P")
        conv_layer(256, 32, 64, 20, 20, 1, torch.float32, "NCHW", label="C3 L4")


if __name__ == "__main__":
    main()
