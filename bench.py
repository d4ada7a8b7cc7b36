"""bench.py -- BASELINE config 5: data-parallel training step of the 6-layer
hexagonal CNN (256 images per GPU, 96x96 offset-column grid, bf16 NHWC, fp32
master weights, weight-gradient allreduce over NCCL), reported as images/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, one rank per GPU)

One JSON line on rank 0:
  value     images/s of the whole job with inputs resident in HBM (device timed,
            CUDA events, barrier + synchronize on both sides, max over ranks)
  e2e       the same metric through the public API with each step's batch
            copied from pinned host memory and the loss read back
  roofline  the dominant kernel family (tcgen05 implicit-GEMM conv) against the
            measured sustained bf16 tensor-core peak, from live CUDA events
  cpu_baseline  the fp64 oracle (test infrastructure) on a bounded sample
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hex-conv TFLOP/s (valid taps) & pool/conv HBM GB/s vs B200 roofline; images/s 1–8 GPU"
WORKLOAD = "c5: 6-layer hex CNN (1-64-128-128-256-256-256, n=2,1,2,1,2,1, maxpool n1 s2 after L2/L4, GAP, linear->2, CE) DP train step, 256 img/GPU, 96x96"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        """Start nvidia-smi sampling every 100 ms and wait (<= 3 s) for its first sample, so that sampling is
        live when the timed region begins (nvidia-smi takes a few hundred ms to start)."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.first = len(self.lines)

    def mark(self):
        """Samples from here on belong to the measured region."""
        self.first = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        end = len(self.lines)  # samples taken while the measured region ran
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # the samples taken during the region; a region shorter than the 100 ms sampling period may hold
        # none: then the first one after it (<= 150 ms later), else the last one before it
        lines = (self.lines[self.first:end] or self.lines[end:end + 1] or
                 self.lines[max(0, self.first - 1):self.first])
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [v for v in sm if v > 0.5 * (mx or max(sm))] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ data
def make_batches(nb, B, H, W, R, seed):
    import numpy as np

    import synth
    xs, ys = [], []
    for i in range(nb):
        img = synth.shower_images(B, H, W, R, seed + i)            # [B,1,H,W] float32
        xs.append(np.ascontiguousarray(img.transpose(0, 2, 3, 1)))  # NHWC, C = 1
        ys.append(synth.labels(B, seed + 100 + i))
    return xs, ys


# ------------------------------------------------------------------ oracle legs (test infrastructure)
def oracle_train_sample(n_images: int, seed: int = 0):
    """One C5 training step of the fp64 oracle on n_images (a bounded sample of
    the workload): convs + ReLU + max pools forward, GAP/linear/CE head, full
    backward (dgrad, wgrad, pool bwd) and the SGD-momentum update.  Returns
    (seconds, threads)."""
    import numpy as np

    import oracle
    import synth
    ch = (1, 64, 128, 128, 256, 256, 256)
    ns = (2, 1, 2, 1, 2, 1)
    rng = np.random.default_rng(seed)
    Ws = [rng.uniform(-1, 1, size=(ch[l + 1], ch[l], oracle.num_taps(ns[l]))) * (6.0 / (ch[l] * oracle.num_taps(ns[l]))) ** 0.5
          for l in range(6)]
    bs = [np.zeros(ch[l + 1]) for l in range(6)]
    wl = rng.uniform(-1, 1, size=(2, 256)) / 16.0
    bl = np.zeros(2)
    x = synth.round_bf16(synth.shower_images(n_images, 96, 96, 47, seed + 7).astype(np.float64))
    lab = synth.labels(n_images, seed + 8)
    t0 = time.perf_counter()
    acts, inputs, pools = [], [], {}
    h = x
    for l in range(6):
        inputs.append(h)
        a = np.maximum(oracle.conv2d_fwd(h, Ws[l], bs[l], n=ns[l]), 0.0)
        acts.append(a)
        h = a
        if l in (1, 3):
            p, am = oracle.pool2d_fwd(a, n=1, s=2, mode="max")
            pools[l] = (p, am, a.shape[-2:])
            h = p
    gap = h.mean(axis=(2, 3))
    logits = gap @ wl.T + bl
    z = logits - logits.max(1, keepdims=True)
    pr = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    dlog = (pr - np.eye(2)[lab]) / n_images
    dwl, dbl = dlog.T @ gap, dlog.sum(0)
    g = (dlog @ wl)[:, :, None, None] / (h.shape[2] * h.shape[3]) * np.ones_like(h)
    for l in reversed(range(6)):
        g = g * (acts[l] > 0) if l not in (1, 3) else g
        if l in (1, 3):
            p, am, (H, W) = pools[l]
            g = oracle.pool2d_bwd(g, am, H, W, n=1, s=2, mode="max") * (acts[l] > 0)
        dx, dw, db = oracle.conv2d_bwd(inputs[l], Ws[l], g, n=ns[l], need=("dx", "dw", "db") if l else ("dw", "db"))
        Ws[l] -= 0.01 * dw
        bs[l] -= 0.01 * db
        g = dx
    wl -= 0.01 * dwl
    bl -= 0.01 * dbl
    return time.perf_counter() - t0, oracle.max_threads()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    n_img = 1
    for _ in range(args.warmup):
        oracle_train_sample(n_img)
    ts = []
    for _ in range(args.steps):
        dt, threads = oracle_train_sample(n_img)
        ts.append(dt)
    tot = sum(ts)
    value = n_img * len(ts) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / len(ts) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "global_batch": 256 * args.gpus, "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{n_img} image per step through the full C5 fwd+bwd+SGD in fp64 "
                                   f"(bounded sample of the 256-image batch)"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ secondary configs (BASELINE configs 1-4)
def ffma_peak():
    """Measured FP32 FFMA peak (TFLOP/s) for the CUDA-core conv rooflines: tools/ffma_peak.bin run live when
    it was built, else the committed profiles/r02/ffma_peak.json; the 'reg' form (three register operands,
    a convolution's weight x activation FFMA) is the denominator."""
    exe = os.path.join(ROOT, "tools", "ffma_peak.bin")
    if os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
            d = json.loads(out.stdout.strip().splitlines()[-1])
            d["source"] = "measured live (tools/ffma_peak.bin)"
            return d
        except Exception:
            pass
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "ffma_peak.json")) as f:
            d = json.load(f)
        d["source"] = "profiles/r02/ffma_peak.json (measured on this pool, committed)"
        return d
    except Exception:
        return {"ffma_tflops_reg": 74.4, "source": "derived 148 x 128 x 2 x 1.965 GHz (no measurement)"}


class GraphTimer:
    """Times a sequence of library calls as CUDA-graph replays (no host dispatch inside the timed region):
    'hot' = replays back to back (inputs L2-resident as in a steady training loop), 'flushed' = median of
    single replays each preceded by a 256 MB L2-evicting write outside the timed events."""

    def __init__(self, dev):
        import torch
        self.torch = torch
        self.flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def capture(self, fn):
        torch = self.torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()  # first-call work (allocations, function attributes) outside the capture
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    def time(self, g, iters=20):
        torch = self.torch
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        hot = e0.elapsed_time(e1) / iters
        evs = []
        for _ in range(iters):
            self.flush_buf.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        flushed = statistics.median(a.elapsed_time(b) for a, b in evs)
        return hot, flushed


def _pass_entry(hot, flushed, flops, nbytes, ffma, hbm):
    """One pass: times (us), achieved rates and the fraction of its roofline t_roof / t (flushed timing);
    t_roof = max(bytes / HBM, FLOPs / FFMA) -- SURVEY.md 8(d) 'Rooflines'."""
    e = {"us_flushed": flushed * 1e3, "us_hot": hot * 1e3}
    t_roof = max(nbytes / (hbm * 1e9), (flops or 0.0) / (ffma * 1e12))
    if flops:
        e["tflops"] = flops / (flushed * 1e-3) / 1e12
    e["gbs"] = nbytes / (flushed * 1e-3) / 1e9
    e["roofline_us"] = t_roof * 1e6
    e["bound"] = "ffma" if (flops or 0.0) / (ffma * 1e12) > nbytes / (hbm * 1e9) else "hbm"
    e["frac_of_roofline"] = t_roof / (flushed * 1e-3)
    e["frac_of_roofline_hot"] = t_roof / (hot * 1e-3)
    return e


def secondary_measurements(dev, peak_tf, peak_gbs):
    """BASELINE configs 1-4 (and the f2 conv3d shape), each pass captured in a CUDA graph and timed hot and
    L2-flushed (GraphTimer).  Rooflines: FP32 FFMA (measured, ffma_peak()) for the fp32 convs, HBM for pools
    and the Cin = 1 layer, the measured bf16 burst peak for the tensor-core convs; FLOPs count in-grid taps
    only ('valid taps'); bytes = inputs + weights + outputs moved once."""
    import numpy as np
    import torch

    import synth
    from paper_1903_01814_b200 import functional as F
    fp = ffma_peak()
    ffma = fp["ffma_tflops_reg"]
    gt = GraphTimer(dev)
    out = {"ffma_peak": fp}

    def vt(H, W, n, s=1):
        return int((F.gather_map(H, W, n, stride=s) >= 0).sum().item())

    # ---- C1: 4 x 1 -> 4, 16 x 16, n = 1, fp32 (BASELINE configs[0]): latency
    c = synth.CONFIGS["c1"]
    x1 = torch.from_numpy(synth.normal((4, 1, 16, 16), 0).astype(np.float32)).to(dev)
    w1 = torch.from_numpy((synth.normal((4, 1, 7), 1) * 0.1).astype(np.float32)).to(dev)
    b1 = torch.zeros(4, device=dev)
    y1 = torch.empty(4, 4, 16, 16, device=dev)
    g = gt.capture(lambda: F.conv2d_fwd(x1, w1, b1, n=1, out=y1))
    hot, fl = gt.time(g, 50)
    lat = []
    for _ in range(200):
        t0 = time.perf_counter()
        F.conv2d_fwd(x1, w1, b1, n=1, out=y1)
        torch.cuda.synchronize()
        lat.append(time.perf_counter() - t0)
    out["c1_4x1to4_16x16_f32"] = {
        "device_us_hot": hot * 1e3, "device_us_flushed": fl * 1e3,
        "host_call_to_sync_us_median": statistics.median(lat) * 1e6,
        "note": "launch-latency bound (20 KB, 53 kFLOP); device time = CUDA events around one graph replay of "
                "the single kernel; host latency = one eager ABI call + cudaDeviceSynchronize"}

    # ---- C2: 32 x 16 -> 32, 48 x 48, n2 s2 conv + max pool n1 s2, fp32, fwd + bwd
    B, Ci, Co, H, W = 32, 16, 32, 48, 48
    x = torch.from_numpy(synth.normal((B, Ci, H, W), 0).astype(np.float32)).to(dev)
    w = torch.from_numpy(synth.kaiming_uniform((Co, Ci, 19), 1).astype(np.float32)).to(dev)
    Ho, Wo, _ = F.output_shape(H, W, 2)
    y = torch.empty(B, Co, Ho, Wo, device=dev)
    F.conv2d_fwd(x, w, None, n=2, stride=2, out=y)
    gy = torch.from_numpy(synth.normal((B, Co, Ho, Wo), 2).astype(np.float32)).to(dev)
    pyv, am = F.pool2d_fwd(y, n=1, stride=2, mode="max")
    gp = torch.randn_like(pyv)
    dx = torch.empty_like(x)
    dw = torch.empty(Co, Ci, 19, device=dev)
    db = torch.empty(Co, device=dev)
    dyp = torch.empty_like(y)
    fl_c2 = 2.0 * B * vt(H, W, 2, 2) * Ci * Co
    xb, yb, wb = x.numel() * 4, y.numel() * 4, w.numel() * 4
    pb_in, pb_out = y.numel() * 4, pyv.numel() * 4
    c2 = {}
    for name, fn, f, nb in (
            ("conv_fwd", lambda: F.conv2d_fwd(x, w, None, n=2, stride=2, out=y), fl_c2, xb + wb + yb),
            ("conv_dgrad", lambda: F.conv2d_bwd_data(gy, w, (H, W), n=2, stride=2, out=dx), fl_c2, yb + wb + xb),
            ("conv_wgrad", lambda: F.conv2d_bwd_weight(x, gy, n=2, stride=2, dw=dw, dbias=db), fl_c2, xb + yb + wb),
            ("pool_fwd", lambda: F.pool2d_fwd(y, n=1, stride=2, mode="max"), None, pb_in + pb_out + pyv.numel()),
            ("pool_bwd", lambda: F.pool2d_bwd(gp, am, (Ho, Wo), n=1, stride=2, mode="max", out=dyp), None,
             pb_out + pyv.numel() + pb_in)):
        hot, fl = gt.time(gt.capture(fn))
        c2[name] = _pass_entry(hot, fl, f, nb, ffma, peak_gbs)
    out["c2_16to32_48x48_f32"] = c2

    # ---- C3: 256 camera images 40 x 40, fp32 4-layer net (conv 1->16 n1, conv 16->32 n2, avg pool n1 s2,
    # conv 32->64 n1, ReLU), forward + backward, every elementwise step in library kernels
    c = synth.CONFIGS["c3"]
    B, H, W = c["B"], c["H"], c["W"]
    H2, W2, _ = F.output_shape(H, W, 2)
    x = torch.from_numpy(synth.shower_images(B, H, W, c["R"], 3).astype(np.float32)).to(dev)
    convs = [(1, 16, 1), (16, 32, 2), (32, 64, 1)]
    ws = [torch.from_numpy(synth.kaiming_uniform((co, ci, F.num_taps(n)), 20 + i).astype(np.float32)).to(dev)
          for i, (ci, co, n) in enumerate(convs)]
    bs = [torch.zeros(co, device=dev) for _, co, _ in convs]
    t = {k: torch.empty(shape, device=dev) for k, shape in (
        ("y1", (B, 16, H, W)), ("y2", (B, 32, H, W)), ("p", (B, 32, H2, W2)), ("y4", (B, 64, H2, W2)),
        ("dy4", (B, 64, H2, W2)), ("dp", (B, 32, H2, W2)), ("dy2u", (B, 32, H, W)), ("dy2", (B, 32, H, W)),
        ("dy1", (B, 16, H, W)))}
    g4 = torch.from_numpy(synth.normal((B, 64, H2, W2), 4).astype(np.float32)).to(dev)
    dws = [(torch.empty(co, ci, F.num_taps(n), device=dev), torch.empty(co, device=dev)) for ci, co, n in convs]

    def relu_bwd(dyv, yv, outv):
        from paper_1903_01814_b200 import _abi as A_
        A_.check(A_.lib().hex_relu_bwd(dyv.numel(), A_.F32, F._ptr(dyv), F._ptr(yv), F._ptr(outv), F._stream()),
                 "relu_bwd")

    passes = [
        ("L1 fwd", lambda: F.conv2d_fwd(x, ws[0], bs[0], n=1, relu=True, out=t["y1"])),
        ("L2 fwd", lambda: F.conv2d_fwd(t["y1"], ws[1], bs[1], n=2, relu=True, out=t["y2"])),
        ("pool fwd", lambda: F.pool2d_fwd(t["y2"], n=1, stride=2, mode="avg", out=t["p"])),
        ("L4 fwd", lambda: F.conv2d_fwd(t["p"], ws[2], bs[2], n=1, relu=True, out=t["y4"])),
        ("L4 relu bwd", lambda: relu_bwd(g4, t["y4"], t["dy4"])),
        ("L4 wgrad", lambda: F.conv2d_bwd_weight(t["p"], t["dy4"], n=1, dw=dws[2][0], dbias=dws[2][1])),
        ("L4 dgrad", lambda: F.conv2d_bwd_data(t["dy4"], ws[2], (H2, W2), n=1, out=t["dp"])),
        ("pool bwd + L2 relu bwd", lambda: F.pool2d_bwd(t["dp"], None, (H, W), n=1, stride=2, mode="avg",
                                                         out=t["dy2"], relu_y=t["y2"])),
        ("L2 wgrad", lambda: F.conv2d_bwd_weight(t["y1"], t["dy2"], n=2, dw=dws[1][0], dbias=dws[1][1])),
        ("L2 dgrad", lambda: F.conv2d_bwd_data(t["dy2"], ws[1], (H, W), n=2, relu_y=t["y1"], out=t["dy1"])),
        ("L1 wgrad", lambda: F.conv2d_bwd_weight(x, t["dy1"], n=1, dw=dws[0][0], dbias=dws[0][1])),
    ]
    vt1, vt2, vt4 = vt(H, W, 1), vt(H, W, 2), vt(H2, W2, 1)
    px, px2 = B * H * W, B * H2 * W2
    acct = {  # (FLOPs, bytes) per pass
        "L1 fwd": (2.0 * B * vt1 * 16, px * 4 * (1 + 16)),
        "L2 fwd": (2.0 * B * vt2 * 16 * 32, px * 4 * (16 + 32)),
        "pool fwd": (None, px * 32 * 4 + px2 * 32 * 4),
        "L4 fwd": (2.0 * B * vt4 * 32 * 64, px2 * 4 * (32 + 64)),
        "L4 relu bwd": (None, px2 * 64 * 4 * 3),
        "L4 wgrad": (2.0 * B * vt4 * 32 * 64, px2 * 4 * (32 + 64)),
        "L4 dgrad": (2.0 * B * vt4 * 32 * 64, px2 * 4 * (32 + 64)),
        "pool bwd + L2 relu bwd": (None, px2 * 32 * 4 + px * 32 * 4 * 2),
        "L2 wgrad": (2.0 * B * vt2 * 16 * 32, px * 4 * (16 + 32)),
        "L2 dgrad": (2.0 * B * vt2 * 16 * 32, px * 4 * (32 + 16 + 16)),
        "L1 wgrad": (2.0 * B * vt1 * 16, px * 4 * (1 + 16)),
    }
    c3p = {}
    for name, fn in passes:
        hot, fl = gt.time(gt.capture(fn))
        c3p[name] = _pass_entry(hot, fl, acct[name][0], acct[name][1], ffma, peak_gbs)
    step = gt.capture(lambda: [fn() for _, fn in passes])
    hot, fl = gt.time(step)
    fl_all = sum(v[0] or 0.0 for v in acct.values())
    t_roof = sum(max(b_ / (peak_gbs * 1e9), (f_ or 0.0) / (ffma * 1e12)) for f_, b_ in acct.values())
    out["c3_camera_40x40_f32"] = {
        "images_per_s": B / (fl * 1e-3), "images_per_s_hot": B / (hot * 1e-3),
        "ms_per_fwd_bwd_flushed": fl, "ms_per_fwd_bwd_hot": hot, "tflops": fl_all / (fl * 1e-3) / 1e12,
        "roofline_ms": t_roof * 1e3, "frac_of_roofline": t_roof / (fl * 1e-3), "frac_of_roofline_hot": t_roof / (hot * 1e-3),
        "passes": c3p,
        "note": "whole fwd+bwd = one CUDA graph of the 11 library calls; per-pass entries are each pass's own graph "
                "(flushed = L2 evicted before the pass, hot = back-to-back replays)"}

    # ---- C4: 128 x 256 -> 256, 64 x 64, bf16, n = 1 and 2: fwd / dgrad / wgrad (268 MB tensors > L2)
    B, C, H, W = 128, 256, 64, 64
    x = torch.randn(B, H, W, C, device=dev).to(torch.bfloat16)
    gq = torch.randn(B, H, W, C, device=dev).to(torch.bfloat16)
    yq = torch.empty_like(x)
    dxq = torch.empty_like(x)
    c4 = {}
    for n in (1, 2):
        T = F.num_taps(n)
        w = (torch.randn(C, C, T, device=dev) / (C * T) ** 0.5).to(torch.bfloat16)
        dwq, dbq = torch.empty(C, C, T, device=dev), torch.empty(C, device=dev)
        fl4 = 2.0 * B * vt(H, W, n) * C * C
        for name, fn in (("fwd", lambda: F.conv2d_fwd(x, w, None, n=n, layout="NHWC", out=yq)),
                         ("dgrad", lambda: F.conv2d_bwd_data(gq, w, (H, W), n=n, layout="NHWC", out=dxq)),
                         ("wgrad", lambda: F.conv2d_bwd_weight(x, gq, n=n, layout="NHWC", dw=dwq, dbias=dbq))):
            hot, fl = gt.time(gt.capture(fn), 10)
            tf = fl4 / (fl * 1e-3) / 1e12
            c4[f"n{n}_{name}"] = {"us_flushed": fl * 1e3, "us_hot": hot * 1e3, "tflops": tf,
                                  "frac_of_bf16_peak": tf / peak_tf}
    out["c4_256x256_64x64_bf16"] = c4
    del x, gq, yq, dxq

    # ---- f2: 3-D hex conv (hex x-y, equidistant z), bf16 NDHWC.
    # Synthetic shape (no paper workload): 16 volumes x 16 slices x 64x64, 64 -> 128 channels, n = 1, kd = 3.
    B, D, H, W, C, Co, kd, n = 16, 16, 64, 64, 64, 128, 3, 1
    T = F.num_taps(n)
    x = torch.randn(B, D, H, W, C, device=dev).to(torch.bfloat16)
    g3 = torch.randn(B, D, H, W, Co, device=dev).to(torch.bfloat16)
    w = (torch.randn(Co, C, kd, T, device=dev) / (C * kd * T) ** 0.5).to(torch.bfloat16)
    fl3 = 2.0 * B * vt(H, W, n) * (kd * D - 2) * C * Co
    c3d = {}
    for name, fn in (("fwd", lambda: F.conv3d_fwd(x, w, None, n=n, layout="NDHWC")),
                     ("dgrad", lambda: F.conv3d_bwd_data(g3, w, (D, H, W), n=n, layout="NDHWC")),
                     ("wgrad", lambda: F.conv3d_bwd_weight(x, g3, kd, n=n, layout="NDHWC"))):
        hot, fl = gt.time(gt.capture(fn), 10)
        tf = fl3 / (fl * 1e-3) / 1e12
        c3d[name] = {"us_flushed": fl * 1e3, "us_hot": hot * 1e3, "tflops": tf, "frac_of_bf16_peak": tf / peak_tf}
    c3d["note"] = ("fwd / dgrad: depth taps inside the K loop of the tcgen05 tap-reuse kernel (out-of-volume "
                   "slices are zero-fill boxes); wgrad: depth taps as channel-chunk units of the tcgen05 tap-reuse "
                   "weight gradient (no unfolded copy); FLOPs count in-range depth taps only")
    out["conv3d_64to128_16x64x64_kd3_bf16"] = c3d
    del x, g3

    # ---- f4: strided layers on the tensor cores (forward by element-stride-s boxes, bwd-data by phase classes,
    # weight gradient on the lattice), bf16 NHWC 64 images 96x96 -> 48x48 (s = 2) / 32x32 (s = 3), 128 -> 128,
    # n = 1 and 2.  Synthetic shape; FLOPs of the in-grid (lattice) taps only.
    B, H, W, C = 64, 96, 96, 128
    x = torch.randn(B, H, W, C, device=dev).to(torch.bfloat16)
    dx2 = torch.empty_like(x)
    for s in (2, 3):
        Ho, Wo, _ = F.output_shape(H, W, s)
        g2 = torch.randn(B, Ho, Wo, C, device=dev).to(torch.bfloat16)
        y2 = torch.empty_like(g2)
        dw2 = {}
        ent = {}
        for n in (1, 2):
            T = F.num_taps(n)
            w = (torch.randn(C, C, T, device=dev) / (C * T) ** 0.5).to(torch.bfloat16)
            dw2[n] = torch.empty(C, C, T, device=dev)
            fl2 = 2.0 * B * vt(H, W, n, s) * C * C  # in-grid taps of the lattice outputs
            for name, fn in (("fwd", lambda w=w, s=s, n=n, g2=g2, y2=y2:
                              F.conv2d_fwd(x, w, None, n=n, stride=s, layout="NHWC", out=y2)),
                             ("dgrad", lambda w=w, s=s, n=n, g2=g2:
                              F.conv2d_bwd_data(g2, w, (H, W), n=n, stride=s, layout="NHWC", out=dx2)),
                             ("wgrad", lambda s=s, n=n, g2=g2:
                              F.conv2d_bwd_weight(x, g2, n=n, stride=s, layout="NHWC", dw=dw2[n]))):
                hot, fl = gt.time(gt.capture(fn), 10)
                tf = fl2 / (fl * 1e-3) / 1e12
                ent[f"n{n}_{name}"] = {"us_flushed": fl * 1e3, "us_hot": hot * 1e3, "tflops": tf,
                                       "frac_of_bf16_peak": tf / peak_tf}
        ent["note"] = (f"bf16 NHWC stride {s}, tcgen05: forward with element-stride-{s} input boxes, bwd-data by "
                       f"phase classes (TMA boxes of dy parity views), weight gradient on the lattice "
                       f"(element-stride-{s} x boxes); FLOPs of the in-grid taps of the lattice outputs")
        out[f"stride{s}_128to128_96x96_bf16"] = ent
    return out


# ------------------------------------------------------------------ launcher
def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch_under_torchrun(n: int) -> int:
    """Re-run this script as n ranks under torch.distributed.run (nnodes 1, 127.0.0.1); the ranks see
    WORLD_SIZE = n and take the normal path.  Returns torchrun's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config 2-4 measurements")
    ap.add_argument("--sustain-s", type=float, default=2.5,
                    help="seconds of back-to-back steps for the sustained (power-capped) rate; 0 = skip")
    ap.add_argument("--launch-check", action="store_true",
                    help="print each rank's (rank, world) and exit before touching a GPU (launcher test)")
    ap.add_argument("--no-graph", action="store_true", help="device-timed and e2e legs as eager steps (no CUDA graph)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        # the oracle arm runs on rank 0's host cores only; the other ranks (under torchrun) exit 0
        run_reference(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start the N ranks here (one per GPU, torchrun on
        # 127.0.0.1) and pass their exit status through, so a multi-GPU request never quietly becomes a
        # one-rank line
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.launch_check:
        print(json.dumps({"rank": rank, "world": world, "local_rank": local}), flush=True)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_1903_01814_b200 import _abi
    from paper_1903_01814_b200.hexcnn import HexCNN

    B = args.batch
    model = HexCNN(batch=B, device=dev, seed=0)
    NB = 4
    xs_np, ys_np = make_batches(NB, B, 96, 96, 47, seed=1000 + 17 * rank)
    xs = [torch.from_numpy(a).to(dev).to(torch.bfloat16) for a in xs_np]
    ys = [torch.from_numpy(a).to(dev) for a in ys_np]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # warm-up
    for i in range(args.warmup):
        model.step(xs[i % NB], ys[i % NB])
    torch.cuda.synchronize()

    def capture(xb, yb):
        """HexCNN.graphed_step on every rank (the per-layer NCCL allreduces are captured too); if any
        rank fails to capture, every rank falls back to eager steps so the collectives stay matched."""
        if args.no_graph:
            return None, None
        try:
            g, loss = model.graphed_step(xb, yb)
            ok = 1.0
        except Exception as ex:  # reported in the line as cuda_graph: false
            print(f"bench.py: CUDA-graph capture failed, eager steps: {ex!r}", file=sys.stderr)
            g, loss, ok = None, None, 0.0
        torch.cuda.synchronize()
        if world > 1:
            t = torch.tensor([ok], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            if t.item() < 1.0:
                return None, None
        return g, loss

    # ---- device-resident timed region: each step is one CUDA-graph replay of the whole step
    # (HexCNN.graphed_step: every kernel, the per-layer NCCL gradient allreduces when N > 1, and SGD;
    # the batch is copied device -> device into the graph's static input buffer, 4.7 MB)
    xg, yg = torch.empty_like(xs[0]), torch.empty_like(ys[0])
    xg.copy_(xs[0])
    yg.copy_(ys[0])
    graph_v, _ = capture(xg, yg)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    clocks.mark()
    l0 = _abi.launch_count()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record()
    for i in range(args.steps):
        if graph_v is not None:
            xg.copy_(xs[i % NB], non_blocking=True)
            yg.copy_(ys[i % NB], non_blocking=True)
            graph_v.replay()
        else:
            model.step(xs[i % NB], ys[i % NB])
    t_end.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    value = world * B * args.steps / (ms / 1e3)

    # ---- sustained rate: the same replayed step looped for >= --sustain-s seconds (power-capped steady
    # state), reported beside the K-step value against the driver's sustained bf16 figure
    sustained = None
    if args.sustain_s > 0:
        n_s = max(1, int(args.sustain_s / (ms_step / 1e3)))
        sclk = ClockSampler(local)
        sclk.start()
        barrier()
        torch.cuda.synchronize()
        sclk.mark()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for i in range(n_s):
            if graph_v is not None:
                xg.copy_(xs[i % NB], non_blocking=True)
                yg.copy_(ys[i % NB], non_blocking=True)
                graph_v.replay()
            else:
                model.step(xs[i % NB], ys[i % NB])
        s1.record()
        torch.cuda.synchronize()
        barrier()
        sc = sclk.stop()
        s_ms = max_over_ranks(s0.elapsed_time(s1))
        flops_img_, _ = model.flops_per_image()
        sustained = {"images_per_s": world * B * n_s / (s_ms / 1e3), "steps": n_s, "seconds": s_ms / 1e3,
                     "ms_per_step": s_ms / n_s,
                     "step_tflops_per_gpu": flops_img_ * B * n_s / (s_ms / 1e3) / 1e12, "clocks": sc}

    # ---- per kernel family: CUDA events recorded around every conv / pool call (on the stream it is
    # launched on) over K eager steps of the same workload; launches counted by the library
    model.timer = []
    barrier()
    torch.cuda.synchronize()
    l0 = _abi.launch_count()
    for i in range(args.steps):
        model.step(xs[i % NB], ys[i % NB])
    torch.cuda.synchronize()
    barrier()
    launches = _abi.launch_count() - l0
    events = model.timer
    model.timer = None

    # per kernel family, from CUDA events recorded around every call inside the timed region
    flops_img, per_layer = model.flops_per_image()
    fam = {}  # name -> [ms, algorithmic units, unit, launches]

    def add(name, ms_, units, unit):
        f = fam.setdefault(name, [0.0, 0.0, unit, 0])
        f[0] += ms_
        f[1] += units
        f[3] += 1

    share = {}
    for kind, l, e0, e1 in events:
        dt = e0.elapsed_time(e1)
        share[kind] = share.get(kind, 0.0) + dt
        if kind in ("fwd", "dgrad", "wgrad"):
            fl = per_layer[l][0] * B
            if l == 0:  # Cin = 1: warp-level tensor-core kernels bound by the y / dy stream (HBM bytes)
                add("smallc_mma (layer 1 fwd + wgrad, mma.sync, HBM-bound)", dt, model.l1_bytes(kind), "GB/s")
            elif kind == "wgrad":
                add("tc_conv_wgrad (tcgen05, layers 2-6)", dt, fl, "TFLOP/s")
            else:
                add("tc_conv_fwd (tcgen05 fwd + bwd-data, layers 2-6)", dt, fl, "TFLOP/s")
        elif kind == "fwd_pool":  # fused conv + ReLU + max pool: the conv's algorithmic FLOPs (no halo recompute)
            add("tc_conv_maxpool (fused conv+ReLU+maxpool, tcgen05)", dt, per_layer[l][0] * B, "TFLOP/s")
        else:
            add("pool (max n1 s2 fwd + bwd)", dt, model.pool_bytes(l, kind), "GB/s")
    peaks, peak_src = load_peaks()
    # the contract's ceiling for a kernel timed inside a long step is the driver's SUSTAINED figure; the
    # tcgen05 families measure above it in-step, so the burst figure (the higher one) is reported instead
    peak_tf = max(peaks.get("bf16_tflops_sustained", 0.0), peaks["bf16_tflops"])
    peak_gbs = peaks["hbm_gbs"]
    kernels = {}
    for name, (fms, units, unit, n) in fam.items():
        ach = units / (fms / 1e3) / (1e12 if unit == "TFLOP/s" else 1e9)
        pk = peak_gbs if unit == "GB/s" else peak_tf
        kernels[name] = {"ms_per_step": fms / args.steps, "achieved": ach, "unit": unit, "peak": pk,
                         "frac": ach / pk, "launches_per_step": n / args.steps}
    dom = max(fam, key=lambda k: fam[k][0])
    tc_name = "tc_conv_fwd (tcgen05 fwd + bwd-data, layers 2-6)"
    achieved = kernels[tc_name]["achieved"]
    total_tf = flops_img * B / (ms_step / 1e3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "tc_fwd_traffic.json")) as f:
            traffic = json.load(f).get("bytes_per_launch")
    except Exception:
        pass

    # ---- end-to-end through the public API with host buffers: each step copies its batch from pinned
    # host memory into the model's input buffers, runs the step (one CUDA-graph replay of
    # HexCNN.graphed_step) and reads the loss back
    pin_x = [torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).pin_memory() for a in xs_np]
    pin_y = [torch.from_numpy(a).pin_memory() for a in ys_np]
    xd = torch.empty_like(xs[0])
    yd = torch.empty_like(ys[0])
    loss_h = torch.empty(1, dtype=torch.float32).pin_memory()
    xd.copy_(xs[0])
    yd.copy_(ys[0])
    graph, gloss = capture(xd, yd)
    # Input pipeline: the H2D copy of batch i+1 (pinned host -> device staging buffer, copy stream)
    # overlaps step i; step i starts with a 4.7 MB device copy staging -> model input.  The loss of
    # step i is copied to pinned host memory and read (host sync on its event) after step i+1 has
    # been issued, so the host turnaround does not idle the GPU.  Every step's H2D copy and D2H
    # read happen inside the timed region.
    main = torch.cuda.current_stream()
    cstream = torch.cuda.Stream()
    stage_x = [torch.empty_like(xs[0]) for _ in range(2)]
    stage_y = [torch.empty_like(ys[0]) for _ in range(2)]
    loaded = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    loss_hs = [torch.empty(1, dtype=torch.float32).pin_memory() for _ in range(2)]
    got = [torch.cuda.Event() for _ in range(2)]
    losses = []

    def h2d(i):
        k = i % 2
        with torch.cuda.stream(cstream):
            if i >= 2:
                cstream.wait_event(freed[k])  # step i-2 consumed this staging buffer
            stage_x[k].copy_(pin_x[i % NB], non_blocking=True)
            stage_y[k].copy_(pin_y[i % NB], non_blocking=True)
            loaded[k].record(cstream)

    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h2d(0)
    for i in range(args.steps):
        k = i % 2
        main.wait_event(loaded[k])
        xd.copy_(stage_x[k], non_blocking=True)
        yd.copy_(stage_y[k], non_blocking=True)
        freed[k].record(main)
        if i + 1 < args.steps:
            h2d(i + 1)
        if graph is not None:
            graph.replay()
            loss = gloss
        else:
            loss = model.step(xd, yd)
        loss_hs[k].copy_(loss, non_blocking=True)
        got[k].record(main)
        if i >= 1:  # read step i-1's loss now that step i is queued
            got[(i - 1) % 2].synchronize()
            losses.append(float(loss_hs[(i - 1) % 2][0]))
    got[(args.steps - 1) % 2].synchronize()
    losses.append(float(loss_hs[(args.steps - 1) % 2][0]))
    e1.record()
    torch.cuda.synchronize()
    barrier()
    assert len(losses) == args.steps
    if os.environ.get("HEXBENCH_PRINT_LOSS"):
        print("e2e losses:", losses, file=sys.stderr)
    loss_info = {"last": losses[-1], "all_finite": all(math.isfinite(v) for v in losses)}
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = world * B * args.steps / (e2e_ms / 1e3)
    h2d = pin_x[0].numel() * pin_x[0].element_size() + pin_y[0].numel() * pin_y[0].element_size()

    # ---- secondary configs (rank 0, N = 1 only; not part of the timed step)
    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary:
        try:
            peaks_, _ = load_peaks()
            secondary = secondary_measurements(dev, peaks_["bf16_tflops"], peaks_["hbm_gbs"])
        except Exception as ex:  # a failure here must not hide the headline line
            secondary = {"error": repr(ex)}

    # ---- oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        threads_all = oracle.max_threads()
        dt, threads = oracle_train_sample(1)
        oracle.set_threads(1)
        dt1, _ = oracle_train_sample(1)
        oracle.set_threads(threads_all)
        cpu = {"value": 1.0 / dt, "unit": "images/s", "cores": threads, "kind": "oracle",
               "single_thread_value": 1.0 / dt1, "cpu_model": cpu_model(),
               "sample": "1 image through the full C5 fwd+bwd+SGD step in fp64 (bounded sample of the "
                         "256-image batch), all host cores and one thread"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": B * world, "per_gpu_batch": B, "grid": "96x96",
                       "parallelism": f"dp{world}", "l2": "working set > L2 (activations ~2.5 GB/step)",
                       "cuda_graph": graph_v is not None},
            "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4,
                    "loss": loss_info,
                    "cuda_graph": graph is not None},
            "roofline": {"bound": "tensor", "kernel": "tc_fwd_vpair_kernel (layer-2 bwd-data) / tc_fwd_tr_kernel "
                                                      "(layers 3-4) / tc_conv_fwd2_kernel (layers 5-6): tcgen05 "
                                                      "implicit-GEMM hex conv, fwd + bwd-data",
                         "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic,
                         "peak_source": f"{peak_src} bf16_tflops (burst): the in-step achieved rate exceeds the "
                                        f"sustained figure {peaks.get('bf16_tflops_sustained')}, so the higher "
                                        "measured peak is the ceiling",
                         "launches_per_step": kernels[tc_name]["launches_per_step"],
                         "dominant_by_time": dom == tc_name},
            "kernels": kernels,
            "step_tflops": total_tf,
            "sustained": dict(sustained, bf16_tflops_sustained_peak=peaks.get("bf16_tflops_sustained"),
                              frac_of_sustained_peak=sustained["step_tflops_per_gpu"] / peaks["bf16_tflops_sustained"]
                              if peaks.get("bf16_tflops_sustained") else None) if sustained else None,
            "step_share_ms": {k: v / args.steps for k, v in share.items()},
            "secondary_configs": secondary,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
