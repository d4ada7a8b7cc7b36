"""Seeded synthetic inputs shared by tests/ and bench.py (both the CUDA path and
the oracle consume the same buffers).  Holds none of the method's arithmetic:
only random draws, rounding to the storage dtype, and the BASELINE.json
workload shapes.  (Reading A18 in DESIGN.md fixes the shower recipe.)

Camera images (configs 3 and 5) place an elliptical 2-D Gaussian "shower"
plus Poisson night-sky noise on the pixels of a hexagonal camera (a hex disc
of radius R around the grid centre); all other tensor cells are 0.  The pixel
positions come from the addressing description: column c
at x = c*sqrt(3)/2, row r at y = -(r + 0.5*((c+pi) mod 2)).
"""
from __future__ import annotations

import math

import numpy as np

# BASELINE.json configs[0..4] as concrete workload descriptions
CONFIGS = {
    "c1": dict(B=4, Cin=1, Cout=4, H=16, W=16, n=1, s=1, dtype="f32"),
    "c2": dict(B=32, Cin=16, Cout=32, H=48, W=48, n=2, s=2, pool_n=1, pool_s=2, dtype="f32"),
    "c3": dict(B=256, H=40, W=40, R=18, dtype="f32",
               layers=[("conv", 1, 16, 1, 1), ("conv", 16, 32, 2, 1), ("avgpool", 32, 32, 1, 2),
                       ("conv", 32, 64, 1, 1)]),
    "c4": dict(B=128, Cin=256, Cout=256, H=64, W=64, ns=(1, 2), s=1, dtype="bf16"),
    "c5": dict(B=256, H=96, W=96, R=47, K=2, dtype="bf16",
               channels=[1, 64, 128, 128, 256, 256, 256], ns=[2, 1, 2, 1, 2, 1], pool_after=(2, 4)),
}


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def normal(shape, seed: int, std: float = 1.0) -> np.ndarray:
    return rng(seed).standard_normal(shape) * std


def uniform(shape, seed: int, lo: float, hi: float) -> np.ndarray:
    return rng(seed).uniform(lo, hi, size=shape)


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round to bf16 (RNE) and return the rounded values as float64."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def round_f32(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def pixel_xy(H: int, W: int, pi: int = 0):
    c = np.arange(W)[None, :].repeat(H, 0)
    r = np.arange(H)[:, None].repeat(W, 1)
    x = c * (math.sqrt(3) / 2)
    y = -(r + 0.5 * ((c + pi) % 2))
    return x, y


def camera_mask(H: int, W: int, R: int, pi: int = 0) -> np.ndarray:
    """Hexagonal camera: all pixels within hex distance R of the centre pixel
    (H//2, W//2).  Distances on the triangular lattice from pixel positions."""
    x, y = pixel_xy(H, W, pi)
    xc, yc = x[H // 2, W // 2], y[H // 2, W // 2]
    # hex distance of a lattice vector (dx, dy): project on the three axes
    dx, dy = x - xc, y - yc
    a = dx / (math.sqrt(3) / 2)            # diagonal-axis steps (q)
    b = -dy - a / 2                        # vertical-axis steps (r)
    q, r = np.rint(a), np.rint(b)
    d = (np.abs(q) + np.abs(r) + np.abs(q + r)) / 2
    return d <= R


def shower_images(B: int, H: int, W: int, R: int, seed: int, pi: int = 0) -> np.ndarray:
    """float32 [B, 1, H, W] synthetic Cherenkov-camera images (BASELINE config 3/5)."""
    g = rng(seed)
    mask = camera_mask(H, W, R, pi)
    x, y = pixel_xy(H, W, pi)
    xc, yc = x[H // 2, W // 2], y[H // 2, W // 2]
    inner = camera_mask(H, W, max(R - 3, 0), pi)
    cand = np.argwhere(inner)
    out = np.zeros((B, 1, H, W), dtype=np.float32)
    for b in range(B):
        rr, cc = cand[g.integers(0, len(cand))]
        x0, y0 = x[rr, cc], y[rr, cc]
        sl = g.uniform(2.0, 8.0)
        sw = g.uniform(0.5, 2.0)
        th = g.uniform(0.0, math.pi)
        amp = math.exp(g.uniform(math.log(50.0), math.log(5000.0)))
        u = (x - x0) * math.cos(th) + (y - y0) * math.sin(th)
        v = -(x - x0) * math.sin(th) + (y - y0) * math.cos(th)
        img = amp * np.exp(-0.5 * (u * u / (sl * sl) + v * v / (sw * sw)))
        img = img + g.poisson(3.0, size=(H, W))
        out[b, 0] = np.where(mask, img, 0.0)
    _ = (xc, yc)
    return out


def labels(B: int, seed: int) -> np.ndarray:
    return rng(seed).integers(0, 2, size=(B,)).astype(np.int32)


def kaiming_uniform(shape, seed: int) -> np.ndarray:
    """C2 weights: U(+-sqrt(6/fan_in)), fan_in = Cin*T (reading A19)."""
    fan_in = shape[1] * shape[2]
    lim = math.sqrt(6.0 / fan_in)
    return uniform(shape, seed, -lim, lim)
