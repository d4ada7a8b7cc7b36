"""torch.nn modules over the autograd wrappers of functional.py -- "By adopting the PyTorch-API, these
operations can easily be incorporated in CNN models defined in PyTorch" (Sec. 2
"Software Functionalities").  Every forward / backward runs in libhexconv.

    HexConv2d(in_channels, out_channels, kernel_size, stride=1, bias=True, debug=False, ...)
    HexConv3d(in_channels, out_channels, kernel_size, kernel_depth, stride=1, depth_stride=1, ...)
    HexMaxPool2d(kernel_size, stride=1, ...), HexAvgPool2d(kernel_size, stride=1, count_include_pad=False, ...)

kernel_size is the paper's n (T(n) = 3n(n+1)+1 taps).  Weights are stored as
[Cout][Cin][T] in canonical tap order (A2) -- a custom kernel is set by writing that tensor
(functional.custom_kernel / ring_kernel build one).  debug=True sets every kernel element to 1 and the bias
to 0 ("Enabling the debug mode sets all kernel elements to 1").  Initialisation:
He-uniform U(+-sqrt(6 / fan_in)) with fan_in = Cin * T (* kd) (A19), bias 0.
"""
from __future__ import annotations

import math

import torch

from . import functional as F


class HexConv2d(torch.nn.Module):
    def __init__(self, in_channels: int, out_channels: int, kernel_size: int = 1, stride: int = 1,
                 bias: bool = True, debug: bool = False, parity: int = 0, relu: bool = False, layout: str = "NCHW",
                 dtype=torch.float32, device=None):
        super().__init__()
        if kernel_size < 0 or stride < 1:
            raise ValueError("kernel_size >= 0 and stride >= 1 required")
        self.in_channels, self.out_channels = in_channels, out_channels
        self.kernel_size, self.stride, self.parity, self.relu, self.layout = kernel_size, stride, parity, relu, layout
        T = F.num_taps(kernel_size)
        self.weight = torch.nn.Parameter(torch.empty(out_channels, in_channels, T, dtype=dtype, device=device))
        # the library takes an fp32 bias for every dtype
        self.bias = torch.nn.Parameter(torch.zeros(out_channels, dtype=torch.float32, device=device)) if bias else None
        self.debug = debug
        self.reset_parameters()

    def reset_parameters(self):
        with torch.no_grad():
            if self.debug:
                self.weight.fill_(1.0)
            else:
                lim = math.sqrt(6.0 / (self.in_channels * self.weight.shape[-1]))
                self.weight.uniform_(-lim, lim)
            if self.bias is not None:
                self.bias.zero_()

    def forward(self, x):
        return F.hex_conv2d(x, self.weight, self.bias, self.kernel_size, self.stride, self.parity, self.relu,
                            self.layout)

    def extra_repr(self):
        return (f"{self.in_channels}, {self.out_channels}, kernel_size={self.kernel_size}, stride={self.stride}, "
                f"parity={self.parity}, relu={self.relu}, layout={self.layout}, debug={self.debug}")


class HexConv3d(torch.nn.Module):
    def __init__(self, in_channels: int, out_channels: int, kernel_size: int = 1, kernel_depth: int = 1,
                 stride: int = 1, depth_stride: int = 1, bias: bool = True, debug: bool = False, parity: int = 0,
                 layout: str = "NCDHW", dtype=torch.float32, device=None):
        super().__init__()
        if kernel_size < 0 or stride < 1 or depth_stride < 1 or kernel_depth < 1 or kernel_depth % 2 == 0:
            raise ValueError("kernel_size >= 0, odd kernel_depth >= 1, strides >= 1 required")
        self.in_channels, self.out_channels = in_channels, out_channels
        self.kernel_size, self.kernel_depth = kernel_size, kernel_depth
        self.stride, self.depth_stride, self.parity, self.layout = stride, depth_stride, parity, layout
        T = F.num_taps(kernel_size)
        self.weight = torch.nn.Parameter(torch.empty(out_channels, in_channels, kernel_depth, T, dtype=dtype,
                                                     device=device))
        self.bias = torch.nn.Parameter(torch.zeros(out_channels, dtype=torch.float32, device=device)) if bias else None
        self.debug = debug
        self.reset_parameters()

    def reset_parameters(self):
        with torch.no_grad():
            if self.debug:
                self.weight.fill_(1.0)
            else:
                fan_in = self.in_channels * self.kernel_depth * self.weight.shape[-1]
                lim = math.sqrt(6.0 / fan_in)
                self.weight.uniform_(-lim, lim)
            if self.bias is not None:
                self.bias.zero_()

    def forward(self, x):
        return F.hex_conv3d(x, self.weight, self.bias, self.kernel_size, self.stride, self.depth_stride,
                            self.parity, self.layout)


class _HexPool2d(torch.nn.Module):
    mode = "max"

    def __init__(self, kernel_size: int = 1, stride: int = 1, parity: int = 0, layout: str = "NCHW"):
        super().__init__()
        if kernel_size < 1 or stride < 1:
            raise ValueError("pooling needs kernel_size >= 1 and stride >= 1")
        self.kernel_size, self.stride, self.parity, self.layout = kernel_size, stride, parity, layout

    def extra_repr(self):
        return f"kernel_size={self.kernel_size}, stride={self.stride}, parity={self.parity}, layout={self.layout}"


class HexMaxPool2d(_HexPool2d):
    """Max over the in-grid cells of the size-n hexagonal window (first strict maximum in canonical order,
    DESIGN.md A8/A9)."""

    def forward(self, x):
        return F.hex_max_pool2d(x, self.kernel_size, self.stride, self.parity, self.layout)


class HexAvgPool2d(_HexPool2d):
    """Mean over the in-grid cells of the window (count_include_pad=True: over all T(n) taps, off-grid = 0)."""

    def __init__(self, kernel_size: int = 1, stride: int = 1, parity: int = 0, layout: str = "NCHW",
                 count_include_pad: bool = False):
        super().__init__(kernel_size, stride, parity, layout)
        self.count_include_pad = count_include_pad

    def forward(self, x):
        return F.hex_avg_pool2d(x, self.kernel_size, self.stride, self.parity, self.layout, self.count_include_pad)
