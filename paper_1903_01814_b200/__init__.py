"""paper_1903_01814_b200 -- B200-native hexagonal convolution and pooling
(HexagDLy, arXiv 1903.01814) over a C-ABI CUDA library (libhexconv.so).

The hot path (hex conv fwd / bwd-data / bwd-weight, hex max/avg pool fwd/bwd)
runs in hand-written sm_100a kernels behind include/hexconv.h; this package
is the thin Python binding.  Importing it without the built library raises:
there is no CPU fallback.
"""
from . import _abi  # noqa: F401  (raises ImportError if libhexconv.so is missing)
from . import nn  # noqa: F401  (torch.nn modules: HexConv2d, HexConv3d, HexMaxPool2d, HexAvgPool2d)
from .functional import (  # noqa: F401
    conv2d_bwd_data,
    conv2d_bwd_weight,
    conv2d_fwd,
    gather_map,
    hex_avg_pool2d,
    hex_conv2d,
    hex_max_pool2d,
    num_taps,
    output_shape,
    pool2d_bwd,
    pool2d_fwd,
)

__version__ = "0.1.0"
