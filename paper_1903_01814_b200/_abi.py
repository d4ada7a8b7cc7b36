"""ctypes binding of include/hexconv.h (libhexconv.so).

Argument marshalling only: every entry point forwards device pointers, sizes
and the current CUDA stream to the C ABI; all tensor arithmetic runs in the
library's sm_100a kernels.  There is no fallback: if the shared library is
missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhexconv.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build the CUDA library first "
        "(python -m paper_1903_01814_b200.build or __graft_entry__.build()). "
        "There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

HEX_OK = 0
STATUS_NAMES = {
    0: "HEX_OK", 1: "HEX_ERR_INVALID_ARG", 2: "HEX_ERR_SHAPE", 3: "HEX_ERR_EMPTY_LATTICE",
    4: "HEX_ERR_DTYPE", 5: "HEX_ERR_LAYOUT", 6: "HEX_ERR_ALIGNMENT", 7: "HEX_ERR_WORKSPACE",
    8: "HEX_ERR_UNSUPPORTED", 9: "HEX_ERR_CUDA",
}
F32, BF16 = 0, 1
NCHW, NHWC = 0, 1
POOL_MAX, POOL_AVG, POOL_AVG_PAD = 0, 1, 2
MAX_N = 7


class HexError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        name = STATUS_NAMES.get(status, str(status))
        msg = _lib.hex_status_string(status).decode()
        super().__init__(f"{where}: {name} ({msg})")


class ConvDesc(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in (
        "batch", "in_channels", "out_channels", "height", "width",
        "kernel_size", "stride", "parity", "dtype", "layout")]


class Conv3dDesc(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in (
        "batch", "in_channels", "out_channels", "depth", "height", "width",
        "kernel_size", "kernel_depth", "stride", "depth_stride", "parity", "dtype", "layout")]


class PoolDesc(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in (
        "batch", "channels", "height", "width", "kernel_size", "stride",
        "parity", "dtype", "layout", "mode")]


_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_f32 = ctypes.c_float
_i32p = ctypes.POINTER(ctypes.c_int32)
_szp = ctypes.POINTER(ctypes.c_size_t)
_CDP = ctypes.POINTER(ConvDesc)
_PDP = ctypes.POINTER(PoolDesc)
_C3P = ctypes.POINTER(Conv3dDesc)

_SIGS = {
    "hex_num_taps": (_i32, [_i32]),
    "hex_version": (_i32, []),
    "hex_debug_set_switch": (_i32, [ctypes.c_char_p, ctypes.c_char_p]),
    "hex_launch_count": (_i64, []),
    "hex_status_string": (ctypes.c_char_p, [_i32]),
    "hex_output_shape": (_i32, [_i32, _i32, _i32, _i32, _i32p, _i32p, _i32p]),
    "hex_tap_offsets": (_i32, [_i32, _i32, _i32p]),
    "hex_tap_axial": (_i32, [_i32, _i32p]),
    "hex_conv2d_gather_map": (_i32, [_CDP, _vp, _vp]),
    "hex_conv2d_workspace_size": (_i32, [_CDP, _i32, _szp]),
    "hex_conv2d_algo": (_i32, [_CDP, _i32, _i32p]),
    "hex_conv2d_fwd": (_i32, [_CDP, _vp, _vp, _vp, _i32, _vp, _vp, _sz, _vp]),
    "hex_conv2d_fwd_maxpool_supported": (_i32, [_CDP]),
    "hex_conv2d_fwd_maxpool": (_i32, [_CDP, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _sz, _vp]),
    "hex_conv2d_fwd_pool_supported": (_i32, [_CDP, _i32]),
    "hex_conv2d_fwd_pool": (_i32, [_CDP, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _sz, _vp]),
    "hex_conv2d_bwd_data": (_i32, [_CDP, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "hex_conv2d_bwd_weight": (_i32, [_CDP, _vp, _vp, _vp, _vp, _i32, _vp, _sz, _vp]),
    "hex_conv2d_pack_weights": (_i32, [_i32, _CDP, _i32p, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _szp, _vp]),
    "hex_conv3d_output_shape": (_i32, [_C3P, _i32p, _i32p, _i32p]),
    "hex_conv3d_workspace_size": (_i32, [_C3P, _i32, _szp]),
    "hex_conv3d_fwd": (_i32, [_C3P, _vp, _vp, _vp, _i32, _vp, _vp, _sz, _vp]),
    "hex_conv3d_bwd_data": (_i32, [_C3P, _vp, _vp, _vp, _vp, _sz, _vp]),
    "hex_conv3d_bwd_weight": (_i32, [_C3P, _vp, _vp, _vp, _vp, _i32, _vp, _sz, _vp]),
    "hex_pool2d_fwd": (_i32, [_PDP, _vp, _vp, _vp, _vp]),
    "hex_pool2d_bwd": (_i32, [_PDP, _vp, _vp, _vp, _vp]),
    "hex_pool2d_bwd_relu": (_i32, [_PDP, _vp, _vp, _vp, _vp, _vp]),
    "hex_head_workspace_size": (_sz, [_i32, _i32, _i32]),
    "hex_head_fwd_bwd": (_i32, [_i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "hex_sgd_momentum": (_i32, [_i64, _vp, _vp, _vp, _f32, _f32, _f32, _vp, _vp]),
    "hex_cast_f32_bf16": (_i32, [_i64, _vp, _vp, _vp]),
    "hex_relu_bwd": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp]),
    "hex_nvls_supported": (_i32, [_i32, _i32p]),
    "hex_nvls_open": (_i32, [_i32, _i32, _i32, _sz, _i32, _i32p, ctypes.POINTER(_vp)]),
    "hex_nvls_open_local": (_i32, [_i32, _sz, ctypes.POINTER(_vp)]),
    "hex_nvls_map": (_i32, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _szp]),
    "hex_nvls_allreduce_f32": (_i32, [_vp, _i64, _i64, _i32, _vp]),
    "hex_nvls_close": (_i32, [_vp]),
    "hex_nvls_plan": (_i32, [_i64, _i32, _i32, _i32, _i32p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


def lib():
    return _lib


def check(status: int, where: str):
    if status != HEX_OK:
        raise HexError(status, where)


def num_taps(n: int) -> int:
    return int(_lib.hex_num_taps(n))


def output_shape(H: int, W: int, stride: int = 1, parity: int = 0):
    """(Ho, Wo, parity_out) of the stride lattice; raises HexError."""
    ho, wo, po = _i32(), _i32(), _i32()
    check(_lib.hex_output_shape(H, W, stride, parity, ctypes.byref(ho), ctypes.byref(wo), ctypes.byref(po)),
          "hex_output_shape")
    return ho.value, wo.value, po.value


def tap_offsets(n: int, p: int):
    T = num_taps(n)
    buf = (_i32 * (2 * max(T, 1)))()
    check(_lib.hex_tap_offsets(n, p, buf), "hex_tap_offsets")
    return [(buf[2 * t], buf[2 * t + 1]) for t in range(T)]


def tap_axial(n: int):
    """The T(n) taps as axial (dq, dr) in canonical order (library geometry)."""
    T = num_taps(n) if n >= 0 else 0
    buf = (_i32 * (2 * max(T, 1)))()
    check(_lib.hex_tap_axial(n, buf), "hex_tap_axial")
    return [(buf[2 * t], buf[2 * t + 1]) for t in range(T)]


class PackArgs:
    """Marshalled argument arrays of hex_conv2d_pack_weights for a fixed set of (desc, pass, weight pointer,
    workspace pointer, workspace bytes) entries -- built once, then `run(stream)` is one library call."""

    def __init__(self, entries):
        n = len(entries)
        self.n = n
        self.descs = (ConvDesc * max(n, 1))(*[e[0] for e in entries])
        self.passes = (_i32 * max(n, 1))(*[e[1] for e in entries])
        self.w = (_vp * max(n, 1))(*[e[2] for e in entries])
        self.ws = (_vp * max(n, 1))(*[e[3] for e in entries])
        self.ws_bytes = (_sz * max(n, 1))(*[e[4] for e in entries])

    def run(self, stream):
        check(lib().hex_conv2d_pack_weights(self.n, self.descs, self.passes, self.w, self.ws, self.ws_bytes, stream),
              "hex_conv2d_pack_weights")


class switch:
    """Context manager for A/B tests: override one HEXCONV_* kernel-selection switch (read from the
    environment once at library load) and restore its previous setting on exit."""

    def __init__(self, name: str, value="1"):
        import os
        self.name, self.value, self.prev = name, value, os.environ.get(name)

    def __enter__(self):
        check(_lib.hex_debug_set_switch(self.name.encode(), None if self.value is None else str(self.value).encode()),
              "hex_debug_set_switch")
        return self

    def __exit__(self, *exc):
        check(_lib.hex_debug_set_switch(self.name.encode(), None if self.prev is None else self.prev.encode()),
              "hex_debug_set_switch")


def launch_count() -> int:
    return int(_lib.hex_launch_count())
