"""fp64 CPU oracle for hexagonal convolution / pooling (HexagDLy, arXiv 1903.01814).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1903_01814_b200``) never imports it, and it
shares no code with the CUDA library.

The arithmetic lives in ``hexoracle.c`` (plain C, fp64, OpenMP over independent
output planes).  This module only marshals numpy arrays through ctypes.  Every
function cites the paper passage it follows in ``hexoracle.c``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hexoracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile hexoracle.c into liboracle.so (gcc, -O2 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64p = ctypes.POINTER(ctypes.c_int64)
        ip = ctypes.POINTER(ctypes.c_int)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_offset_to_axial.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, i64p, i64p]
        L.oracle_axial_to_offset.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, i64p, i64p]
        L.oracle_pixel_center.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double, dp, dp]
        L.oracle_hex_distance.argtypes = [ctypes.c_int64] * 4
        L.oracle_hex_distance.restype = ctypes.c_int64
        L.oracle_tap_list.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip]
        L.oracle_num_taps.argtypes = [ctypes.c_int]
        L.oracle_tap_offsets.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, ip]
        L.oracle_out_shape.argtypes = [ctypes.c_int] * 4 + [ip, ip, ip]
        L.oracle_gather_map.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p]
        L.oracle_conv2d_fwd.argtypes = [ctypes.c_int] * 8 + [ctypes.c_void_p] * 4
        L.oracle_conv2d_bwd.argtypes = [ctypes.c_int] * 8 + [ctypes.c_void_p] * 6
        L.oracle_pool2d_fwd.argtypes = [ctypes.c_int] * 8 + [ctypes.c_void_p] * 3
        L.oracle_conv3d_out_depth.argtypes = [ctypes.c_int] * 3
        L.oracle_conv3d_fwd.argtypes = [ctypes.c_int] * 11 + [ctypes.c_void_p] * 4
        L.oracle_conv3d_bwd.argtypes = [ctypes.c_int] * 11 + [ctypes.c_void_p] * 6
        L.oracle_pool2d_bwd.argtypes = [ctypes.c_int] * 8 + [ctypes.c_void_p] * 3
        L.oracle_conv2d_bwd_weight_at.argtypes = [ctypes.c_int] * 6 + [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- geometry
def offset_to_axial(row: int, col: int, pi: int = 0):
    q, r = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_offset_to_axial(row, col, pi, ctypes.byref(q), ctypes.byref(r))
    return q.value, r.value


def axial_to_offset(q: int, ra: int, pi: int = 0):
    r, c = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_axial_to_offset(q, ra, pi, ctypes.byref(r), ctypes.byref(c))
    return r.value, c.value


def pixel_center(row: int, col: int, pi: int = 0, pitch: float = 1.0):
    x, y = ctypes.c_double(), ctypes.c_double()
    lib().oracle_pixel_center(row, col, pi, pitch, ctypes.byref(x), ctypes.byref(y))
    return x.value, y.value


def hex_distance(a, b) -> int:
    return int(lib().oracle_hex_distance(a[0], a[1], b[0], b[1]))


def num_taps(n: int) -> int:
    return int(lib().oracle_num_taps(n))


def tap_list(n: int):
    """Axial (dq, dr) of every tap, canonical order."""
    T = num_taps(n)
    dq = (ctypes.c_int * T)()
    dr = (ctypes.c_int * T)()
    lib().oracle_tap_list(n, T, dq, dr)
    return list(zip(list(dq), list(dr)))


def tap_offsets(n: int, p: int):
    """Offset (dc, drow) of every tap for a centre column of parity p."""
    T = num_taps(n)
    dc = (ctypes.c_int * T)()
    dr = (ctypes.c_int * T)()
    assert lib().oracle_tap_offsets(n, p, T, dc, dr) == T
    return list(zip(list(dc), list(dr)))


def out_shape(H: int, W: int, s: int, pi: int = 0):
    """(Ho, Wo, pi_out); raises ValueError on an empty lattice."""
    Ho, Wo, po = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    st = lib().oracle_out_shape(H, W, s, pi, ctypes.byref(Ho), ctypes.byref(Wo), ctypes.byref(po))
    if st == 2:
        raise ValueError("invalid argument")
    if st == 1:
        raise ValueError("empty lattice")
    return Ho.value, Wo.value, po.value


def gather_map(H: int, W: int, n: int, s: int, pi: int = 0) -> np.ndarray:
    """int32 [Ho, Wo, T]: r*W+c of each tap's neighbour, or -1 when off-grid."""
    Ho, Wo, _ = out_shape(H, W, s, pi)
    T = num_taps(n)
    m = np.empty((Ho, Wo, T), dtype=np.int32)
    st = lib().oracle_gather_map(H, W, n, s, pi, _ptr(m))
    assert st == 0
    return m


# ---------------------------------------------------------------- ops
def conv2d_fwd(x, w, bias=None, n: int = 1, s: int = 1, pi: int = 0) -> np.ndarray:
    """x [B,Ci,H,W], w [Co,Ci,T] -> y [B,Co,Ho,Wo] (fp64)."""
    x = _f64(x)
    w = _f64(w)
    B, Ci, H, W = x.shape
    Co, Ci2, T = w.shape
    if Ci2 != Ci:
        raise ValueError("channel mismatch")
    if T != num_taps(n):
        raise ValueError("weight tap count does not match kernel size")
    Ho, Wo, _ = out_shape(H, W, s, pi)
    b = None if bias is None else _f64(bias)
    y = np.empty((B, Co, Ho, Wo), dtype=np.float64)
    st = lib().oracle_conv2d_fwd(B, Ci, Co, H, W, n, s, pi, _ptr(x), _ptr(w), _ptr(b), _ptr(y))
    assert st == 0
    return y


def conv2d_bwd(x, w, dy, n: int = 1, s: int = 1, pi: int = 0, need=("dx", "dw", "db")):
    """Returns (dx, dw, dbias) as the literal adjoint of conv2d_fwd."""
    x = _f64(x)
    w = _f64(w)
    dy = _f64(dy)
    B, Ci, H, W = x.shape
    Co = w.shape[0]
    Ho, Wo, _ = out_shape(H, W, s, pi)
    if dy.shape != (B, Co, Ho, Wo):
        raise ValueError("shape mismatch")
    dx = np.empty_like(x) if "dx" in need else None
    dw = np.empty_like(w) if "dw" in need else None
    db = np.empty((Co,), dtype=np.float64) if "db" in need else None
    st = lib().oracle_conv2d_bwd(B, Ci, Co, H, W, n, s, pi, _ptr(x), _ptr(w), _ptr(dy),
                                 _ptr(dx), _ptr(dw), _ptr(db))
    assert st == 0
    return dx, dw, db


def conv3d_out_depth(D: int, kd: int, sd: int) -> int:
    """Do = (D-1)/sd + 1 (depth centres 0, sd, 2sd, ...; kd odd), hexoracle.c."""
    Do = lib().oracle_conv3d_out_depth(D, kd, sd)
    if Do < 0:
        raise ValueError("kernel depth must be odd and >= 1, depth stride >= 1")
    return Do


def conv3d_fwd(x, w, bias=None, n: int = 1, s: int = 1, sd: int = 1, pi: int = 0) -> np.ndarray:
    """3-D hex conv: x [B,Ci,D,H,W], w [Co,Ci,kd,T] -> y [B,Co,Do,Ho,Wo] (fp64)."""
    x = _f64(x)
    w = _f64(w)
    B, Ci, D, H, W = x.shape
    Co, Ci2, kd, T = w.shape
    if Ci2 != Ci:
        raise ValueError("channel mismatch")
    if T != num_taps(n):
        raise ValueError("weight tap count does not match kernel size")
    Do = conv3d_out_depth(D, kd, sd)
    Ho, Wo, _ = out_shape(H, W, s, pi)
    b = None if bias is None else _f64(bias)
    y = np.empty((B, Co, Do, Ho, Wo), dtype=np.float64)
    st = lib().oracle_conv3d_fwd(B, Ci, Co, D, H, W, n, kd, s, sd, pi, _ptr(x), _ptr(w), _ptr(b), _ptr(y))
    assert st == 0
    return y


def conv3d_bwd(x, w, dy, n: int = 1, s: int = 1, sd: int = 1, pi: int = 0, need=("dx", "dw", "db")):
    """(dx, dw, dbias): the literal adjoint of conv3d_fwd."""
    x = _f64(x)
    w = _f64(w)
    dy = _f64(dy)
    B, Ci, D, H, W = x.shape
    Co, _, kd, _ = w.shape
    Do = conv3d_out_depth(D, kd, sd)
    Ho, Wo, _ = out_shape(H, W, s, pi)
    if dy.shape != (B, Co, Do, Ho, Wo):
        raise ValueError("shape mismatch")
    dx = np.empty_like(x) if "dx" in need else None
    dw = np.empty_like(w) if "dw" in need else None
    db = np.empty((Co,), dtype=np.float64) if "db" in need else None
    st = lib().oracle_conv3d_bwd(B, Ci, Co, D, H, W, n, kd, s, sd, pi, _ptr(x), _ptr(w), _ptr(dy),
                                 _ptr(dx), _ptr(dw), _ptr(db))
    assert st == 0
    return dx, dw, db


_POOL_MODES = {"max": 0, "avg": 1, "avg_pad": 2}


def pool2d_fwd(x, n: int = 1, s: int = 1, pi: int = 0, mode: str = "max"):
    """Returns (y, argmax uint8 or None). mode: "max", "avg" (A8: in-grid count) or "avg_pad"
    (include-pad: in-grid sum / T(n))."""
    x = _f64(x)
    B, C, H, W = x.shape
    Ho, Wo, _ = out_shape(H, W, s, pi)
    y = np.empty((B, C, Ho, Wo), dtype=np.float64)
    am = np.empty((B, C, Ho, Wo), dtype=np.uint8) if mode == "max" else None
    st = lib().oracle_pool2d_fwd(B, C, H, W, n, s, pi, _POOL_MODES[mode],
                                 _ptr(x), _ptr(y), _ptr(am))
    if st == 2:
        raise ValueError("invalid argument")
    assert st == 0
    return y, am


def pool2d_bwd(dy, argmax, H: int, W: int, n: int = 1, s: int = 1, pi: int = 0, mode: str = "max"):
    dy = _f64(dy)
    B, C, Ho, Wo = dy.shape
    if (Ho, Wo) != out_shape(H, W, s, pi)[:2]:
        raise ValueError(f"dy grid {(Ho, Wo)} is not the ({H}, {W}) s={s} lattice {out_shape(H, W, s, pi)[:2]}")
    dx = np.empty((B, C, H, W), dtype=np.float64)
    am = None if argmax is None else np.ascontiguousarray(argmax, dtype=np.uint8)
    if mode == "max" and (am is None or am.shape != dy.shape):
        raise ValueError("max-pool backward needs an argmax of dy's shape")
    st = lib().oracle_pool2d_bwd(B, C, H, W, n, s, pi, _POOL_MODES[mode],
                                 _ptr(dy), _ptr(am), _ptr(dx))
    if st == 3:
        raise ValueError("argmax names a tap index >= T or an off-grid neighbour")
    if st == 2:
        raise ValueError("invalid argument")
    assert st == 0
    return dx


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def set_threads(n: int) -> None:
    """OpenMP thread count of the oracle's loops (bench.py times it on all cores and on one)."""
    lib().oracle_set_threads(int(n))


def _storage(a):
    """(contiguous array, fmt) for float32 arrays or bf16 bit patterns (uint16)."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.float32:
        return a, 0
    if a.dtype == np.uint16:
        return a, 1
    raise TypeError("x / dy must be float32 or uint16 (bf16 bits)")


def conv2d_bwd_weight_at(x, dy, pts, n: int = 1, s: int = 1, pi: int = 0, layout: str = "NCHW"):
    """dw[co, ci, t] at the listed (co, ci, t) points; x, dy in storage format
    (float32, or uint16 bf16 bits) and `layout` ("NCHW" (B,C,H,W) / "NHWC" (B,H,W,C))."""
    x, xf = _storage(x)
    dy, df = _storage(dy)
    if layout == "NCHW":
        B, _, H, W = x.shape
        xs = [x.strides[i] // x.itemsize for i in (0, 1, 2, 3)]
        dys = [dy.strides[i] // dy.itemsize for i in (0, 1, 2, 3)]
    else:
        B, H, W, _ = x.shape
        xs = [x.strides[i] // x.itemsize for i in (0, 3, 1, 2)]
        dys = [dy.strides[i] // dy.itemsize for i in (0, 3, 1, 2)]
    pts = np.ascontiguousarray(pts, dtype=np.int32).reshape(-1, 3)
    out = np.empty(len(pts), dtype=np.float64)
    xs = np.array(xs, dtype=np.int64)
    dys = np.array(dys, dtype=np.int64)
    st = lib().oracle_conv2d_bwd_weight_at(B, H, W, n, s, pi, _ptr(x), xf, _ptr(xs), _ptr(dy), df, _ptr(dys),
                                           len(pts), _ptr(pts), _ptr(out))
    assert st == 0
    return out
