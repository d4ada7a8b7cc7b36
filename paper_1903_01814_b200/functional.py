"""Torch-facing hexagonal conv / pool ops over the C ABI (libhexconv.so).

PyTorch supplies device memory, streams and autograd bookkeeping only; each
op is one (or a few) calls into the library's CUDA kernels.  Shapes follow
the declared layout: "NCHW" tensors are (B, C, H, W), "NHWC" tensors are
(B, H, W, C).  Weights are (Cout, Cin, T) with taps in canonical order
(A2).  Parity 0 = odd columns physically lower
(A1).
"""
from __future__ import annotations

import ctypes

import torch

from . import _abi as A

_DTYPES = {torch.float32: A.F32, torch.bfloat16: A.BF16}
_LAYOUTS = {"NCHW": A.NCHW, "NHWC": A.NHWC}


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check_cuda(*ts):
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("hexconv ops take CUDA tensors (there is no CPU path)")
        if not t.is_contiguous():
            raise ValueError("hexconv ops take contiguous tensors in the declared layout")


def _expect(t, shape, dtype, name):
    """Validate a tensor against the descriptor before its pointer crosses the C ABI (the library sees
    only the descriptor, so a wrong shape here would be an out-of-bounds access there)."""
    if t is None:
        return
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)} does not match the descriptor's {tuple(shape)}")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")


def _dtype_ok(t):
    if t.dtype not in _DTYPES:
        raise ValueError(f"unsupported dtype {t.dtype} (float32 or bfloat16)")


def _dims(x, layout):
    if layout == "NCHW":
        B, C, H, W = x.shape
    elif layout == "NHWC":
        B, H, W, C = x.shape
    else:
        raise ValueError(f"unknown layout {layout}")
    return B, C, H, W


def _shape(layout, B, C, H, W):
    return (B, C, H, W) if layout == "NCHW" else (B, H, W, C)


def num_taps(n: int) -> int:
    return A.num_taps(n)


def output_shape(H: int, W: int, stride: int = 1, parity: int = 0):
    return A.output_shape(H, W, stride, parity)


def conv_desc(B, Cin, Cout, H, W, n, stride, parity, dtype, layout) -> A.ConvDesc:
    return A.ConvDesc(B, Cin, Cout, H, W, n, stride, parity, _DTYPES[dtype], _LAYOUTS[layout])


def conv_algo(B, Cin, Cout, H, W, n, stride, parity, dtype, layout, pass_id=0) -> str:
    """'tcgen05' (bf16 tensor cores), 'tcgen05-tf32' (fp32 in 3xTF32 on the tensor cores) or 'stencil'
    (CUDA cores): the kernel family the library picks for this call."""
    d = conv_desc(B, Cin, Cout, H, W, n, stride, parity, dtype, layout)
    a = ctypes.c_int32()
    A.check(A.lib().hex_conv2d_algo(ctypes.byref(d), pass_id, ctypes.byref(a)), "hex_conv2d_algo")
    return {1: "tcgen05", 2: "tcgen05-tf32"}.get(a.value, "stencil")


def _workspace(desc, pass_id, device):
    nbytes = ctypes.c_size_t()
    A.check(A.lib().hex_conv2d_workspace_size(ctypes.byref(desc), pass_id, ctypes.byref(nbytes)),
            "hex_conv2d_workspace_size")
    if nbytes.value == 0:
        return None, 0
    return torch.empty(nbytes.value, dtype=torch.uint8, device=device), nbytes.value


# ------------------------------------------------------------------ convolution
def conv2d_fwd(x, w, bias=None, n: int = 1, stride: int = 1, parity: int = 0, relu: bool = False,
               layout: str = "NCHW", out=None):
    """y = hexconv(x, w) + bias (then ReLU if relu)."""
    _check_cuda(x, w, bias, out)
    B, Cin, H, W = _dims(x, layout)
    Cout, Ci2, T = w.shape
    if Ci2 != Cin:
        raise ValueError("channel mismatch")
    if T != A.num_taps(n):
        raise ValueError("weight tap count does not match kernel size")
    if w.dtype != x.dtype:
        raise ValueError("x and w must share a dtype")
    _dtype_ok(x)
    _expect(bias, (Cout,), torch.float32, "bias")
    Ho, Wo, _ = A.output_shape(H, W, stride, parity)
    d = conv_desc(B, Cin, Cout, H, W, n, stride, parity, x.dtype, layout)
    if out is None:
        out = torch.empty(_shape(layout, B, Cout, Ho, Wo), dtype=x.dtype, device=x.device)
    _expect(out, _shape(layout, B, Cout, Ho, Wo), x.dtype, "out")
    ws, nb = _workspace(d, 0, x.device)
    A.check(A.lib().hex_conv2d_fwd(ctypes.byref(d), _ptr(x), _ptr(w), _ptr(bias), int(relu), _ptr(out),
                                   _ptr(ws), nb, _stream()), "hex_conv2d_fwd")
    return out


def conv2d_fwd_maxpool(x, w, bias=None, n: int = 1, parity: int = 0, relu: bool = True, layout: str = "NHWC"):
    """(y, argmax) = hex max pool (n = 1, stride 2) of relu?(hexconv(x, w) + bias), fused: the conv
    output is never materialised (bf16 NHWC, stride 1).  Bit-identical to conv2d_fwd followed by
    pool2d_fwd; raises HexError(HEX_ERR_UNSUPPORTED) where no fused kernel applies."""
    _check_cuda(x, w, bias)
    B, Cin, H, W = _dims(x, layout)
    _dtype_ok(x)
    Cout = w.shape[0]
    _expect(w, (Cout, Cin, A.num_taps(n)), x.dtype, "w")
    _expect(bias, (Cout,), torch.float32, "bias")
    d = conv_desc(B, Cin, Cout, H, W, n, 1, parity, x.dtype, layout)
    Ho, Wo, _ = A.output_shape(H, W, 2, parity)
    y = torch.empty(_shape(layout, B, Cout, Ho, Wo), dtype=x.dtype, device=x.device)
    am = torch.empty(_shape(layout, B, Cout, Ho, Wo), dtype=torch.uint8, device=x.device)
    ws, nb = _workspace(d, 0, x.device)
    A.check(A.lib().hex_conv2d_fwd_maxpool(ctypes.byref(d), _ptr(x), _ptr(w), _ptr(bias), int(relu), _ptr(y),
                                           _ptr(am), _ptr(ws), nb, _stream()), "hex_conv2d_fwd_maxpool")
    return y, am


def conv2d_fwd_avgpool(x, w, bias=None, n: int = 1, parity: int = 0, relu: bool = True, layout: str = "NHWC"):
    """y = hex average pool (n = 1, stride 2, in-grid count) of relu?(hexconv(x, w) + bias), fused
    (hex_conv2d_fwd_pool, HEX_POOL_AVG); bit-identical to conv2d_fwd followed by pool2d_fwd(mode="avg")."""
    _check_cuda(x, w, bias)
    B, Cin, H, W = _dims(x, layout)
    _dtype_ok(x)
    Cout = w.shape[0]
    _expect(w, (Cout, Cin, A.num_taps(n)), x.dtype, "w")
    _expect(bias, (Cout,), torch.float32, "bias")
    d = conv_desc(B, Cin, Cout, H, W, n, 1, parity, x.dtype, layout)
    Ho, Wo, _ = A.output_shape(H, W, 2, parity)
    y = torch.empty(_shape(layout, B, Cout, Ho, Wo), dtype=x.dtype, device=x.device)
    ws, nb = _workspace(d, 0, x.device)
    A.check(A.lib().hex_conv2d_fwd_pool(ctypes.byref(d), A.POOL_AVG, _ptr(x), _ptr(w), _ptr(bias), int(relu),
                                        _ptr(y), None, _ptr(ws), nb, _stream()), "hex_conv2d_fwd_pool")
    return y


def conv2d_fwd_pool_supported(B, Cin, Cout, H, W, n, parity=0, mode="max", dtype=torch.bfloat16,
                              layout="NHWC") -> bool:
    d = conv_desc(B, Cin, Cout, H, W, n, 1, parity, dtype, layout)
    m = {"max": A.POOL_MAX, "avg": A.POOL_AVG, "avg_pad": A.POOL_AVG_PAD}[mode]
    return bool(A.lib().hex_conv2d_fwd_pool_supported(ctypes.byref(d), m))


def conv2d_fwd_maxpool_supported(B, Cin, Cout, H, W, n, parity=0, dtype=torch.bfloat16, layout="NHWC") -> bool:
    d = conv_desc(B, Cin, Cout, H, W, n, 1, parity, dtype, layout)
    return bool(A.lib().hex_conv2d_fwd_maxpool_supported(ctypes.byref(d)))


def conv2d_bwd_data(dy, w, in_hw, n: int = 1, stride: int = 1, parity: int = 0, layout: str = "NCHW",
                    relu_y=None, out=None):
    """dx = adjoint of conv2d_fwd applied to dy; optionally masked by relu_y > 0."""
    _check_cuda(dy, w, relu_y, out)
    B, Cout, Ho, Wo = _dims(dy, layout)
    _dtype_ok(dy)
    Co2, Cin, T = w.shape
    H, W = in_hw
    if Co2 != Cout:
        raise ValueError("channel mismatch")
    _expect(w, (Cout, Cin, A.num_taps(n)), dy.dtype, "w")
    Ho_, Wo_, _ = A.output_shape(H, W, stride, parity)
    _expect(dy, _shape(layout, B, Cout, Ho_, Wo_), dy.dtype, "dy")
    _expect(relu_y, _shape(layout, B, Cin, H, W), dy.dtype, "relu_y")
    d = conv_desc(B, Cin, Cout, H, W, n, stride, parity, dy.dtype, layout)
    if out is None:
        out = torch.empty(_shape(layout, B, Cin, H, W), dtype=dy.dtype, device=dy.device)
    _expect(out, _shape(layout, B, Cin, H, W), dy.dtype, "out")
    ws, nb = _workspace(d, 1, dy.device)
    A.check(A.lib().hex_conv2d_bwd_data(ctypes.byref(d), _ptr(dy), _ptr(w), _ptr(relu_y), _ptr(out),
                                        _ptr(ws), nb, _stream()), "hex_conv2d_bwd_data")
    return out


def conv2d_bwd_weight(x, dy, n: int = 1, stride: int = 1, parity: int = 0, layout: str = "NCHW",
                      with_bias: bool = True, dw=None, dbias=None, accumulate: bool = False):
    """(dw fp32 [Cout,Cin,T], dbias fp32 [Cout] or None)."""
    _check_cuda(x, dy, dw, dbias)
    B, Cin, H, W = _dims(x, layout)
    _dtype_ok(x)
    Cout = _dims(dy, layout)[1]
    T = A.num_taps(n)
    Ho, Wo, _ = A.output_shape(H, W, stride, parity)
    _expect(dy, _shape(layout, B, Cout, Ho, Wo), x.dtype, "dy")
    d = conv_desc(B, Cin, Cout, H, W, n, stride, parity, x.dtype, layout)
    if dw is None:
        dw = torch.empty((Cout, Cin, T), dtype=torch.float32, device=x.device)
    if with_bias and dbias is None:
        dbias = torch.empty((Cout,), dtype=torch.float32, device=x.device)
    _expect(dw, (Cout, Cin, T), torch.float32, "dw")
    _expect(dbias if with_bias else None, (Cout,), torch.float32, "dbias")
    ws, nb = _workspace(d, 2, x.device)
    A.check(A.lib().hex_conv2d_bwd_weight(ctypes.byref(d), _ptr(x), _ptr(dy), _ptr(dw),
                                          _ptr(dbias if with_bias else None), int(accumulate),
                                          _ptr(ws), nb, _stream()), "hex_conv2d_bwd_weight")
    return dw, (dbias if with_bias else None)


# ------------------------------------------------------------------ custom kernels
def tap_axial(n: int):
    """The T(n) taps of a size-n hexagonal kernel as axial displacements (dq, dr), in the canonical
    weight order (A2: column-major left to right, top to bottom = lexicographic (dq, dr))."""
    if n < 0:
        raise ValueError("kernel size n >= 0")
    return A.tap_axial(n)


def custom_kernel(n: int, value, out_channels: int = 1, in_channels: int = 1, dtype=torch.float32, device="cuda"):
    """A hexagonal kernel with user-defined element values ("structure detecting kernels ... smoothing",
    PAPER.md:207-210): value(dq, dr) -> float for each axial tap displacement, or a dict {(dq, dr): v}
    (missing taps are 0).  Returns weights [out_channels, in_channels, T(n)] with every (co, ci) pair
    set to the same kernel, ready for conv2d_fwd / hex_conv2d."""
    taps = tap_axial(n)
    fn = (lambda dq, dr: value.get((dq, dr), 0.0)) if isinstance(value, dict) else value
    k = torch.tensor([float(fn(dq, dr)) for dq, dr in taps], dtype=torch.float32)
    return k.view(1, 1, -1).expand(out_channels, in_channels, -1).contiguous().to(device=device, dtype=dtype)


def ring_kernel(ring_values, out_channels: int = 1, in_channels: int = 1, dtype=torch.float32, device="cuda"):
    """A rotationally symmetric kernel of size n = len(ring_values) - 1: the value of a tap is
    ring_values[d] for hexagonal distance d from the centre (e.g. [1/7] * 2 = 7-cell mean smoothing)."""
    n = len(ring_values) - 1
    return custom_kernel(n, lambda dq, dr: ring_values[(abs(dq) + abs(dr) + abs(dq + dr)) // 2], out_channels,
                         in_channels, dtype, device)


# ------------------------------------------------------------------ 3-D convolution
_LAYOUTS3 = {"NCDHW": A.NCHW, "NDHWC": A.NHWC}


def _dims3(x, layout):
    if layout == "NCDHW":
        B, C, D, H, W = x.shape
    elif layout == "NDHWC":
        B, D, H, W, C = x.shape
    else:
        raise ValueError(f"unknown 3-D layout {layout}")
    return B, C, D, H, W


def _shape3(layout, B, C, D, H, W):
    return (B, C, D, H, W) if layout == "NCDHW" else (B, D, H, W, C)


def conv3d_desc(B, Cin, Cout, D, H, W, n, kd, stride, depth_stride, parity, dtype, layout) -> A.Conv3dDesc:
    return A.Conv3dDesc(B, Cin, Cout, D, H, W, n, kd, stride, depth_stride, parity, _DTYPES[dtype], _LAYOUTS3[layout])


def conv3d_output_shape(desc):
    Do, Ho, Wo = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    A.check(A.lib().hex_conv3d_output_shape(ctypes.byref(desc), ctypes.byref(Do), ctypes.byref(Ho),
                                            ctypes.byref(Wo)), "hex_conv3d_output_shape")
    return Do.value, Ho.value, Wo.value


def _workspace3(desc, pass_id, device):
    nbytes = ctypes.c_size_t()
    A.check(A.lib().hex_conv3d_workspace_size(ctypes.byref(desc), pass_id, ctypes.byref(nbytes)),
            "hex_conv3d_workspace_size")
    return torch.empty(max(nbytes.value, 1), dtype=torch.uint8, device=device), nbytes.value


def conv3d_fwd(x, w, bias=None, n: int = 1, stride: int = 1, depth_stride: int = 1, parity: int = 0,
               relu: bool = False, layout: str = "NCDHW", out=None):
    """3-D hex conv: w [Cout, Cin, kd, T]; y = conv3d(x, w) + bias (ReLU optional)."""
    _check_cuda(x, w, bias, out)
    B, Cin, D, H, W = _dims3(x, layout)
    Cout, Ci2, kd, T = w.shape
    if Ci2 != Cin:
        raise ValueError("channel mismatch")
    if T != A.num_taps(n):
        raise ValueError("weight tap count does not match kernel size")
    if w.dtype != x.dtype:
        raise ValueError("x and w must share a dtype")
    d = conv3d_desc(B, Cin, Cout, D, H, W, n, kd, stride, depth_stride, parity, x.dtype, layout)
    Do, Ho, Wo = conv3d_output_shape(d)
    if out is None:
        out = torch.empty(_shape3(layout, B, Cout, Do, Ho, Wo), dtype=x.dtype, device=x.device)
    ws, nb = _workspace3(d, 0, x.device)
    A.check(A.lib().hex_conv3d_fwd(ctypes.byref(d), _ptr(x), _ptr(w), _ptr(bias), int(relu), _ptr(out),
                                   _ptr(ws), nb, _stream()), "hex_conv3d_fwd")
    return out


def conv3d_bwd_data(dy, w, in_dhw, n: int = 1, stride: int = 1, depth_stride: int = 1, parity: int = 0,
                    layout: str = "NCDHW", out=None):
    _check_cuda(dy, w, out)
    B, Cout = _dims3(dy, layout)[:2]
    Co2, Cin, kd, T = w.shape
    D, H, W = in_dhw
    if Co2 != Cout:
        raise ValueError("channel mismatch")
    d = conv3d_desc(B, Cin, Cout, D, H, W, n, kd, stride, depth_stride, parity, dy.dtype, layout)
    if out is None:
        out = torch.empty(_shape3(layout, B, Cin, D, H, W), dtype=dy.dtype, device=dy.device)
    ws, nb = _workspace3(d, 1, dy.device)
    A.check(A.lib().hex_conv3d_bwd_data(ctypes.byref(d), _ptr(dy), _ptr(w), _ptr(out), _ptr(ws), nb, _stream()),
            "hex_conv3d_bwd_data")
    return out


def conv3d_bwd_weight(x, dy, kd: int, n: int = 1, stride: int = 1, depth_stride: int = 1, parity: int = 0,
                      layout: str = "NCDHW", with_bias: bool = True, dw=None, dbias=None, accumulate: bool = False):
    """(dw fp32 [Cout, Cin, kd, T], dbias fp32 [Cout] or None)."""
    _check_cuda(x, dy, dw, dbias)
    B, Cin, D, H, W = _dims3(x, layout)
    Cout = _dims3(dy, layout)[1]
    T = A.num_taps(n)
    d = conv3d_desc(B, Cin, Cout, D, H, W, n, kd, stride, depth_stride, parity, x.dtype, layout)
    if dw is None:
        dw = torch.empty((Cout, Cin, kd, T), dtype=torch.float32, device=x.device)
    if with_bias and dbias is None:
        dbias = torch.empty((Cout,), dtype=torch.float32, device=x.device)
    ws, nb = _workspace3(d, 2, x.device)
    A.check(A.lib().hex_conv3d_bwd_weight(ctypes.byref(d), _ptr(x), _ptr(dy), _ptr(dw),
                                          _ptr(dbias if with_bias else None), int(accumulate), _ptr(ws), nb,
                                          _stream()), "hex_conv3d_bwd_weight")
    return dw, (dbias if with_bias else None)


class HexConv3dFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, bias, n, stride, depth_stride, parity, layout):
        ctx.save_for_backward(x, w)
        ctx.cfg = (n, stride, depth_stride, parity, layout, bias is not None)
        return conv3d_fwd(x, w, bias, n, stride, depth_stride, parity, False, layout)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        n, stride, depth_stride, parity, layout, has_bias = ctx.cfg
        gy = gy.contiguous()
        B, Cin, D, H, W = _dims3(x, layout)
        dx = conv3d_bwd_data(gy, w, (D, H, W), n, stride, depth_stride, parity, layout) \
            if ctx.needs_input_grad[0] else None
        dw, db = conv3d_bwd_weight(x, gy, w.shape[2], n, stride, depth_stride, parity, layout, with_bias=has_bias)
        return dx, dw.to(w.dtype), db, None, None, None, None, None


def hex_conv3d(x, w, bias=None, n=1, stride=1, depth_stride=1, parity=0, layout="NCDHW"):
    """Autograd 3-D hex convolution (hexagonal x-y, equidistant z)."""
    return HexConv3dFn.apply(x, w, bias, n, stride, depth_stride, parity, layout)


def gather_map(H: int, W: int, n: int, stride: int = 1, parity: int = 0, device="cuda"):
    Ho, Wo, _ = A.output_shape(H, W, stride, parity)
    T = A.num_taps(n)
    m = torch.empty((Ho, Wo, T), dtype=torch.int32, device=device)
    d = A.ConvDesc(1, 1, 1, H, W, n, stride, parity, A.F32, A.NCHW)
    A.check(A.lib().hex_conv2d_gather_map(ctypes.byref(d), _ptr(m), _stream()), "hex_conv2d_gather_map")
    return m


# ------------------------------------------------------------------ pooling
_POOL_MODES = {"max": A.POOL_MAX, "avg": A.POOL_AVG, "avg_pad": A.POOL_AVG_PAD}


def pool_desc(B, C, H, W, n, stride, parity, dtype, layout, mode) -> A.PoolDesc:
    """mode: "max", "avg" (in-grid count, A8) or "avg_pad" (include-pad: divide by T(n))."""
    return A.PoolDesc(B, C, H, W, n, stride, parity, _DTYPES[dtype], _LAYOUTS[layout], _POOL_MODES[mode])


def pool2d_fwd(x, n: int = 1, stride: int = 1, parity: int = 0, mode: str = "max", layout: str = "NCHW",
               need_argmax: bool = True, out=None):
    """(y, argmax uint8 or None)."""
    _check_cuda(x, out)
    B, C, H, W = _dims(x, layout)
    _dtype_ok(x)
    Ho, Wo, _ = A.output_shape(H, W, stride, parity)
    d = pool_desc(B, C, H, W, n, stride, parity, x.dtype, layout, mode)
    if out is None:
        out = torch.empty(_shape(layout, B, C, Ho, Wo), dtype=x.dtype, device=x.device)
    _expect(out, _shape(layout, B, C, Ho, Wo), x.dtype, "out")
    am = None
    if mode == "max" and need_argmax:
        am = torch.empty(_shape(layout, B, C, Ho, Wo), dtype=torch.uint8, device=x.device)
    A.check(A.lib().hex_pool2d_fwd(ctypes.byref(d), _ptr(x), _ptr(out), _ptr(am), _stream()), "hex_pool2d_fwd")
    return out, am


def pool2d_bwd(dy, argmax, in_hw, n: int = 1, stride: int = 1, parity: int = 0, mode: str = "max",
               layout: str = "NCHW", out=None, relu_y=None):
    """dx of the pool; with relu_y (the pool's post-ReLU input) the ReLU backward is
    fused: dx *= (relu_y > 0)."""
    _check_cuda(dy, argmax, out, relu_y)
    B, C, Ho, Wo = _dims(dy, layout)
    _dtype_ok(dy)
    H, W = in_hw
    Ho_, Wo_, _ = A.output_shape(H, W, stride, parity)
    _expect(dy, _shape(layout, B, C, Ho_, Wo_), dy.dtype, "dy")
    if mode == "max":
        if argmax is None:
            raise ValueError("max-pool backward needs the forward's argmax")
        _expect(argmax, _shape(layout, B, C, Ho_, Wo_), torch.uint8, "argmax")
    d = pool_desc(B, C, H, W, n, stride, parity, dy.dtype, layout, mode)
    if out is None:
        out = torch.empty(_shape(layout, B, C, H, W), dtype=dy.dtype, device=dy.device)
    _expect(out, _shape(layout, B, C, H, W), dy.dtype, "out")
    if relu_y is not None:
        _expect(relu_y, _shape(layout, B, C, H, W), dy.dtype, "relu_y")
        A.check(A.lib().hex_pool2d_bwd_relu(ctypes.byref(d), _ptr(dy), _ptr(argmax), _ptr(relu_y), _ptr(out),
                                            _stream()), "hex_pool2d_bwd_relu")
        return out
    A.check(A.lib().hex_pool2d_bwd(ctypes.byref(d), _ptr(dy), _ptr(argmax), _ptr(out), _stream()),
            "hex_pool2d_bwd")
    return out


# ------------------------------------------------------------------ autograd
def relu_bwd(dy, y):
    """dy * (y > 0) in one library kernel (y = the post-ReLU forward output)."""
    _check_cuda(dy, y)
    _expect(y, tuple(dy.shape), dy.dtype, "y")
    _dtype_ok(dy)
    dx = torch.empty_like(dy)
    A.check(A.lib().hex_relu_bwd(dy.numel(), _DTYPES[dy.dtype], _ptr(dy), _ptr(y), _ptr(dx), _stream()),
            "hex_relu_bwd")
    return dx


class HexConv2dFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, bias, n, stride, parity, relu, layout):
        y = conv2d_fwd(x, w, bias, n, stride, parity, relu, layout)
        ctx.save_for_backward(x, w, y if relu else None)
        ctx.cfg = (n, stride, parity, relu, layout, bias is not None)
        return y

    @staticmethod
    def backward(ctx, gy):
        x, w, y = ctx.saved_tensors
        n, stride, parity, relu, layout, has_bias = ctx.cfg
        gy = gy.contiguous()
        if relu:
            gy = relu_bwd(gy, y)
        B, Cin, H, W = _dims(x, layout)
        dx = conv2d_bwd_data(gy, w, (H, W), n, stride, parity, layout) if ctx.needs_input_grad[0] else None
        dw, db = conv2d_bwd_weight(x, gy, n, stride, parity, layout, with_bias=has_bias)
        return dx, dw.to(w.dtype), db, None, None, None, None, None


class HexPool2dFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, n, stride, parity, mode, layout):
        y, am = pool2d_fwd(x, n, stride, parity, mode, layout)
        ctx.save_for_backward(am) if am is not None else ctx.save_for_backward()
        B, C, H, W = _dims(x, layout)
        ctx.cfg = (n, stride, parity, mode, layout, H, W)
        return y

    @staticmethod
    def backward(ctx, gy):
        n, stride, parity, mode, layout, H, W = ctx.cfg
        am = ctx.saved_tensors[0] if mode == "max" else None
        return pool2d_bwd(gy.contiguous(), am, (H, W), n, stride, parity, mode, layout), None, None, None, None, None


def hex_conv2d(x, w, bias=None, n=1, stride=1, parity=0, relu=False, layout="NCHW"):
    return HexConv2dFn.apply(x, w, bias, n, stride, parity, relu, layout)


def hex_max_pool2d(x, n=1, stride=1, parity=0, layout="NCHW"):
    return HexPool2dFn.apply(x, n, stride, parity, "max", layout)


def hex_avg_pool2d(x, n=1, stride=1, parity=0, layout="NCHW", count_include_pad=False):
    return HexPool2dFn.apply(x, n, stride, parity, "avg_pad" if count_include_pad else "avg", layout)
