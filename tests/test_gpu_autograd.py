"""The autograd wrappers -- the "adopting the PyTorch-API" feature (PAPER.md:206-207,
Sec. 2 "Software Functionalities"): hex_conv2d, hex_max_pool2d and
hex_avg_pool2d used as ordinary differentiable torch ops.  For a random
cotangent R, loss = <op(x), R>; torch's backward through the wrapper must give
the fp64 oracle's adjoint (PAPER.md:144-151 conv, 202-205 pool) applied to R
(ReLU mask taken on the GPU's own forward output, reading A17):
fp32 1e-5 and bf16 2e-2 normwise (A14), weight gradients 1e-3 for bf16.
A two-op chain (conv -> ReLU -> max pool -> conv) checks the wrappers compose."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1903_01814_b200 import functional
    return functional


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


def dev(a, dtype=torch.float32, grad=False):
    t = torch.tensor(np.asarray(a, np.float32), dtype=torch.float32, device="cuda").to(dtype)
    return t.requires_grad_(grad)


def np64(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("n,s,pi", [(1, 1, 0), (2, 1, 1), (2, 2, 0), (1, 3, 1)])
def test_hex_conv2d_autograd_f32(F, oracle, relu, n, s, pi):
    import synth
    B, Cin, Cout, H, W = 2, 3, 5, 11, 12
    T = F.num_taps(n)
    x = synth.round_f32(synth.normal((B, Cin, H, W), 1))
    w = synth.round_f32(synth.normal((Cout, Cin, T), 2, 0.4))
    b = synth.round_f32(synth.normal((Cout,), 3))
    Ho, Wo, _ = F.output_shape(H, W, s, pi)
    R = synth.round_f32(synth.normal((B, Cout, Ho, Wo), 4))
    xd, wd, bd = dev(x, grad=True), dev(w, grad=True), dev(b, grad=True)
    y = F.hex_conv2d(xd, wd, bd, n=n, stride=s, parity=pi, relu=relu)
    (y * dev(R)).sum().backward()
    yref = oracle.conv2d_fwd(x, w, b, n=n, s=s, pi=pi)
    assert rel(np64(y), np.maximum(yref, 0) if relu else yref) <= 1e-5
    g = R * (np64(y) > 0) if relu else R
    dxr, dwr, dbr = oracle.conv2d_bwd(x, w, g, n=n, s=s, pi=pi)
    assert rel(np64(xd.grad), dxr) <= 1e-5
    assert rel(np64(wd.grad), dwr) <= 1e-5
    assert rel(np64(bd.grad), dbr) <= 1e-5


def test_hex_conv2d_autograd_bf16_nhwc_tensor_cores(F, oracle):
    import synth
    B, C, H, W, n = 2, 64, 10, 13, 1
    T = F.num_taps(n)
    assert F.conv_algo(B, C, C, H, W, n, 1, 0, torch.bfloat16, "NHWC", 0) == "tcgen05"
    x = synth.round_bf16(synth.normal((B, C, H, W), 5))
    w = synth.round_bf16(synth.normal((C, C, T), 6, 1.0 / np.sqrt(C * T)))
    R = synth.round_bf16(synth.normal((B, C, H, W), 7))
    nhwc = lambda a, g=False: dev(a.transpose(0, 2, 3, 1), torch.bfloat16).contiguous().requires_grad_(g)
    xd = nhwc(x, True)
    wd = dev(w, torch.bfloat16, grad=True)
    y = F.hex_conv2d(xd, wd, None, n=n, relu=True, layout="NHWC")
    (y.float() * nhwc(R).float()).sum().backward()
    yg = np64(y).transpose(0, 3, 1, 2)
    assert rel(yg, np.maximum(oracle.conv2d_fwd(x, w, None, n=n), 0)) <= 2e-2
    g = synth.round_bf16(R * (yg > 0))
    dxr, dwr, _ = oracle.conv2d_bwd(x, w, g, n=n)
    assert rel(np64(xd.grad).transpose(0, 3, 1, 2), dxr) <= 2e-2
    assert rel(np64(wd.grad), dwr) <= 2e-2     # the fp32 gradient is returned in the weight's dtype (bf16)


@pytest.mark.parametrize("mode", ["max", "avg", "avg_pad"])
@pytest.mark.parametrize("n,s,pi", [(1, 2, 0), (1, 1, 1), (2, 2, 1)])
def test_hex_pool2d_autograd(F, oracle, mode, n, s, pi):
    import synth
    B, C, H, W = 2, 3, 12, 11
    x = synth.round_f32(synth.normal((B, C, H, W), 8))
    Ho, Wo, _ = F.output_shape(H, W, s, pi)
    R = synth.round_f32(synth.normal((B, C, Ho, Wo), 9))
    xd = dev(x, grad=True)
    if mode == "max":
        y = F.hex_max_pool2d(xd, n=n, stride=s, parity=pi)
    else:
        y = F.hex_avg_pool2d(xd, n=n, stride=s, parity=pi, count_include_pad=(mode == "avg_pad"))
    (y * dev(R)).sum().backward()
    yr, am = oracle.pool2d_fwd(x, n=n, s=s, pi=pi, mode=mode)
    assert rel(np64(y), yr) <= 1e-5
    assert rel(np64(xd.grad), oracle.pool2d_bwd(R, am, H, W, n=n, s=s, pi=pi, mode=mode)) <= 1e-5


def test_autograd_chain_conv_pool_conv(F, oracle):
    import synth
    B, H, W = 2, 14, 13
    x = synth.round_f32(synth.normal((B, 2, H, W), 10))
    w1 = synth.round_f32(synth.normal((4, 2, 7), 11, 0.5))
    w2 = synth.round_f32(synth.normal((3, 4, 19), 12, 0.3))
    xd, w1d, w2d = dev(x, grad=True), dev(w1, grad=True), dev(w2, grad=True)
    a = F.hex_conv2d(xd, w1d, None, n=1, relu=True)
    p = F.hex_max_pool2d(a, n=1, stride=2)
    y = F.hex_conv2d(p, w2d, None, n=2)
    R = synth.round_f32(synth.normal(tuple(y.shape), 13))
    (y * dev(R)).sum().backward()
    # oracle chain, each op fed the GPU's own forward tensors (A17)
    an, pn = np64(a), np64(p)
    assert rel(pn, oracle.pool2d_fwd(an, n=1, s=2)[0]) <= 1e-5
    dp, dw2, _ = oracle.conv2d_bwd(pn, w2, R, n=2)
    _, am = oracle.pool2d_fwd(an, n=1, s=2)
    da = oracle.pool2d_bwd(dp, am, H, W, n=1, s=2) * (an > 0)
    dx, dw1, _ = oracle.conv2d_bwd(x, w1, da, n=1)
    assert rel(np64(w2d.grad), dw2) <= 1e-5
    assert rel(np64(w1d.grad), dw1) <= 1e-5
    assert rel(np64(xd.grad), dx) <= 1e-5


def test_wrappers_reject_mismatched_shapes(F):
    x = torch.zeros(1, 2, 8, 9, device="cuda")
    w = torch.zeros(3, 2, 7, device="cuda")
    dy_bad = torch.zeros(1, 3, 4, 5, device="cuda")          # stride-1 output is 8 x 9
    with pytest.raises(ValueError):
        F.conv2d_bwd_data(dy_bad, w, (8, 9), n=1)
    with pytest.raises(ValueError):
        F.conv2d_bwd_weight(x, dy_bad, n=1)
    with pytest.raises(ValueError):
        F.conv2d_fwd(x, w, None, n=1, out=torch.zeros(1, 3, 8, 8, device="cuda"))
    with pytest.raises(ValueError):
        F.conv2d_bwd_weight(x, torch.zeros(1, 3, 8, 9, device="cuda"), n=1,
                            dw=torch.zeros(3, 2, 7, device="cuda", dtype=torch.float64))
    y, am = F.pool2d_fwd(x, n=1, stride=2)
    with pytest.raises(ValueError):
        F.pool2d_bwd(y, am[..., :-1].contiguous(), (8, 9), n=1, stride=2)
    with pytest.raises(ValueError):
        F.pool2d_bwd(y, None, (8, 9), n=1, stride=2, mode="max")


@pytest.mark.parametrize("mode", ["max", "avg"])
@pytest.mark.parametrize("pi", [0, 1])
@pytest.mark.parametrize("layout,dtype", [("NCHW", torch.float32), ("NHWC", torch.bfloat16)])
def test_pool_bwd_fused_relu_mask(F, oracle, mode, pi, layout, dtype):
    # hex_pool2d_bwd_relu: dx = pool_bwd(dy) * (relu_y > 0) (fused for NCHW n = 1 s = 2, two passes otherwise)
    import synth
    B, C, H, W = 2, 16, 13, 12
    x = synth.round_bf16(synth.normal((B, C, H, W), 14)) if dtype == torch.bfloat16 else \
        synth.round_f32(synth.normal((B, C, H, W), 14))
    Ho, Wo, _ = F.output_shape(H, W, 2, pi)
    g = synth.round_bf16(synth.normal((B, C, Ho, Wo), 15)) if dtype == torch.bfloat16 else \
        synth.round_f32(synth.normal((B, C, Ho, Wo), 15))
    to = (lambda a: dev(a, dtype).permute(0, 2, 3, 1).contiguous()) if layout == "NHWC" else (lambda a: dev(a, dtype))
    back = (lambda t: np64(t).transpose(0, 3, 1, 2)) if layout == "NHWC" else np64
    xd = to(x)
    y, am = F.pool2d_fwd(xd, n=1, stride=2, parity=pi, mode=mode, layout=layout)
    _, amr = oracle.pool2d_fwd(x, n=1, s=2, pi=pi, mode=mode)
    dx = F.pool2d_bwd(to(g), am, (H, W), n=1, stride=2, parity=pi, mode=mode, layout=layout, relu_y=xd)
    ref = oracle.pool2d_bwd(g, amr, H, W, n=1, s=2, pi=pi, mode=mode) * (x > 0)
    assert rel(back(dx), ref) <= (1e-5 if dtype == torch.float32 else 2e-2)
