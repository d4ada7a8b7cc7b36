"""GPU parity of the 3-D hexagonal convolution through the C ABI
(hex_conv3d_fwd / _bwd_data / _bwd_weight) against the fp64 oracle (oracle.conv3d_*).

Bars as tests/test_gpu_parity.py: fp32 normwise <= 1e-5, bf16 (inputs rounded on both sides, fp32
accumulation) <= 2e-2.  bf16 NDHWC with in-plane stride 1 and channels multiples of 64 runs the
depth taps inside the K loop of the tcgen05 tap-reuse kernel (forward; backward-data for depth stride 1);
HEXCONV_CONV3D_UNFOLD=1 selects the unfold + 2-D path, which the weight gradient always takes.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5
TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1903_01814_b200 import functional
    return functional


def rel(gpu, ref):
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(np.asarray(gpu, dtype=np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def rnd(shape, seed, dtype, scale=1.0):
    a = np.random.default_rng(seed).standard_normal(shape) * scale
    if dtype == torch.bfloat16:
        from synth import round_bf16
        return round_bf16(a)
    return a.astype(np.float32).astype(np.float64)


def dev(a, dtype, layout):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    if layout == "NDHWC":
        t = t.permute(0, 2, 3, 4, 1).contiguous()
    return t.to(dtype).cuda()


def back(t, layout):
    t = t.detach().float().cpu()
    if layout == "NDHWC":
        t = t.permute(0, 4, 1, 2, 3).contiguous()
    return t.numpy().astype(np.float64)


def case(F, oracle, B, Ci, Co, D, H, W, n, kd, s, sd, pi, dtype, layout, seed, bias=True):
    T = oracle.num_taps(n)
    x = rnd((B, Ci, D, H, W), seed, dtype)
    w = rnd((Co, Ci, kd, T), seed + 1, dtype, 1.0 / np.sqrt(Ci * kd * T))
    b = rnd((Co,), seed + 2, torch.float32, 0.5) if bias else None
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    xd, wd = dev(x, dtype, layout), torch.from_numpy(w.astype(np.float32)).to(dtype).cuda()
    bd = None if b is None else torch.from_numpy(b.astype(np.float32)).cuda()
    y = F.conv3d_fwd(xd, wd, bd, n=n, stride=s, depth_stride=sd, parity=pi, layout=layout)
    yref = oracle.conv3d_fwd(x, w, b, n=n, s=s, sd=sd, pi=pi)
    assert tuple(back(y, layout).shape) == yref.shape
    assert rel(back(y, layout), yref) <= tol, ("fwd", n, kd, s, sd, pi, layout)
    g = rnd(yref.shape, seed + 3, dtype)
    gd = dev(g, dtype, layout)
    dx = F.conv3d_bwd_data(gd, wd, (D, H, W), n=n, stride=s, depth_stride=sd, parity=pi, layout=layout)
    dw, db = F.conv3d_bwd_weight(xd, gd, kd, n=n, stride=s, depth_stride=sd, parity=pi, layout=layout)
    dxr, dwr, dbr = oracle.conv3d_bwd(x, w, g, n=n, s=s, sd=sd, pi=pi)
    assert rel(back(dx, layout), dxr) <= tol, ("dgrad", n, kd, s, sd, pi, layout)
    assert rel(dw.cpu().numpy(), dwr) <= tol, ("wgrad", n, kd, s, sd, pi, layout)
    assert rel(db.cpu().numpy(), dbr) <= tol, ("dbias", n, kd, s, sd, pi, layout)
    # accumulate adds to dw / dbias
    dw2, db2 = F.conv3d_bwd_weight(xd, gd, kd, n=n, stride=s, depth_stride=sd, parity=pi, layout=layout,
                                   dw=dw.clone(), dbias=db.clone(), accumulate=True)
    assert rel(dw2.cpu().numpy(), 2 * dwr) <= tol and rel(db2.cpu().numpy(), 2 * dbr) <= tol


@pytest.mark.parametrize("layout", ["NCDHW", "NDHWC"])
def test_conv3d_f32(F, oracle, layout):
    for k, (n, kd, s, sd, pi) in enumerate([(1, 3, 1, 1, 0), (2, 3, 2, 2, 1), (1, 5, 1, 3, 1), (0, 1, 1, 1, 0),
                                             (1, 1, 3, 2, 0)]):
        case(F, oracle, 2, 3, 5, 7, 9, 10, n, kd, s, sd, pi, torch.float32, layout, 10 * k)
    # depth smaller than the kernel depth, single slice
    case(F, oracle, 1, 2, 3, 1, 6, 7, 1, 3, 1, 1, 0, torch.float32, layout, 90)


def test_conv3d_bf16_tensor_cores(F, oracle):
    # Cin' = kd * Cin = 192 / 64 and Cout = 64 / 128: the tcgen05 2-D paths on B*Do images
    for k, (Ci, Co, D, n, kd, sd, pi) in enumerate([(64, 64, 5, 1, 3, 1, 0), (64, 128, 6, 1, 3, 2, 1),
                                                      (64, 64, 4, 2, 1, 1, 0), (32, 64, 3, 1, 3, 1, 1)]):
        case(F, oracle, 2, Ci, Co, D, 16, 16, n, kd, 1, sd, pi, torch.bfloat16, "NDHWC", 200 + k)
    d = F.conv3d_desc(2, 64, 64, 5, 16, 16, 1, 3, 1, 1, 0, torch.bfloat16, "NDHWC")
    assert F.conv_algo(2 * 5, 3 * 64, 64, 16, 16, 1, 1, 0, torch.bfloat16, "NHWC") == "tcgen05"
    assert F.conv3d_output_shape(d) == (5, 16, 16)


def test_conv3d_bf16_unfold_path_agrees(F, oracle):
    from paper_1903_01814_b200 import _abi as A
    # the depth-in-K-loop tcgen05 path (default) and the unfold + 2-D path both meet the bar
    for k, (Ci, Co, D, n, kd, sd, pi) in enumerate([(64, 128, 7, 1, 3, 1, 1), (128, 64, 3, 1, 5, 1, 0),
                                                      (64, 64, 9, 2, 3, 2, 1)]):
        case(F, oracle, 1, Ci, Co, D, 20, 18, n, kd, 1, sd, pi, torch.bfloat16, "NDHWC", 300 + k)
        with A.switch("HEXCONV_CONV3D_UNFOLD"):
            case(F, oracle, 1, Ci, Co, D, 20, 18, n, kd, 1, sd, pi, torch.bfloat16, "NDHWC", 300 + k)


def test_conv3d_autograd_and_errors(F, oracle):
    from paper_1903_01814_b200._abi import HexError
    x = torch.randn(1, 2, 4, 6, 7, device="cuda", dtype=torch.float32, requires_grad=True)
    w = torch.randn(3, 2, 3, 7, device="cuda", dtype=torch.float32, requires_grad=True)
    y = F.hex_conv3d(x, w, None, n=1)
    y.square().sum().backward()
    g = (2 * y).detach().cpu().numpy().astype(np.float64)
    dxr, dwr, _ = oracle.conv3d_bwd(x.detach().cpu().numpy(), w.detach().cpu().numpy(), g, n=1)
    assert rel(x.grad.cpu().numpy(), dxr) <= TOL_F32 and rel(w.grad.cpu().numpy(), dwr) <= TOL_F32
    with pytest.raises(HexError) as e:  # even kernel depth
        F.conv3d_fwd(x.detach(), torch.zeros(3, 2, 2, 7, device="cuda"), n=1)
    assert e.value.status == 1


def test_conv3d_bf16_wgrad_depth_units(F, oracle):
    # bf16 NDHWC weight gradient with the depth taps folded into the tcgen05 tap-reuse kernel's channel-chunk
    # units (no unfolded copy of x): one wgrad launch + reduce + permute instead of unfold + the 2-D call;
    # depth strides 1 and 2, a kernel deeper than the volume (kd = 5, D = 3: zero-fill slices), n = 1 and 2
    from paper_1903_01814_b200 import _abi as A
    for k, (B, Ci, Co, D, n, kd, sd, pi) in enumerate([(2, 64, 128, 5, 1, 3, 1, 0), (1, 64, 128, 6, 2, 3, 2, 1),
                                                        (2, 128, 128, 3, 1, 5, 1, 1)]):
        case(F, oracle, B, Ci, Co, D, 16, 16, n, kd, 1, sd, pi, torch.bfloat16, "NDHWC", 400 + k)
        x = torch.randn(B, D, 16, 16, Ci, device="cuda").to(torch.bfloat16)
        Do = (D - 1) // sd + 1
        g = torch.randn(B, Do, 16, 16, Co, device="cuda").to(torch.bfloat16)
        n0 = A.launch_count()
        dw, db = F.conv3d_bwd_weight(x, g, kd, n=n, depth_stride=sd, parity=pi, layout="NDHWC")
        direct = A.launch_count() - n0
        with A.switch("HEXCONV_CONV3D_UNFOLD"):
            n0 = A.launch_count()
            dw2, db2 = F.conv3d_bwd_weight(x, g, kd, n=n, depth_stride=sd, parity=pi, layout="NDHWC")
            unfolded = A.launch_count() - n0
        assert direct == unfolded - 1, (direct, unfolded)  # no unfold launch
        assert torch.equal(dw, dw2) and torch.equal(db, db2)  # same partials, same fixed-order reduction
