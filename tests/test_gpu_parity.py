"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle.

Bars (BASELINE.json north_star):
  * integer / index work (gather maps, argmax, output shapes): bit-exact
  * fp32 path: normwise relative error max|gpu-ref| / max|ref| <= 1e-5
  * bf16 path (inputs rounded to bf16 on both sides, fp32 accumulation,
    bf16 output): normwise <= 2e-2
  * max-pool values: bit-exact (a copy of the selected input)
"""
import itertools

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
    gpu = np.asarray(gpu, dtype=np.float64)
    den = max(np.abs(ref).max(), 1e-30)
    return float(np.abs(gpu - ref).max() / den)


def to_dev(a, dtype, layout="NCHW"):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    if layout == "NHWC" and t.dim() == 4:
        t = t.permute(0, 2, 3, 1).contiguous()
    return t.to(dtype).cuda()


def to_np(t, layout="NCHW"):
    t = t.detach().float().cpu()
    if layout == "NHWC" and t.dim() == 4:
        t = t.permute(0, 3, 1, 2).contiguous()
    return t.numpy().astype(np.float64)


def rnd(shape, seed, dtype):
    a = np.random.default_rng(seed).standard_normal(shape)
    if dtype == torch.bfloat16:
        from synth import round_bf16
        return round_bf16(a)
    return a.astype(np.float32).astype(np.float64)


GRIDS = [(1, 1), (1, 6), (5, 5), (6, 7), (12, 13), (11, 12), (9, 4)]


# ------------------------------------------------------------------ geometry
def test_gather_map_bit_exact(F, oracle):
    for pi, n, s in itertools.product((0, 1), (0, 1, 2, 3), (1, 2, 3)):
        for H, W in GRIDS + [(16, 16), (7, 13)]:
            try:
                ref = oracle.gather_map(H, W, n, s, pi)
            except ValueError:
                continue
            got = F.gather_map(H, W, n, s, pi).cpu().numpy()
            assert np.array_equal(got, ref), (pi, n, s, H, W)


# ------------------------------------------------------------------ convolution, CUDA-core path
ENVELOPE = [(pi, n, s, H, W) for pi in (0, 1) for n in (0, 1, 2, 3) for s in (1, 2, 3) for (H, W) in GRIDS]


def _conv_case(F, oracle, pi, n, s, H, W, B, Cin, Cout, dtype, layout, seed):
    try:
        oracle.out_shape(H, W, s, pi)
    except ValueError:
        return
    T = oracle.num_taps(n)
    x = rnd((B, Cin, H, W), seed, dtype)
    w = rnd((Cout, Cin, T), seed + 1, dtype) * 0.5
    if dtype == torch.bfloat16:
        from synth import round_bf16
        w = round_bf16(w)
    bias = np.random.default_rng(seed + 2).standard_normal(Cout).astype(np.float32).astype(np.float64)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    xd, wd = to_dev(x, dtype, layout), torch.from_numpy(w.astype(np.float32)).to(dtype).cuda()
    bd = torch.from_numpy(bias.astype(np.float32)).cuda()
    # forward (+ bias)
    y = F.conv2d_fwd(xd, wd, bd, n=n, stride=s, parity=pi, layout=layout)
    yref = oracle.conv2d_fwd(x, w, bias, n=n, s=s, pi=pi)
    assert rel(to_np(y, layout), yref) <= tol, ("fwd", pi, n, s, H, W)
    # fused relu
    yr = F.conv2d_fwd(xd, wd, bd, n=n, stride=s, parity=pi, relu=True, layout=layout)
    assert rel(to_np(yr, layout), np.maximum(yref, 0)) <= tol
    # backward
    g = rnd(yref.shape, seed + 3, dtype)
    gd = to_dev(g, dtype, layout)
    dx = F.conv2d_bwd_data(gd, wd, (H, W), n=n, stride=s, parity=pi, layout=layout)
    dw, db = F.conv2d_bwd_weight(xd, gd, n=n, stride=s, parity=pi, layout=layout)
    dxr, dwr, dbr = oracle.conv2d_bwd(x, w, g, n=n, s=s, pi=pi)
    assert rel(to_np(dx, layout), dxr) <= tol, ("dgrad", pi, n, s, H, W)
    wtol = TOL_F32 if dtype == torch.float32 else 1e-4  # dw is fp32 accumulated from exact bf16 inputs
    assert rel(dw.cpu().numpy(), dwr) <= wtol, ("wgrad", pi, n, s, H, W)
    assert rel(db.cpu().numpy(), dbr) <= wtol, ("dbias", pi, n, s, H, W)


@pytest.mark.parametrize("pi,n,s", [(pi, n, s) for pi in (0, 1) for n in (0, 1, 2, 3) for s in (1, 2, 3)])
def test_conv_f32_nchw_envelope(F, oracle, pi, n, s):
    for k, (H, W) in enumerate(GRIDS):
        B, Cin, Cout = (1, 1, 3) if k % 2 else (2, 3, 1)
        _conv_case(F, oracle, pi, n, s, H, W, B, Cin, Cout, torch.float32, "NCHW", 100 + k)


@pytest.mark.parametrize("layout,dtype", [("NHWC", torch.float32), ("NHWC", torch.bfloat16),
                                          ("NCHW", torch.bfloat16)])
def test_conv_other_layouts(F, oracle, layout, dtype):
    for pi, n, s in [(0, 1, 1), (1, 2, 2), (0, 3, 3), (0, 2, 1), (1, 0, 2)]:
        for (H, W) in [(12, 13), (9, 4)]:
            _conv_case(F, oracle, pi, n, s, H, W, 2, 5, 6, dtype, layout, 7)


def test_conv_many_channels_f32(F, oracle):
    # channel blocks > 1 and ragged tails (Cout 37 > 32, Cin 40 > 32), several pixel blocks
    _conv_case(F, oracle, 0, 1, 1, 23, 21, 2, 40, 37, torch.float32, "NCHW", 11)
    _conv_case(F, oracle, 0, 2, 2, 24, 30, 1, 17, 70, torch.float32, "NCHW", 12)


def test_conv_deterministic(F):
    x = torch.randn(4, 16, 20, 20, device="cuda")
    w = torch.randn(32, 16, 19, device="cuda")
    g = torch.randn(4, 32, 20, 20, device="cuda")
    a = F.conv2d_bwd_weight(x, g, n=2)[0]
    b = F.conv2d_bwd_weight(x, g, n=2)[0]
    assert torch.equal(a, b)
    assert torch.equal(F.conv2d_fwd(x, w, n=2), F.conv2d_fwd(x, w, n=2))


def test_conv_fused_relu_mask_dgrad(F, oracle):
    x = rnd((2, 4, 10, 11), 5, torch.float32)
    w = rnd((3, 4, 7), 6, torch.float32)
    g = rnd((2, 3, 10, 11), 7, torch.float32)
    ry = rnd((2, 4, 10, 11), 8, torch.float32)
    dx = F.conv2d_bwd_data(to_dev(g, torch.float32), to_dev(w, torch.float32), (10, 11), n=1,
                           relu_y=to_dev(ry, torch.float32))
    ref = oracle.conv2d_bwd(x, w, g, n=1)[0] * (ry > 0)
    assert rel(to_np(dx), ref) <= TOL_F32


# ------------------------------------------------------------------ pooling
def _pool_case(F, oracle, pi, n, s, H, W, B, C, dtype, layout, mode, seed, data=None):
    try:
        oracle.out_shape(H, W, s, pi)
    except ValueError:
        return
    x = rnd((B, C, H, W), seed, dtype) if data is None else data
    xd = to_dev(x, dtype, layout)
    y, am = F.pool2d_fwd(xd, n=n, stride=s, parity=pi, mode=mode, layout=layout)
    yref, amref = oracle.pool2d_fwd(x, n=n, s=s, pi=pi, mode=mode)
    if mode == "max":
        assert np.array_equal(to_np(y, layout), yref), ("maxpool value", pi, n, s, H, W)
        amg = am.cpu()
        if layout == "NHWC":
            amg = amg.permute(0, 3, 1, 2)
        assert np.array_equal(amg.numpy(), amref), ("argmax", pi, n, s, H, W)
    else:
        tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
        assert rel(to_np(y, layout), yref) <= tol
    g = rnd(yref.shape, seed + 1, dtype)
    dx = F.pool2d_bwd(to_dev(g, dtype, layout), am, (H, W), n=n, stride=s, parity=pi, mode=mode, layout=layout)
    dxr = oracle.pool2d_bwd(g, amref, H, W, n=n, s=s, pi=pi, mode=mode)
    tol = TOL_F32 if dtype == torch.float32 else TOL_BF16
    assert rel(to_np(dx, layout), dxr) <= tol, ("pool bwd", mode, pi, n, s, H, W)


@pytest.mark.parametrize("mode", ["max", "avg", "avg_pad"])
@pytest.mark.parametrize("pi", [0, 1])
def test_pool_envelope(F, oracle, mode, pi):
    for n in (1, 2, 3):
        for s in (1, 2, 3):
            for k, (H, W) in enumerate(GRIDS):
                _pool_case(F, oracle, pi, n, s, H, W, 2, 3, torch.float32, "NCHW", mode, 200 + k)


@pytest.mark.parametrize("mode", ["max", "avg", "avg_pad"])
def test_pool_bf16_nhwc_vectorised(F, oracle, mode):
    for pi, n, s in [(0, 1, 2), (1, 1, 1), (0, 2, 3), (1, 2, 2)]:
        for C in (8, 16, 3, 32, 96):
            _pool_case(F, oracle, pi, n, s, 12, 13, 2, C, torch.bfloat16, "NHWC", mode, 300 + C)


@pytest.mark.parametrize("pi", [0, 1])
def test_maxpool_tma_band_kernel(F, oracle, pi):
    from paper_1903_01814_b200 import _abi as A
    # bf16 NHWC, C % 64 == 0, n = 1, s = 2: the TMA-staged band kernel (pool_tma.cu); bit-exact values
    # and argmax vs the oracle, and identical to the stencil kernel (HEXCONV_NO_POOL_TMA=1)
    for k, (B, C, H, W) in enumerate([(3, 64, 17, 65), (2, 128, 48, 96), (1, 192, 5, 64), (2, 64, 30, 96),
                                       (1, 64, 2, 70), (1, 256, 3, 64), (2, 128, 96, 96), (2, 256, 48, 48),
                                       (1, 64, 9, 13)]):
        x = rnd((B, C, H, W), 700 + k, torch.bfloat16)
        xd = to_dev(x, torch.bfloat16, "NHWC")
        y, am = F.pool2d_fwd(xd, n=1, stride=2, parity=pi, mode="max", layout="NHWC")
        yref, amref = oracle.pool2d_fwd(x, n=1, s=2, pi=pi, mode="max")
        assert np.array_equal(to_np(y, "NHWC"), yref), (pi, B, C, H, W)
        assert np.array_equal(am.permute(0, 3, 1, 2).cpu().numpy(), amref), (pi, B, C, H, W)
        with A.switch("HEXCONV_NO_POOL_TMA"):
            y2, am2 = F.pool2d_fwd(xd, n=1, stride=2, parity=pi, mode="max", layout="NHWC")
        assert torch.equal(y.view(torch.int16), y2.view(torch.int16)) and torch.equal(am, am2)
        # backward through the pool of these shapes: oracle within the bf16 bar
        g = rnd(yref.shape, 800 + k, torch.bfloat16)
        dx = F.pool2d_bwd(to_dev(g, torch.bfloat16, "NHWC"), am, (H, W), n=1, stride=2, parity=pi, mode="max",
                          layout="NHWC")
        dxr = oracle.pool2d_bwd(g, amref, H, W, n=1, s=2, pi=pi, mode="max")
        assert rel(to_np(dx, "NHWC"), dxr) <= TOL_BF16, (pi, B, C, H, W)


def test_maxpool_ties_first_in_canonical_order(F, oracle):
    # ReLU-like data with many exact zeros: the first in-grid tap wins
    x = np.maximum(rnd((2, 8, 11, 12), 9, torch.bfloat16), 0)
    x[:, :, 3:6, 3:6] = 0.0
    for layout in ("NCHW", "NHWC"):
        _pool_case(F, oracle, 0, 1, 2, 11, 12, 2, 8, torch.bfloat16, layout, "max", 0, data=x)
        _pool_case(F, oracle, 0, 1, 1, 11, 12, 2, 8, torch.bfloat16, layout, "max", 0, data=x)


@pytest.mark.parametrize("pi", [0, 1])
def test_pool_n1s2_nchw_f32_pairs(F, oracle, pi):
    # the fp32 NCHW n = 1, s = 2 output-pair forward (W % 4 == 0, float4 row loads; pool_nchw.cu) and its
    # backward: top / bottom / left edges, odd and even H, ReLU-like data with exact-zero ties (first
    # in-grid tap wins), several planes
    for k, (H, W) in enumerate([(11, 12), (12, 8), (2, 4), (40, 40), (9, 48)]):
        x = np.maximum(rnd((2, 3, H, W), 30 + k, torch.float32), 0)
        for mode in ("max", "avg"):
            _pool_case(F, oracle, pi, 1, 2, H, W, 2, 3, torch.float32, "NCHW", mode, 40 + k, data=x)


# ------------------------------------------------------------------ BASELINE configs 1 and 2 at full size
def test_config1_full(F, oracle):
    import synth
    c = synth.CONFIGS["c1"]
    x = synth.round_f32(synth.normal((c["B"], c["Cin"], c["H"], c["W"]), 0))
    w = synth.round_f32(synth.normal((c["Cout"], c["Cin"], 7), 1, 0.1))
    y = F.conv2d_fwd(to_dev(x, torch.float32), to_dev(w, torch.float32), torch.zeros(4, device="cuda"), n=1)
    assert rel(to_np(y), oracle.conv2d_fwd(x, w, np.zeros(4), n=1)) <= TOL_F32
    # the gather map of the config, bit-exact
    assert np.array_equal(F.gather_map(16, 16, 1).cpu().numpy(), oracle.gather_map(16, 16, 1, 1))


def test_config2_full(F, oracle):
    import synth
    c = synth.CONFIGS["c2"]
    B, Ci, Co, H, W = c["B"], c["Cin"], c["Cout"], c["H"], c["W"]
    x = synth.round_f32(synth.normal((B, Ci, H, W), 0))
    w = synth.round_f32(synth.kaiming_uniform((Co, Ci, 19), 1))
    xd, wd = to_dev(x, torch.float32), to_dev(w, torch.float32)
    y = F.conv2d_fwd(xd, wd, None, n=2, stride=2)
    yref = oracle.conv2d_fwd(x, w, None, n=2, s=2)
    assert y.shape == (32, 32, 24, 24)
    assert rel(to_np(y), yref) <= TOL_F32
    # max pool n1 s2 on the GPU's own conv output (reading A17)
    y64 = to_np(y)
    p, am = F.pool2d_fwd(y, n=1, stride=2, mode="max")
    pref, amref = oracle.pool2d_fwd(y64, n=1, s=2, mode="max")
    assert p.shape == (32, 32, 12, 12)
    assert np.array_equal(to_np(p), pref) and np.array_equal(am.cpu().numpy(), amref)
    gp = synth.round_f32(synth.normal(pref.shape, 3))
    gy = F.pool2d_bwd(to_dev(gp, torch.float32), am, (24, 24), n=1, stride=2, mode="max")
    gyref = oracle.pool2d_bwd(gp, amref, 24, 24, n=1, s=2, mode="max")
    assert rel(to_np(gy), gyref) <= TOL_F32
    gy64 = to_np(gy)
    dx = F.conv2d_bwd_data(gy, wd, (H, W), n=2, stride=2)
    dw, db = F.conv2d_bwd_weight(xd, gy, n=2, stride=2)
    dxr, dwr, dbr = oracle.conv2d_bwd(x, w, gy64, n=2, s=2)
    assert rel(to_np(dx), dxr) <= TOL_F32
    assert rel(dw.cpu().numpy(), dwr) <= TOL_F32
    assert rel(db.cpu().numpy(), dbr) <= TOL_F32


def test_single_input_channel_bf16_nhwc(F, oracle):
    # the Cin = 1 stencil kernels (config 5 layer 1): both n, both parities, strides 1 and 2, ragged grids
    for pi, n, s, (H, W), Cout in [(0, 2, 1, (13, 11), 64), (1, 1, 1, (9, 12), 128), (0, 2, 2, (12, 13), 64),
                                   (1, 2, 2, (11, 10), 64)]:
        _conv_case(F, oracle, pi, n, s, H, W, 3, 1, Cout, torch.bfloat16, "NHWC", 40 + n)


@pytest.mark.parametrize("pi,n", [(0, 2), (1, 2), (0, 1), (1, 1)])
def test_single_input_channel_mma_bands(F, oracle, pi, n):
    # the stride-1 Cin = 1 tensor-core kernels (smallc_mma.cu): several 16-row bands with a ragged
    # last band, ragged 16-pixel items (W % 16 != 0), two 64-channel blocks, both parities
    # (W % 8 == 0 takes the bulk-copy band staging; B * bands > 2 * 148 makes the persistent blocks loop;
    # the host picks the band height so the last round is nearly full: 10 rows at B = 120 / H = 40, and
    # at B = 100 / H = 47 10 rows with a ragged 7-row last band)
    for (H, W), Cout, B in [((37, 45), 128, 3), ((16, 16), 64, 2), ((5, 70), 64, 1), ((35, 40), 64, 2),
                            ((40, 24), 64, 120), ((47, 24), 64, 100)]:
        _conv_case(F, oracle, pi, n, 1, H, W, B, 1, Cout, torch.bfloat16, "NHWC", 60 + n + H)


@pytest.mark.parametrize("pi,n", [(0, 1), (1, 1), (0, 2), (1, 2)])
def test_single_input_channel_f32_bands(F, oracle, pi, n):
    # the fp32 NCHW Cin = 1 kernels (config 3 layer 1, plane_kernels.cu c1_*): several bands per image with
    # a ragged last band, channel groups of 8 (n = 1) / 4 (n = 2) with a ragged and an empty group
    # (Cout = 20), rows wider than a 128-thread group (W = 150), more bands than persistent
    # weight-gradient blocks (B = 300), both parities
    for (B, H, W, Cout) in [(3, 37, 45, 16), (2, 40, 40, 20), (1, 5, 150, 8), (300, 9, 7, 8)]:
        _conv_case(F, oracle, pi, n, 1, H, W, B, 1, Cout, torch.float32, "NCHW", 700 + H + Cout)


@pytest.mark.parametrize("pi,n", [(0, 1), (1, 1), (0, 2), (1, 2)])
def test_f32_mid_channel_wgrad(F, oracle, pi, n):
    # the column-walking fp32 weight gradient (f32_wgrad.cu): ragged 8-row bands (H = 13), odd W,
    # one and two output-channel tiles, many bands per persistent block (B = 40)
    for (B, Cin, Cout, H, W) in [(3, 16, 32, 13, 11), (2, 32, 64, 9, 10), (40, 8, 16, 16, 7)]:
        _conv_case(F, oracle, pi, n, 1, H, W, B, Cin, Cout, torch.float32, "NCHW", 500 + Cin + H)


def test_maxpool_n1s2_closed_form_backward(F, oracle):
    # the specialised n=1, s=2 max-pool backward (config 5): both parities, odd/even grids, C % 8 == 0
    for pi in (0, 1):
        for (H, W) in [(12, 13), (13, 12), (9, 9), (2, 7)]:
            for C in (8, 24):
                _pool_case(F, oracle, pi, 1, 2, H, W, 2, C, torch.bfloat16, "NHWC", "max", 400 + H + C)


@pytest.mark.parametrize("n", [4, 5, 7])
def test_conv_pool_largest_kernels(F, oracle, n):
    # the largest kernel sizes the ABI accepts (HEX_MAX_N = 7: T = 169 taps) on grids smaller and
    # larger than the kernel, strides 1 and 2, both parities; pooling up to the uint8 argmax range
    for k, (pi, s, H, W) in enumerate([(0, 1, 9, 11), (1, 2, 20, 17), (0, 3, 4, 3)]):
        _conv_case(F, oracle, pi, n, s, H, W, 1, 2, 3, torch.float32, "NCHW", 900 + 10 * n + k)
        for mode in ("max", "avg", "avg_pad"):
            _pool_case(F, oracle, pi, n, s, H, W, 2, 3, torch.float32, "NCHW", mode, 950 + 10 * n + k)


def test_degenerate_and_invalid_shapes(F, oracle):
    from paper_1903_01814_b200._abi import HexError
    # 1 x 1 grid (every tap off-grid but the centre) and a single column
    _conv_case(F, oracle, 0, 2, 1, 1, 1, 2, 3, 4, torch.float32, "NCHW", 990)
    _conv_case(F, oracle, 1, 1, 1, 7, 1, 1, 2, 2, torch.float32, "NCHW", 991)
    _pool_case(F, oracle, 0, 1, 1, 1, 1, 1, 2, torch.float32, "NCHW", "max", 992)
    x = torch.zeros(1, 2, 5, 5, device="cuda")
    w = torch.zeros(3, 2, 7, device="cuda")
    with pytest.raises(HexError) as e:  # kernel size beyond HEX_MAX_N
        F.conv2d_fwd(x, torch.zeros(3, 2, 3 * 8 * 9 + 1, device="cuda"), n=8)
    assert e.value.status == 8  # HEX_ERR_UNSUPPORTED
    with pytest.raises(HexError) as e:  # empty stride lattice: H = 1 with s = 2 leaves the odd columns empty
        F.conv2d_fwd(torch.zeros(1, 2, 1, 5, device="cuda"), w, n=1, stride=2)
    assert e.value.status == 3  # HEX_ERR_EMPTY_LATTICE
    with pytest.raises(HexError):  # zero batch
        F.conv2d_fwd(torch.zeros(0, 2, 5, 5, device="cuda"), w, n=1)
    with pytest.raises(ValueError):  # channel mismatch is caught before the ABI
        F.conv2d_fwd(x, torch.zeros(3, 4, 7, device="cuda"), n=1)


def test_custom_ring_kernel_smoothing(F, oracle):
    # a user-defined kernel: 7-cell mean smoothing via ring_kernel; the GPU result
    # equals the oracle convolution with the same weights, and a constant image stays constant inside
    x = rnd((2, 1, 11, 12), 1200, torch.float32)
    k = F.ring_kernel([1.0 / 7, 1.0 / 7])
    y = F.conv2d_fwd(torch.from_numpy(x.astype(np.float32)).cuda(), k, None, n=1)
    assert rel(to_np(y), oracle.conv2d_fwd(x, k.cpu().numpy().astype(np.float64), None, n=1)) <= TOL_F32
    yc = F.conv2d_fwd(torch.full((1, 1, 9, 9), 3.5, device="cuda"), k, None, n=1)
    assert torch.allclose(yc[0, 0, 1:-1, 1:-1], torch.tensor(3.5, device="cuda"), atol=1e-6)
    # an edge detector from a dict of axial displacements: zero response on a constant image interior
    e = F.custom_kernel(1, {(0, 0): 6.0, (0, -1): -1.0, (0, 1): -1.0, (1, 0): -1.0, (-1, 0): -1.0,
                            (1, -1): -1.0, (-1, 1): -1.0})
    ye = F.conv2d_fwd(torch.full((1, 1, 9, 9), 2.0, device="cuda"), e, None, n=1)
    assert ye[0, 0, 1:-1, 1:-1].abs().max().item() == 0.0


@pytest.mark.parametrize("s", [2, 3])
@pytest.mark.parametrize("pi", [0, 1])
def test_conv_strided_tensor_core_forward(F, oracle, s, pi):
    # bf16 NHWC stride 2 and 3: the forward runs the tcgen05 kernel with element-stride-s
    # input boxes per output column-parity class (lattice_box)
    for k, (B, Cin, Cout, H, W, n) in enumerate([(2, 64, 64, 20, 23, 1), (1, 128, 256, 31, 30, 2),
                                                  (3, 64, 128, 9, 8, 1), (1, 64, 64, 5 + 3 * (s - 2), 6, 2),
                                                  (1, 64, 64, 26, 25, 3), (2, 64, 64, 3, 4, 1), (1, 128, 64, 4, 5, 2)]):
        assert F.conv_algo(B, Cin, Cout, H, W, n, s, pi, torch.bfloat16, "NHWC", 0) == "tcgen05"
        _conv_case(F, oracle, pi, n, s, H, W, B, Cin, Cout, torch.bfloat16, "NHWC", 1300 + 10 * s + k)


@pytest.mark.parametrize("s", [2, 3])
def test_conv_strided_tensor_core_backward(F, oracle, s):
    # strided backward passes (f4): the stride-1 tcgen05 bwd-data / wgrad on dy scattered onto the full
    # grid (strided.cu; pin P10: a strided conv is the stride-1 conv sampled at the lattice centres)
    for k, (B, Cin, Cout, H, W, n, pi) in enumerate([(2, 64, 128, 20, 23, 1, 0), (1, 128, 128, 17, 16, 2, 1),
                                                      (2, 64, 128, 9, 12, 1, 1)]):
        assert F.conv_algo(B, Cin, Cout, H, W, n, s, pi, torch.bfloat16, "NHWC", 1) == "tcgen05"
        assert F.conv_algo(B, Cin, Cout, H, W, n, s, pi, torch.bfloat16, "NHWC", 2) == "tcgen05"
        _conv_case(F, oracle, pi, n, s, H, W, B, Cin, Cout, torch.bfloat16, "NHWC", 1400 + 10 * s + k)


@pytest.mark.parametrize("s", [2, 3])
@pytest.mark.parametrize("pi", [0, 1])
def test_strided_bwd_data_phase_classes(F, oracle, s, pi):
    # strided bf16 NHWC bwd-data by phase classes (lat_dgrad.cu, f4): only the lattice taps are multiplied;
    # against the oracle (fused ReLU-backward mask included) and against the upsampled route it replaces
    from paper_1903_01814_b200 import _abi as A
    import synth
    for k, (B, Cin, Cout, H, W, n) in enumerate([(2, 64, 128, 21, 22, 1), (1, 128, 64, 17, 19, 2),
                                                  (2, 256, 48, 12, 13, 3)]):
        T = oracle.num_taps(n)
        Ho, Wo, _ = oracle.out_shape(H, W, s, pi)
        g = synth.round_bf16(synth.normal((B, Cout, Ho, Wo), 1500 + k))
        w = synth.round_bf16(synth.normal((Cout, Cin, T), 1510 + k, 1.0 / np.sqrt(Cout * T)))
        m = synth.round_bf16(synth.normal((B, Cin, H, W), 1520 + k))
        gd, md = to_dev(g, torch.bfloat16, "NHWC"), to_dev(m, torch.bfloat16, "NHWC")
        wd = torch.from_numpy(w.astype(np.float32)).to(torch.bfloat16).cuda()
        x0 = np.zeros((B, Cin, H, W))
        dxr, _, _ = oracle.conv2d_bwd(x0, w, g, n=n, s=s, pi=pi)
        dx = F.conv2d_bwd_data(gd, wd, (H, W), n=n, stride=s, parity=pi, layout="NHWC")
        assert rel(to_np(dx, "NHWC"), dxr) <= TOL_BF16, (s, pi, k)
        dxm = F.conv2d_bwd_data(gd, wd, (H, W), n=n, stride=s, parity=pi, layout="NHWC", relu_y=md)
        assert rel(to_np(dxm, "NHWC"), dxr * (m > 0)) <= TOL_BF16, (s, pi, k, "mask")
        if Cout % 8 == 0 and Cin % 64 == 0 and Cout % 64 == 0:
            with A.switch("HEXCONV_NO_LAT_DGRAD"):
                dxu = F.conv2d_bwd_data(gd, wd, (H, W), n=n, stride=s, parity=pi, layout="NHWC", relu_y=md)
            assert rel(to_np(dxm, "NHWC"), to_np(dxu, "NHWC")) <= 1e-2


@pytest.mark.parametrize("s", [2, 3])
@pytest.mark.parametrize("pi", [0, 1])
def test_strided_wgrad_on_the_lattice(F, oracle, s, pi):
    # strided (s = 2, 3) bf16 weight gradient walking the dy lattice directly (x boxes with element stride s;
    # f4): against the oracle, and within fp32 summation order of the scattered-dy route it replaces
    from paper_1903_01814_b200 import _abi as A
    import synth
    for k, (B, Cin, Cout, H, W, n) in enumerate([(2, 64, 128, 21, 22, 1), (1, 128, 256, 17, 19, 2),
                                                  (3, 64, 128, 9, 8, 1), (1, 64, 128, 26, 27, 3),
                                                  (2, 64, 128, 3, 4, 1), (1, 128, 128, 4, 5, 2)]):
        T = oracle.num_taps(n)
        Ho, Wo, _ = oracle.out_shape(H, W, s, pi)
        x = synth.round_bf16(synth.normal((B, Cin, H, W), 1600 + 10 * s + k))
        g = synth.round_bf16(synth.normal((B, Cout, Ho, Wo), 1610 + 10 * s + k))
        xd, gd = to_dev(x, torch.bfloat16, "NHWC"), to_dev(g, torch.bfloat16, "NHWC")
        assert F.conv_algo(B, Cin, Cout, H, W, n, s, pi, torch.bfloat16, "NHWC", 2) == "tcgen05"
        dw, db = F.conv2d_bwd_weight(xd, gd, n=n, stride=s, parity=pi, layout="NHWC")
        _, dwr, dbr = oracle.conv2d_bwd(x, np.zeros((Cout, Cin, T)), g, n=n, s=s, pi=pi)
        assert rel(dw.cpu().numpy(), dwr) <= 1e-4, (s, pi, k)
        assert rel(db.cpu().numpy(), dbr) <= 1e-4, (s, pi, k)
        with A.switch("HEXCONV_NO_TC_WGRAD_LAT"):
            dwu, dbu = F.conv2d_bwd_weight(xd, gd, n=n, stride=s, parity=pi, layout="NHWC")
        assert rel(dw.cpu().numpy(), dwu.cpu().numpy().astype(np.float64)) <= 1e-5
