"""GPU parity of the tcgen05 tensor-core path (bf16 NHWC, stride 1) against the
fp64 oracle fed the same bf16-rounded inputs.  Tolerance 2e-2 normwise for
bf16 outputs (north_star); weight gradients are fp32 sums of exact bf16
products, checked at 1e-3 normwise (fp32 accumulation over up to ~1e5 terms).
Each case asserts the library actually routed it to the tensor-core kernels.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
TOL_WGRAD = 1e-3


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1903_01814_b200 import functional
    return functional


def rel(gpu, ref):
    return float(np.abs(np.asarray(gpu, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def nhwc(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).permute(0, 2, 3, 1).contiguous().to(
        torch.bfloat16).cuda()


def back(t):
    return t.float().permute(0, 3, 1, 2).cpu().numpy().astype(np.float64)


def case(F, oracle, B, Cin, Cout, H, W, n, pi, seed, relu=False, bias=True):
    import synth
    T = oracle.num_taps(n)
    x = synth.round_bf16(synth.normal((B, Cin, H, W), seed))
    w = synth.round_bf16(synth.normal((Cout, Cin, T), seed + 1, 1.0 / np.sqrt(Cin * T)))
    b = synth.round_f32(synth.normal((Cout,), seed + 2)) if bias else None
    g = synth.round_bf16(synth.normal((B, Cout, H, W), seed + 3))
    for pass_id in (0, 1, 2):
        if pass_id == 2 and Cout % 128:
            continue  # the tcgen05 weight-gradient kernel tiles Cout by 128 (stencil path otherwise)
        assert F.conv_algo(B, Cin, Cout, H, W, n, 1, pi, torch.bfloat16, "NHWC", pass_id) == "tcgen05"
    xd, gd = nhwc(x), nhwc(g)
    wd = torch.from_numpy(w.astype(np.float32)).to(torch.bfloat16).cuda()
    bd = None if b is None else torch.from_numpy(b.astype(np.float32)).cuda()
    y = F.conv2d_fwd(xd, wd, bd, n=n, parity=pi, relu=relu, layout="NHWC")
    yref = oracle.conv2d_fwd(x, w, b, n=n, pi=pi)
    if relu:
        yref = np.maximum(yref, 0)
    assert rel(back(y), yref) <= TOL_BF16, ("fwd", B, Cin, Cout, H, W, n, pi)
    dxr, dwr, dbr = oracle.conv2d_bwd(x, w, g, n=n, pi=pi)
    dx = F.conv2d_bwd_data(gd, wd, (H, W), n=n, parity=pi, layout="NHWC")
    assert rel(back(dx), dxr) <= TOL_BF16, ("dgrad", B, Cin, Cout, H, W, n, pi)
    # fused ReLU-backward mask in the dgrad epilogue
    dxm = F.conv2d_bwd_data(gd, wd, (H, W), n=n, parity=pi, layout="NHWC", relu_y=xd)
    assert rel(back(dxm), dxr * (x > 0)) <= TOL_BF16
    dw, db = F.conv2d_bwd_weight(xd, gd, n=n, parity=pi, layout="NHWC")
    assert rel(dw.cpu().numpy(), dwr) <= TOL_WGRAD, ("wgrad", B, Cin, Cout, H, W, n, pi)
    assert rel(db.cpu().numpy(), dbr) <= TOL_WGRAD


@pytest.mark.parametrize("n", [1, 2, 3])
@pytest.mark.parametrize("pi", [0, 1])
def test_tc_small_ragged(F, oracle, n, pi):
    # ragged tiles in every direction: odd W (views of unequal width), H not a box multiple
    case(F, oracle, 3, 64, 128, 13, 11, n, pi, 10 * n + pi)


@pytest.mark.parametrize("Cin,Cout", [(64, 64), (128, 256), (256, 128), (64, 512)])
def test_tc_channel_tiles(F, oracle, Cin, Cout):
    case(F, oracle, 2, Cin, Cout, 10, 12, 1, 0, Cin + Cout, relu=True)


def test_tc_c5_like_shapes(F, oracle):
    # the C5 layer shapes at a small batch (96x96 / 48x48 / 24x24 grids)
    case(F, oracle, 1, 64, 128, 24, 24, 1, 0, 1)
    case(F, oracle, 2, 128, 128, 16, 16, 2, 0, 2)


def test_tc_deterministic(F):
    x = torch.randn(4, 16, 16, 128, device="cuda").to(torch.bfloat16)
    w = (torch.randn(128, 128, 19, device="cuda") * 0.02).to(torch.bfloat16)
    g = torch.randn(4, 16, 16, 128, device="cuda").to(torch.bfloat16)
    assert torch.equal(F.conv2d_fwd(x, w, n=2, layout="NHWC"), F.conv2d_fwd(x, w, n=2, layout="NHWC"))
    a = F.conv2d_bwd_weight(x, g, n=2, layout="NHWC")[0]
    b = F.conv2d_bwd_weight(x, g, n=2, layout="NHWC")[0]
    assert torch.equal(a, b)


def test_tc_matches_stencil_path(F, monkeypatch):
    # same bf16 inputs through both kernel families (fp32 accumulation in both)
    x = torch.randn(2, 12, 14, 64, device="cuda").to(torch.bfloat16)
    w = (torch.randn(64, 64, 7, device="cuda") * 0.05).to(torch.bfloat16)
    y_tc = F.conv2d_fwd(x, w, n=1, layout="NHWC").float()
    xs = x.permute(0, 3, 1, 2).contiguous()
    y_st = F.conv2d_fwd(xs, w, n=1, layout="NCHW").float().permute(0, 2, 3, 1)
    assert (y_tc - y_st).abs().max().item() <= 2e-2 * y_st.abs().max().item()


@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("pi", [0, 1])
def test_tc_tap_reuse_wgrad_shapes(F, oracle, n, pi):
    # shapes the tap-reuse weight-gradient kernel (tc_wgrad_tr.cu) takes: 16-row x 8-sub-column tiles
    # at least 85% filled, here with a ragged last row tile (H = 30) and views of unequal width (W = 31)
    case(F, oracle, 2, 64, 128, 30, 31, n, pi, 100 + 10 * n + pi)


def test_tc_tap_reuse_wgrad_channel_tiles(F, oracle):
    # two Cout tiles x two input-channel chunks (n = 1), and the three n = 2 column groups x two chunks
    case(F, oracle, 1, 128, 256, 16, 16, 1, 0, 7)
    case(F, oracle, 2, 128, 128, 16, 17, 2, 1, 8)
    # CTA-pair forward with an odd number of 128-pixel tiles (the last pair's second tile is empty)
    case(F, oracle, 1, 128, 128, 16, 17, 1, 0, 9)
    case(F, oracle, 1, 256, 256, 16, 17, 2, 1, 10)
    # 2-CTA weight gradient with a short last atom group (24 x 24, n = 1: 28 atoms = 8+8+8+4; the last
    # group gets half the pixel chunks) -- C5 layer 6
    case(F, oracle, 2, 256, 256, 24, 24, 1, 0, 11)


@pytest.mark.parametrize("n", [1])
@pytest.mark.parametrize("pi", [0, 1])
def test_fused_conv_relu_maxpool(F, oracle, n, pi):
    # hex_conv2d_fwd_maxpool: bit-identical to the unfused conv + ReLU + pool, and the
    # pool of the GPU's own conv output matches the oracle pool bit-exactly (values and argmax taps)
    import synth
    # shapes on which the unfused forward also runs the tap-reuse kernel (same fp32 summation order)
    for (B, Cin, Cout, H, W) in [(2, 64, 128, 30, 31), (1, 128, 64, 32, 32), (3, 64, 64, 16, 16)]:
        T = oracle.num_taps(n)
        x = synth.round_bf16(synth.normal((B, Cin, H, W), 70 + H))
        w = synth.round_bf16(synth.normal((Cout, Cin, T), 71 + H, 1.0 / np.sqrt(Cin * T)))
        b = synth.round_f32(synth.normal((Cout,), 72 + H, 0.2))
        xd = nhwc(x)
        wd = torch.from_numpy(w.astype(np.float32)).to(torch.bfloat16).cuda()
        bd = torch.from_numpy(b.astype(np.float32)).cuda()
        assert F.conv2d_fwd_maxpool_supported(B, Cin, Cout, H, W, n, pi)
        yp, am = F.conv2d_fwd_maxpool(xd, wd, bd, n=n, parity=pi)
        yc = F.conv2d_fwd(xd, wd, bd, n=n, parity=pi, relu=True, layout="NHWC")
        yp2, am2 = F.pool2d_fwd(yc, 1, 2, pi, "max", "NHWC")
        torch.cuda.synchronize()
        assert torch.equal(yp.view(torch.int16), yp2.view(torch.int16)), (n, pi, H, W)
        assert torch.equal(am, am2), (n, pi, H, W)
        pr, amr = oracle.pool2d_fwd(back(yc), n=1, s=2, pi=pi, mode="max")
        assert np.array_equal(back(yp), pr)
        assert np.array_equal(am.permute(0, 3, 1, 2).cpu().numpy(), amr)


@pytest.mark.gpu
@pytest.mark.parametrize("pi", [0, 1])
def test_fused_conv_maxpool_strips(F, oracle, pi):
    # batches with >= one strip per SM run the strip-walking mode (rows carried between tiles) plus the
    # region-mode tail; ragged bottom (46 rows), a last tile whose bottom window reaches row H (48 rows).
    import synth
    for (B, Cin, Cout, H, W) in [(25, 64, 128, 46, 96), (25, 64, 64, 48, 90), (44, 128, 64, 32, 48)]:
        T = oracle.num_taps(1)
        g = torch.Generator().manual_seed(900 + H + pi)
        x = (torch.randn(B, H, W, Cin, generator=g)).to(torch.bfloat16).cuda()
        w = (torch.randn(Cout, Cin, T, generator=g) / np.sqrt(Cin * T)).to(torch.bfloat16).cuda()
        b = (0.2 * torch.randn(Cout, generator=g)).cuda()
        assert F.conv2d_fwd_maxpool_supported(B, Cin, Cout, H, W, 1, pi)
        yp, am = F.conv2d_fwd_maxpool(x, w, b, n=1, parity=pi)
        yc = F.conv2d_fwd(x, w, b, n=1, parity=pi, relu=True, layout="NHWC")
        yp2, am2 = F.pool2d_fwd(yc, 1, 2, pi, "max", "NHWC")
        torch.cuda.synchronize()
        assert torch.equal(yp.view(torch.int16), yp2.view(torch.int16)), (pi, B, H, W)
        assert torch.equal(am, am2), (pi, B, H, W)
        # the last image (region-mode tail) against the oracle pool of the GPU conv output
        pr, amr = oracle.pool2d_fwd(back(yc[-1:]), n=1, s=2, pi=pi, mode="max")
        assert np.array_equal(back(yp[-1:]), pr)
        assert np.array_equal(am[-1:].permute(0, 3, 1, 2).cpu().numpy(), amr)


@pytest.mark.parametrize("pi", [0, 1])
def test_fused_conv_maxpool_no_relu_ties(F, oracle, pi):
    # no ReLU and no bias: the window warps take the value of the first tap equal to the maximum
    # (A9); small-integer inputs make many windows tie (several taps with the same value, zeros)
    for (B, Cin, Cout, H, W) in [(2, 64, 128, 30, 31), (3, 64, 64, 16, 16)]:
        g = torch.Generator().manual_seed(950 + H + pi)
        x = torch.randint(-1, 2, (B, H, W, Cin), generator=g).to(torch.bfloat16).cuda()
        w = torch.randint(-1, 2, (Cout, Cin, 7), generator=g).to(torch.bfloat16).cuda()
        yp, am = F.conv2d_fwd_maxpool(x, w, None, n=1, parity=pi, relu=False)
        yc = F.conv2d_fwd(x, w, None, n=1, parity=pi, relu=False, layout="NHWC")
        yp2, am2 = F.pool2d_fwd(yc, 1, 2, pi, "max", "NHWC")
        torch.cuda.synchronize()
        assert torch.equal(yp.view(torch.int16), yp2.view(torch.int16)), (pi, H, W)
        assert torch.equal(am, am2), (pi, H, W)
        pr, amr = oracle.pool2d_fwd(back(yc), n=1, s=2, pi=pi, mode="max")
        assert np.array_equal(back(yp), pr)
        assert np.array_equal(am.permute(0, 3, 1, 2).cpu().numpy(), amr)
        assert (am.float().mean() > 0.5), "expected ties / non-centre maxima"


def test_fused_conv_maxpool_unsupported_shape(F):
    # n = 2 weights do not stay resident next to the fused kernel's buffers: the call reports
    # HEX_ERR_UNSUPPORTED (8) and the caller runs conv + pool separately
    from paper_1903_01814_b200._abi import HexError
    assert not F.conv2d_fwd_maxpool_supported(2, 64, 128, 30, 31, 2, 0)
    x = torch.zeros(2, 30, 31, 64, device="cuda", dtype=torch.bfloat16)
    w = torch.zeros(128, 64, 19, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(HexError) as e:
        F.conv2d_fwd_maxpool(x, w, None, n=2)
    assert e.value.status == 8


@pytest.mark.parametrize("pi", [0, 1])
def test_pack_weights_prepacked_calls_bit_identical(F, pi):
    # hex_conv2d_pack_weights packs several layers / passes in ONE launch; fwd, fwd_maxpool and bwd_data
    # called with w = NULL on those workspaces are bit-identical to the calls that pack per call
    import ctypes
    from paper_1903_01814_b200 import _abi as A
    from paper_1903_01814_b200.functional import _workspace, conv_desc
    L = A.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
    g = torch.Generator().manual_seed(31 + pi)
    layers = [(2, 64, 128, 12, 13, 2), (2, 128, 64, 14, 16, 1)]
    tens, entries = [], []
    for (B, Ci, Co, H, W, n) in layers:
        T = A.num_taps(n)
        d = conv_desc(B, Ci, Co, H, W, n, 1, pi, torch.bfloat16, "NHWC")
        x = torch.randn(B, H, W, Ci, generator=g).to(torch.bfloat16).cuda()
        dy = torch.randn(B, H, W, Co, generator=g).to(torch.bfloat16).cuda()
        w = (torch.randn(Co, Ci, T, generator=g) / np.sqrt(Ci * T)).to(torch.bfloat16).cuda()
        b = (0.1 * torch.randn(Co, generator=g)).cuda()
        ws = [_workspace(d, k, "cuda") for k in (0, 1)]
        tens.append((d, x, dy, w, b, ws))
        for k in (0, 1):
            entries.append((d, k, w.data_ptr(), ws[k][0].data_ptr(), ws[k][1]))

    def run(prepacked):
        outs = []
        for (d, x, dy, w, b, ws) in tens:
            wa = None if prepacked else p(w)
            B, H, W, Ci = x.shape
            Co = dy.shape[-1]
            y = torch.empty(B, H, W, Co, dtype=torch.bfloat16, device="cuda")
            A.check(L.hex_conv2d_fwd(ctypes.byref(d), p(x), wa, p(b), 1, p(y), p(ws[0][0]), ws[0][1], st), "fwd")
            dx = torch.empty_like(x)
            A.check(L.hex_conv2d_bwd_data(ctypes.byref(d), p(dy), wa, p(x), p(dx), p(ws[1][0]), ws[1][1], st), "dgrad")
            outs += [y, dx]
            if L.hex_conv2d_fwd_maxpool_supported(ctypes.byref(d)):
                Ho, Wo, _ = A.output_shape(H, W, 2, pi)
                yp = torch.empty(B, Ho, Wo, Co, dtype=torch.bfloat16, device="cuda")
                am = torch.empty(B, Ho, Wo, Co, dtype=torch.uint8, device="cuda")
                A.check(L.hex_conv2d_fwd_maxpool(ctypes.byref(d), p(x), wa, p(b), 1, p(yp), p(am), p(ws[0][0]),
                                                 ws[0][1], st), "fwd_maxpool")
                outs += [yp, am]
        return outs

    ref = run(False)
    for (d, x, dy, w, b, ws) in tens:
        for k in (0, 1):
            ws[k][0].zero_()
    n0 = A.launch_count()
    A.PackArgs(entries).run(st)
    assert A.launch_count() - n0 == 1  # one launch for every layer and pass
    got = run(True)
    torch.cuda.synchronize()
    assert len(got) == len(ref) and len(ref) >= 5
    for a, r in zip(got, ref):
        assert torch.equal(a.view(torch.uint8), r.view(torch.uint8))


def test_pack_weights_rejects(F):
    import ctypes
    from paper_1903_01814_b200 import _abi as A
    from paper_1903_01814_b200.functional import _workspace, conv_desc
    L = A.lib()
    d32 = conv_desc(2, 16, 32, 8, 8, 1, 1, 0, torch.float32, "NCHW")
    w = torch.zeros(32, 16, 7, device="cuda")
    ws, nb = _workspace(d32, 0, "cuda")
    ws = ws if ws is not None else torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(A.HexError) as e:  # not a bf16 tensor-core pass
        A.PackArgs([(d32, 0, w.data_ptr(), ws.data_ptr(), max(nb, 16))]).run(None)
    assert e.value.status == 8
    x = torch.zeros(2, 16, 8, 8, device="cuda")
    y = torch.zeros(2, 32, 8, 8, device="cuda")
    st = L.hex_conv2d_fwd(ctypes.byref(d32), ctypes.c_void_p(x.data_ptr()), None, None, 0,
                          ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(ws.data_ptr()), nb, None)
    assert st == 1  # w == NULL off the tensor-core path
    assert L.hex_conv2d_pack_weights(17, None, None, None, None, None, None) == 1


@pytest.mark.parametrize("pi", [0, 1])
def test_fused_conv_relu_avgpool(F, oracle, pi):
    # hex_conv2d_fwd_pool(HEX_POOL_AVG) (max/avg pool in the conv epilogue): bit-identical to
    # the unfused conv + ReLU + average pool in strip mode (B = 25: whole rounds of strips) and region mode
    # (B = 2), ragged bottoms and edges (in-grid counts 3..7), and within the bf16 tolerance of the oracle
    # pool of the GPU conv output
    for (B, Cin, Cout, H, W, relu) in [(2, 64, 128, 30, 31, True), (25, 64, 64, 46, 90, True),
                                       (3, 128, 64, 16, 16, False)]:
        g = torch.Generator().manual_seed(980 + H + pi)
        x = torch.randn(B, H, W, Cin, generator=g).to(torch.bfloat16).cuda()
        w = (torch.randn(Cout, Cin, 7, generator=g) / np.sqrt(Cin * 7)).to(torch.bfloat16).cuda()
        b = (0.2 * torch.randn(Cout, generator=g)).cuda()
        assert F.conv2d_fwd_pool_supported(B, Cin, Cout, H, W, 1, pi, mode="avg")
        ya = F.conv2d_fwd_avgpool(x, w, b, n=1, parity=pi, relu=relu)
        yc = F.conv2d_fwd(x, w, b, n=1, parity=pi, relu=relu, layout="NHWC")
        ya2, _ = F.pool2d_fwd(yc, 1, 2, pi, "avg", "NHWC")
        torch.cuda.synchronize()
        assert torch.equal(ya.view(torch.int16), ya2.view(torch.int16)), (pi, B, H, W)
        pr, _ = oracle.pool2d_fwd(back(yc[-1:]), n=1, s=2, pi=pi, mode="avg")
        assert rel(back(ya[-1:]), pr) <= 1e-2
    assert not F.conv2d_fwd_pool_supported(2, 64, 64, 16, 16, 1, pi, mode="avg_pad")
