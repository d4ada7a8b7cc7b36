"""GPU parity of the fp32 3xTF32 tensor-core path (csrc/tf32_conv.cu) against the fp64
oracle: forward at strides 1-3 (lattice PAPER.md:152-154, 172-175) and backward-data
(the adjoint; for s > 1 dy read through the lattice), both parities, n = 1..3, channel counts that are not
multiples of 8 (zero-padded K chunks), output channels not multiples of 16, pixel counts that leave a
ragged last tile and tiles spanning images, fused bias + ReLU, fused ReLU-backward mask.  fp32 bar:
normwise 1e-5 (A14); the routing to the tf32 kernel is asserted, and the FFMA kernels (HEXCONV_NO_TF32)
agree on the same inputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1903_01814_b200 import functional
    return functional


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def np64(t):
    return t.detach().cpu().numpy().astype(np.float64)


CASES = [  # B, Cin, Cout, H, W, n, s, parity
    (2, 16, 32, 11, 12, 2, 1, 0),
    (3, 16, 32, 12, 12, 1, 1, 1),
    (2, 13, 5, 9, 16, 2, 1, 0),      # Cin not a multiple of 8, Cout < 16
    (1, 32, 64, 20, 20, 1, 1, 0),    # config-3 layer-4 shape (one image; 20 columns = 8 + 8 + 4)
    (2, 8, 16, 7, 8, 3, 1, 1),       # n = 3
    (4, 16, 32, 12, 12, 2, 2, 0),    # config-2 shape family, stride 2
    (3, 16, 24, 11, 16, 2, 2, 1),
    (2, 9, 16, 13, 12, 1, 3, 0),     # stride 3
    (5, 8, 48, 5, 8, 1, 1, 0),       # tiles spanning several small images
    (2, 16, 32, 11, 13, 2, 1, 1),    # odd width: the weight gradient takes the FFMA kernel
]


@pytest.mark.parametrize("case", CASES)
def test_tf32_conv_fwd_bwd_data(F, oracle, case):
    import synth
    B, Ci, Co, H, W, n, s, pi = case
    T = F.num_taps(n)
    assert F.conv_algo(B, Ci, Co, H, W, n, s, pi, torch.float32, "NCHW", 0) == "tcgen05-tf32"
    x = synth.round_f32(synth.normal((B, Ci, H, W), 1 + Ci))
    w = synth.round_f32(synth.normal((Co, Ci, T), 2 + Co, 1.0 / np.sqrt(Ci * T)))
    b = synth.round_f32(synth.normal((Co,), 3))
    Ho, Wo, _ = F.output_shape(H, W, s, pi)
    g = synth.round_f32(synth.normal((B, Co, Ho, Wo), 4))
    xd, wd, bd, gd = dev(x), dev(w), dev(b), dev(g)
    y = F.conv2d_fwd(xd, wd, bd, n=n, stride=s, parity=pi)
    yref = oracle.conv2d_fwd(x, w, b, n=n, s=s, pi=pi)
    assert rel(np64(y), yref) <= TOL, "fwd"
    yr = F.conv2d_fwd(xd, wd, bd, n=n, stride=s, parity=pi, relu=True)
    assert rel(np64(yr), np.maximum(yref, 0)) <= TOL, "fwd relu"
    if Co >= 8:
        assert F.conv_algo(B, Ci, Co, H, W, n, s, pi, torch.float32, "NCHW", 1) == "tcgen05-tf32"
    dxr, _, _ = oracle.conv2d_bwd(x, w, g, n=n, s=s, pi=pi, need=("dx",))
    dx = F.conv2d_bwd_data(gd, wd, (H, W), n=n, stride=s, parity=pi)
    assert rel(np64(dx), dxr) <= TOL, "dgrad"
    dxm = F.conv2d_bwd_data(gd, wd, (H, W), n=n, stride=s, parity=pi, relu_y=xd)
    assert rel(np64(dxm), dxr * (x > 0)) <= TOL, "dgrad masked"
    if (W * 4) % 16 == 0:  # the TMA-staged weight-gradient kernel needs 16-byte row pitch
        assert F.conv_algo(B, Ci, Co, H, W, n, s, pi, torch.float32, "NCHW", 2) == "tcgen05-tf32"
    _, dwr, dbr = oracle.conv2d_bwd(x, w, g, n=n, s=s, pi=pi, need=("dw", "db"))
    dw, db = F.conv2d_bwd_weight(xd, gd, n=n, stride=s, parity=pi)
    assert rel(np64(dw), dwr) <= TOL, "wgrad"
    assert rel(np64(db), dbr) <= TOL, "dbias"
    dw2, db2 = F.conv2d_bwd_weight(xd, gd, n=n, stride=s, parity=pi, dw=dw.clone(), dbias=db.clone(),
                                   accumulate=True)
    assert rel(np64(dw2), 2 * dwr) <= TOL and rel(np64(db2), 2 * dbr) <= TOL, "wgrad accumulate"


def test_tf32_matches_ffma_path(F):
    from paper_1903_01814_b200 import _abi as A
    g = torch.Generator().manual_seed(5)
    x = torch.randn(3, 16, 17, 19, generator=g).cuda()
    w = (torch.randn(32, 16, 19, generator=g) * 0.05).cuda()
    dy = torch.randn(3, 32, 17, 19, generator=g).cuda()
    y1 = F.conv2d_fwd(x, w, None, n=2)
    d1 = F.conv2d_bwd_data(dy, w, (17, 19), n=2)
    with A.switch("HEXCONV_NO_TF32"):
        assert F.conv_algo(3, 16, 32, 17, 19, 2, 1, 0, torch.float32, "NCHW", 0) == "stencil"
        y2 = F.conv2d_fwd(x, w, None, n=2)
        d2 = F.conv2d_bwd_data(dy, w, (17, 19), n=2)
    assert (y1 - y2).abs().max().item() <= 1e-5 * y2.abs().max().item()
    assert (d1 - d2).abs().max().item() <= 1e-5 * d2.abs().max().item()


def test_tf32_deterministic(F):
    x = torch.randn(4, 16, 20, 20, device="cuda")
    w = torch.randn(32, 16, 7, device="cuda")
    a = F.conv2d_fwd(x, w, None, n=1)
    b = F.conv2d_fwd(x, w, None, n=1)
    assert torch.equal(a, b)

