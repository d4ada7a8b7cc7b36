"""BASELINE config 4 at full size -- the launch configuration bench.py's secondary
C4 line times: batch 128, Cin = Cout = 256, 64x64 offset grid, n = 1 and n = 2,
stride 1, bf16 NHWC inputs N(0,1), weights N(0, 1/sqrt(Cin*T)), fp32
accumulation (PAPER.md:144-151, 166-168 define the convolution).

* forward and backward-data: the whole batch runs on the GPU; images 0 and 127
  (first and last; images are independent) are compared element by element
  with the fp64 oracle at the bf16 tolerance 2e-2 (normwise, reading A14);
* weight gradient + dbias: the full 128-image reduction (K = 524,288 pixels)
  is compared at sampled (co, ci, t) points with the oracle's point
  evaluation over all 128 images, and dbias with an fp64 sum.
Each pass is asserted to run on the tcgen05 kernels.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

B, C, H, W = 128, 256, 64, 64
IMGS = [0, B - 1]
TOL = 2e-2


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def data():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import synth
    x = torch.from_numpy(synth.normal((B, H, W, C), 40).astype(np.float32)).to(torch.bfloat16).cuda()
    g = torch.from_numpy(synth.normal((B, H, W, C), 41).astype(np.float32)).to(torch.bfloat16).cuda()
    return x, g


def f64_nchw(t):
    return t.float().permute(0, 3, 1, 2).cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("n", [1, 2])
def test_c4_full_size(data, oracle, n):
    import synth
    from paper_1903_01814_b200 import functional as F
    x, g = data
    T = F.num_taps(n)
    for pass_id in (0, 1, 2):
        assert F.conv_algo(B, C, C, H, W, n, 1, 0, torch.bfloat16, "NHWC", pass_id) == "tcgen05"
    w = torch.from_numpy(synth.normal((C, C, T), 42 + n, 1.0 / np.sqrt(C * T)).astype(np.float32)
                         ).to(torch.bfloat16).cuda()
    wf = w.float().cpu().numpy().astype(np.float64)
    y = F.conv2d_fwd(x, w, None, n=n, layout="NHWC")
    dx = F.conv2d_bwd_data(g, w, (H, W), n=n, layout="NHWC")
    dw, db = F.conv2d_bwd_weight(x, g, n=n, layout="NHWC")
    torch.cuda.synchronize()

    xs, gs = f64_nchw(x[IMGS]), f64_nchw(g[IMGS])
    assert rel(f64_nchw(y[IMGS]), oracle.conv2d_fwd(xs, wf, None, n=n)) <= TOL, "fwd"
    dxr, _, _ = oracle.conv2d_bwd(xs, wf, gs, n=n, need=("dx",))
    assert rel(f64_nchw(dx[IMGS]), dxr) <= TOL, "dgrad"

    rng = np.random.default_rng(n)
    pts = np.stack([rng.integers(0, C, 32), rng.integers(0, C, 32), rng.integers(0, T, 32)], 1)
    xb = x.view(torch.int16).cpu().numpy().view(np.uint16)
    gb = g.view(torch.int16).cpu().numpy().view(np.uint16)
    ref = oracle.conv2d_bwd_weight_at(xb, gb, pts, n=n, layout="NHWC")
    got = dw.cpu().numpy()[pts[:, 0], pts[:, 1], pts[:, 2]]
    # fp32 sums of exact bf16 products over 524,288 pixels: normwise 1e-3 (as tests/test_gpu_tc.py)
    assert np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30) <= 1e-3, "wgrad"
    db_ref = g.float().double().sum(dim=(0, 1, 2)).cpu().numpy()
    assert rel(db.cpu().numpy(), db_ref) <= 1e-3, "dbias"
