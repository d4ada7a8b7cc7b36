"""The torch.nn modules (paper_1903_01814_b200/nn.py; "adopting the PyTorch-API"):
construction and initialisation on the host, and on the GPU module forward / backward against the oracle
(debug mode = all kernel elements 1)."""
import math

import numpy as np
import pytest
import torch


def test_modules_construct_and_init():
    from paper_1903_01814_b200 import nn as hnn
    torch.manual_seed(0)
    c = hnn.HexConv2d(3, 5, kernel_size=2, stride=2)
    assert tuple(c.weight.shape) == (5, 3, 19) and tuple(c.bias.shape) == (5,)
    lim = math.sqrt(6.0 / (3 * 19))
    assert float(c.weight.detach().abs().max()) <= lim and float(c.bias.detach().abs().max()) == 0.0
    d = hnn.HexConv2d(2, 4, kernel_size=1, debug=True, bias=False)
    assert d.bias is None and torch.equal(d.weight, torch.ones(4, 2, 7))
    c3 = hnn.HexConv3d(2, 3, kernel_size=1, kernel_depth=3)
    assert tuple(c3.weight.shape) == (3, 2, 3, 7)
    with pytest.raises(ValueError):
        hnn.HexConv3d(2, 3, kernel_size=1, kernel_depth=2)
    with pytest.raises(ValueError):
        hnn.HexMaxPool2d(kernel_size=0)
    assert len(list(c.parameters())) == 2 and "kernel_size=2" in repr(c)


@pytest.mark.gpu
def test_module_net_matches_oracle(oracle):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import synth
    from paper_1903_01814_b200 import nn as hnn
    B, H, W = 2, 12, 13
    net = torch.nn.Sequential(hnn.HexConv2d(2, 4, kernel_size=1, relu=True), hnn.HexAvgPool2d(1, stride=2),
                              hnn.HexConv2d(4, 3, kernel_size=2)).cuda()
    x = synth.round_f32(synth.normal((B, 2, H, W), 1))
    xd = torch.tensor(x, dtype=torch.float32, device="cuda", requires_grad=True)
    y = net(xd)
    R = synth.round_f32(synth.normal(tuple(y.shape), 2))
    (y * torch.tensor(R, dtype=torch.float32, device="cuda")).sum().backward()
    w1 = net[0].weight.detach().cpu().double().numpy()
    w2 = net[2].weight.detach().cpu().double().numpy()
    a = np.maximum(oracle.conv2d_fwd(x, w1, None, n=1), 0)
    p, _ = oracle.pool2d_fwd(a, n=1, s=2, mode="avg")
    yr = oracle.conv2d_fwd(p, w2, None, n=2)
    rel = lambda g, r: float(np.abs(g - r).max() / np.abs(r).max())
    assert rel(y.detach().cpu().double().numpy(), yr) <= 1e-5
    dp, dw2, db2 = oracle.conv2d_bwd(p, w2, R, n=2)
    assert rel(net[2].weight.grad.cpu().double().numpy(), dw2) <= 1e-5
    assert rel(net[2].bias.grad.cpu().double().numpy(), db2) <= 1e-5
    da = oracle.pool2d_bwd(dp, None, H, W, n=1, s=2, mode="avg") * (a > 0)
    dx, dw1, _ = oracle.conv2d_bwd(x, w1, da, n=1)
    assert rel(net[0].weight.grad.cpu().double().numpy(), dw1) <= 1e-5
    assert rel(xd.grad.cpu().double().numpy(), dx) <= 1e-5


@pytest.mark.gpu
def test_debug_kernel_counts_neighbours(oracle):
    # debug mode (all kernel elements 1) on a constant image: each output is the number of in-grid cells of
    # the centre's hexagonal neighbourhood (SPEC.md:212 conservation, pin P14)
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1903_01814_b200 import nn as hnn
    for n, s, pi in [(1, 1, 0), (2, 2, 1), (3, 1, 1)]:
        m = hnn.HexConv2d(1, 1, kernel_size=n, stride=s, parity=pi, debug=True, bias=False).cuda()
        x = torch.ones(1, 1, 9, 10, device="cuda")
        y = m(x).detach().cpu().double().numpy()
        yr = oracle.conv2d_fwd(np.ones((1, 1, 9, 10)), np.ones((1, 1, 3 * n * (n + 1) + 1)), None, n=n, s=s, pi=pi)
        assert np.array_equal(y, yr)
        assert y.max() == 3 * n * (n + 1) + 1 and y.min() < y.max()
