"""Pins for the 3-D hexagonal convolution oracle (Sec. 2
"Software Functionalities": hexagonal layout in x-y, equidistant z).

Each pin fixes the oracle against something other than itself:
* kd = 1 reduces to the (independently pinned) 2-D oracle slice by slice, and the depth stride
  subsamples slices 0, sd, 2sd, ...;
* a depth impulse through an all-ones n = 0, kd = 3 kernel lands on z-1, z, z+1 only (by hand);
* a separable kernel a[kz] * w2[t] equals the 2-D oracle followed by a zero-padded 1-D depth
  correlation written with numpy;
* the library reduction: torch.nn.functional.conv3d (fp64) with the parity-masked (2n+1)^2 boxes,
  depth padding (kd-1)/2 and depth stride sd, then the in-plane lattice subsample (test-local
  geometry from physical positions), forward and autograd gradients;
* the adjoint identities and central finite differences of the backward.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from test_oracle_pins import masked_box_weights, phys_lattice, rand


def torch_hexconv3d(x, w, b, n, s, sd, pi):
    """x [B,Ci,D,H,W], w [Co,Ci,kd,T] -> hex conv3d via two parity-masked square conv3d + subsample."""
    Co, Ci, kd, T = w.shape
    H, W = x.shape[-2:]
    ys = []
    for p in (0, 1):
        box = torch.stack([masked_box_weights(w[:, :, kz], n, p) for kz in range(kd)], dim=2)
        ys.append(F.conv3d(x, box, bias=b, padding=((kd - 1) // 2, n, n), stride=(sd, 1, 1)))
    colpar = torch.tensor([(c + pi) % 2 for c in range(W)])
    full = torch.where(colpar.view(1, 1, 1, 1, W) == 0, ys[0], ys[1])
    lat = phys_lattice(H, W, s, pi)
    rows = torch.tensor([r for (_, rs) in lat for r in rs]).view(len(lat), -1).T
    cols = torch.tensor([c for (c, _) in lat]).view(1, -1).expand_as(rows)
    return full[:, :, :, rows, cols]


@pytest.mark.parametrize("sd", [1, 2])
def test_kd1_is_per_slice_conv2d(oracle, sd):
    for n, s, pi in [(1, 1, 0), (2, 2, 1), (0, 1, 0)]:
        x = rand((2, 3, 5, 8, 9), 1 + n)
        w = rand((4, 3, 1, oracle.num_taps(n)), 2 + n)
        b = rand((4,), 3)
        y = oracle.conv3d_fwd(x, w, b, n=n, s=s, sd=sd, pi=pi)
        assert y.shape[2] == (5 - 1) // sd + 1
        for zo in range(y.shape[2]):
            y2 = oracle.conv2d_fwd(x[:, :, sd * zo], w[:, :, 0], b, n=n, s=s, pi=pi)
            np.testing.assert_allclose(y[:, :, zo], y2, rtol=0, atol=1e-12)


def test_depth_impulse_all_ones(oracle):
    # n = 0, kd = 3, all-ones weights, s = sd = 1: y[z] = x[z-1] + x[z] + x[z+1] (zero padded)
    x = np.zeros((1, 1, 6, 4, 5))
    x[0, 0, 2] = 2.5
    y = oracle.conv3d_fwd(x, np.ones((1, 1, 3, 1)), None, n=0)
    nz = sorted({int(z) for z in np.argwhere(y[0, 0] != 0)[:, 0]})
    assert nz == [1, 2, 3]
    assert np.all(y[0, 0, 1:4] == 2.5)
    # at the depth boundary only the in-range slices count (zero padding in depth, A4)
    x = np.zeros((1, 1, 4, 3, 3))
    x[0, 0, 0] = 1.0
    y = oracle.conv3d_fwd(x, np.ones((1, 1, 5, 1)), None, n=0)
    assert np.all(y[0, 0, :3] == 1.0) and np.all(y[0, 0, 3] == 0.0)


def test_separable_kernel_is_depth_corr_of_conv2d(oracle):
    n, s, sd, pi, kd = 1, 1, 2, 1, 3
    x = rand((2, 2, 7, 6, 7), 10)
    a = rand((kd,), 11)
    w2 = rand((3, 2, oracle.num_taps(n)), 12)
    w = a[None, None, :, None] * w2[:, :, None, :]
    y = oracle.conv3d_fwd(x, w, None, n=n, s=s, sd=sd, pi=pi)
    per = np.stack([oracle.conv2d_fwd(x[:, :, z], w2, None, n=n, s=s, pi=pi) for z in range(7)], axis=2)
    per = np.pad(per, ((0, 0), (0, 0), (1, 1), (0, 0), (0, 0)))  # zero depth padding
    ref = np.stack([sum(a[k] * per[:, :, sd * zo + k] for k in range(kd)) for zo in range(y.shape[2])], axis=2)
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("pi", [0, 1])
@pytest.mark.parametrize("n,s,sd,kd", [(1, 1, 1, 3), (2, 2, 2, 3), (1, 3, 1, 5), (0, 1, 3, 1)])
def test_library_reduction_torch_conv3d(oracle, n, s, sd, kd, pi):
    H, W, D = 9, 10, 6
    xn = rand((2, 3, D, H, W), 20 + n)
    wn = rand((4, 3, kd, oracle.num_taps(n)), 21 + s)
    bn = rand((4,), 22)
    y = oracle.conv3d_fwd(xn, wn, bn, n=n, s=s, sd=sd, pi=pi)
    x = torch.tensor(xn, requires_grad=True)
    w = torch.tensor(wn, requires_grad=True)
    b = torch.tensor(bn, requires_grad=True)
    yt = torch_hexconv3d(x, w, b, n, s, sd, pi)
    np.testing.assert_allclose(y, yt.detach().numpy(), rtol=0, atol=1e-12)
    g = rand(y.shape, 23)
    yt.backward(torch.tensor(g))
    dx, dw, db = oracle.conv3d_bwd(xn, wn, g, n=n, s=s, sd=sd, pi=pi)
    np.testing.assert_allclose(dx, x.grad.numpy(), atol=1e-11)
    np.testing.assert_allclose(dw, w.grad.numpy(), atol=1e-11)
    np.testing.assert_allclose(db, b.grad.numpy(), atol=1e-11)


def test_adjoint_and_finite_differences(oracle):
    rng = np.random.default_rng(30)
    n, s, sd, pi = 1, 2, 2, 0
    x = rng.standard_normal((1, 2, 5, 6, 7))
    w = rng.standard_normal((2, 2, 3, 7))
    y = oracle.conv3d_fwd(x, w, None, n=n, s=s, sd=sd, pi=pi)
    g = rng.standard_normal(y.shape)
    dx, dw, db = oracle.conv3d_bwd(x, w, g, n=n, s=s, sd=sd, pi=pi)
    # <conv(x), g> = <x, dgrad(g)> = <w, wgrad(x, g)> (linearity in x and in w)
    assert abs((y * g).sum() - (x * dx).sum()) < 1e-10
    assert abs((y * g).sum() - (w * dw).sum()) < 1e-10
    assert abs(db.sum() - g.sum()) < 1e-10
    L = lambda xx, ww: (oracle.conv3d_fwd(xx, ww, None, n=n, s=s, sd=sd, pi=pi) * g).sum()
    h = 1e-6
    for _ in range(8):
        i = tuple(rng.integers(0, d) for d in x.shape)
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        assert abs((L(xp, w) - L(xm, w)) / (2 * h) - dx[i]) <= 1e-6 * max(1.0, abs(dx[i]))
        j = tuple(rng.integers(0, d) for d in w.shape)
        wp, wm = w.copy(), w.copy()
        wp[j] += h
        wm[j] -= h
        assert abs((L(x, wp) - L(x, wm)) / (2 * h) - dw[j]) <= 1e-6 * max(1.0, abs(dw[j]))


def test_errors(oracle):
    with pytest.raises(ValueError):
        oracle.conv3d_fwd(np.zeros((1, 1, 4, 3, 3)), np.zeros((1, 1, 2, 7)), None, n=1)  # even kd
    with pytest.raises(ValueError):
        oracle.conv3d_out_depth(4, 3, 0)
    assert oracle.conv3d_out_depth(7, 3, 2) == 4 and oracle.conv3d_out_depth(1, 5, 3) == 1
