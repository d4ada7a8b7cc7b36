"""BASELINE config 3 at full size: 256 Cherenkov-camera-like images on the
40x40 offset grid, the 4-layer fp32 hex CNN (n1 conv 1->16, n2 conv 16->32,
hex avg-pool n1 stride 2, n1 conv 32->64, ReLU after each conv), forward and
backward through the C ABI.  Every layer is checked against the fp64 oracle
fed the GPU's own inputs of that layer (reading A17): forward, pool and
backward-data on sampled images, weight gradients at sampled points summed
over the whole batch, dbias over the whole batch.  fp32 bar: normwise 1e-5.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL = 1e-5
IMGS = [0, 131, 255]


def np64(t, idx=None):
    t = t if idx is None else t[idx]
    return t.detach().cpu().numpy().astype(np.float64)


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def run():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import synth
    from paper_1903_01814_b200 import functional as F
    c = synth.CONFIGS["c3"]
    B, H, W = c["B"], c["H"], c["W"]
    x = torch.from_numpy(synth.shower_images(B, H, W, c["R"], 3).astype(np.float32)).cuda()
    convs = [(1, 16, 1), (16, 32, 2), (32, 64, 1)]
    ws = [torch.from_numpy(synth.kaiming_uniform((co, ci, synth_taps(n)), 20 + i).astype(np.float32)).cuda()
          for i, (ci, co, n) in enumerate(convs)]
    bs = [torch.from_numpy(synth.normal((co,), 30 + i, 0.1).astype(np.float32)).cuda()
          for i, (ci, co, n) in enumerate(convs)]
    r = {"F": F, "x": x, "w": ws, "b": bs, "ns": [n for _, _, n in convs]}
    # forward
    y1 = F.conv2d_fwd(x, ws[0], bs[0], n=1, relu=True)
    y2 = F.conv2d_fwd(y1, ws[1], bs[1], n=2, relu=True)
    p, _ = F.pool2d_fwd(y2, n=1, stride=2, mode="avg")
    y4 = F.conv2d_fwd(p, ws[2], bs[2], n=1, relu=True)
    # backward from g4 = dL/dy4 (post-ReLU)
    g4 = torch.from_numpy(synth.normal(tuple(y4.shape), 40).astype(np.float32)).cuda()
    dy4 = g4 * (y4 > 0)
    dp = F.conv2d_bwd_data(dy4, ws[2], p.shape[-2:], n=1)
    dy2 = F.pool2d_bwd(dp, None, (H, W), n=1, stride=2, mode="avg") * (y2 > 0)
    dy1 = F.conv2d_bwd_data(dy2, ws[1], (H, W), n=2, relu_y=y1)
    grads = [F.conv2d_bwd_weight(x, dy1, n=1), F.conv2d_bwd_weight(y1, dy2, n=2),
             F.conv2d_bwd_weight(p, dy4, n=1)]
    torch.cuda.synchronize()
    r.update(y1=y1, y2=y2, p=p, y4=y4, dy4=dy4, dp=dp, dy2=dy2, dy1=dy1, grads=grads)
    return r


def synth_taps(n):
    return 3 * n * (n + 1) + 1


def test_c3_forward_layers(run, oracle):
    w = [np64(t) for t in run["w"]]
    b = [np64(t) for t in run["b"]]
    ins = [run["x"], run["y1"], run["p"]]
    outs = [run["y1"], run["y2"], run["y4"]]
    for i in range(3):
        ref = np.maximum(oracle.conv2d_fwd(np64(ins[i], IMGS), w[i], b[i], n=run["ns"][i]), 0)
        assert rel(np64(outs[i], IMGS), ref) <= TOL, f"conv{i + 1} fwd"
    pref, _ = oracle.pool2d_fwd(np64(run["y2"], IMGS), n=1, s=2, mode="avg")
    assert rel(np64(run["p"], IMGS), pref) <= TOL, "avg pool fwd"


def test_c3_backward_data(run, oracle):
    w = [np64(t) for t in run["w"]]
    dx, _, _ = oracle.conv2d_bwd(np64(run["p"], IMGS), w[2], np64(run["dy4"], IMGS), n=1, need=("dx",))
    assert rel(np64(run["dp"], IMGS), dx) <= TOL, "conv4 dgrad"
    H, W = run["y2"].shape[-2:]
    dref = oracle.pool2d_bwd(np64(run["dp"], IMGS), None, H, W, n=1, s=2, mode="avg")
    assert rel(np64(run["dy2"], IMGS), dref * (np64(run["y2"], IMGS) > 0)) <= TOL, "avg pool bwd"
    dx, _, _ = oracle.conv2d_bwd(np64(run["y1"], IMGS), w[1], np64(run["dy2"], IMGS), n=2, need=("dx",))
    assert rel(np64(run["dy1"], IMGS), dx * (np64(run["y1"], IMGS) > 0)) <= TOL, "conv2 dgrad (+ReLU mask)"


def test_c3_weight_gradients_full_batch(run, oracle):
    rng = np.random.default_rng(5)
    ins = [run["x"], run["y1"], run["p"]]
    dys = [run["dy1"], run["dy2"], run["dy4"]]
    for i in range(3):
        dw, db = run["grads"][i]
        co, ci, T = dw.shape
        pts = np.stack([rng.integers(0, co, 32), rng.integers(0, ci, 32), rng.integers(0, T, 32)], 1)
        ref = oracle.conv2d_bwd_weight_at(ins[i].contiguous().cpu().numpy(), dys[i].contiguous().cpu().numpy(),
                                          pts, n=run["ns"][i])
        got = dw.cpu().numpy()[pts[:, 0], pts[:, 1], pts[:, 2]]
        assert np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30) <= TOL, f"conv{i + 1} wgrad"
        db_ref = np64(dys[i]).sum(axis=(0, 2, 3))
        assert rel(db.cpu().numpy(), db_ref) <= TOL, f"conv{i + 1} dbias"
