"""BASELINE config 5 at full size (256 images of 96x96, the launch configuration
bench.py times): one training step of HexCNN, then every layer is checked
against the fp64 oracle fed the GPU's own inputs of that layer (reading A17):

  * conv fwd (+ReLU), pools (values + argmax bit-exact), dgrad (with the fused
    ReLU / pooled mask) on sampled images (images are independent);
  * weight gradients at sampled (co, ci, t) points summed over all 256 images
    (oracle point evaluation);
  * head (GAP, linear, CE) against numpy fp64 on the full batch.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL = 2e-2
IMGS = [0, 255]


@pytest.fixture(scope="module")
def run():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import synth
    from paper_1903_01814_b200.hexcnn import HexCNN
    m = HexCNN(batch=256, seed=0)
    x = torch.from_numpy(np.ascontiguousarray(synth.shower_images(256, 96, 96, 47, 5).transpose(0, 2, 3, 1))
                         ).cuda().to(torch.bfloat16)
    y = torch.from_numpy(synth.labels(256, 6)).cuda()
    w_used = m.params_bf16.clone()
    head_used = m.params.clone()
    loss = m.step(x, y)
    torch.cuda.synchronize()
    return m, x, y, w_used, head_used, loss


def nchw(t, idx=None):
    t = t if idx is None else t[idx]
    return t.float().permute(0, 3, 1, 2).cpu().numpy().astype(np.float64)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def used_weight(m, w_used, l):
    wo, wn, _, _ = m.seg[l]
    ci, co, T = m.channels[l], m.channels[l + 1], m.weight(l).shape[2]
    return w_used[wo:wo + wn].view(co, ci, T).float().cpu().numpy().astype(np.float64)


def test_c5_forward_layers(run, oracle):
    from paper_1903_01814_b200 import functional as F
    m, x, _, w_used, head_used, _ = run
    for l in range(m.L):
        xin = nchw(m.layer_input(l, x), IMGS)
        w = used_weight(m, w_used, l)
        _, _, bo, bn = m.seg[l]
        b = head_used[bo:bo + bn].cpu().numpy().astype(np.float64)
        ref = np.maximum(oracle.conv2d_fwd(xin, w, b, n=m.ns[l]), 0)
        act = m.act[l]
        if l in m.pool_geo and m.fused_pool[l]:
            # fused conv + pool: the step never wrote act[l]; recompute the GPU's own conv output for the
            # sampled images with the unfused kernel (bit-identical to the fused kernel's internal values)
            wb = w_used[m.seg[l][0]:m.seg[l][0] + m.seg[l][1]].view(m.channels[l + 1], m.channels[l], -1)
            act = F.conv2d_fwd(m.layer_input(l, x)[IMGS].contiguous(), wb, head_used[bo:bo + bn], n=m.ns[l],
                               relu=True, layout="NHWC")
            act = torch.zeros_like(m.act[l]).index_copy_(0, torch.tensor(IMGS, device=act.device), act)
        assert rel(nchw(act, IMGS), ref) <= TOL, f"conv{l + 1} fwd"
        if l in m.pool_geo:
            a = nchw(act, IMGS)
            p, am = oracle.pool2d_fwd(a, n=1, s=2, mode="max")
            assert np.array_equal(nchw(m.pooled[l], IMGS), p), f"pool{l + 1} value"
            assert np.array_equal(m.argmax[l][IMGS].permute(0, 3, 1, 2).cpu().numpy(), am), f"pool{l + 1} argmax"


def test_c5_head(run):
    m, _, y, _, head_used, loss = run
    feat = m.act[-1].float().cpu().numpy().astype(np.float64)       # [B,h,w,C]
    C, K = m.channels[-1], m.K
    wl = head_used[m.head_w:m.head_w + K * C].view(K, C).cpu().numpy().astype(np.float64)
    bl = head_used[m.head_b:m.head_b + K].cpu().numpy().astype(np.float64)
    gap = feat.mean(axis=(1, 2))
    lg = gap @ wl.T + bl
    z = lg - lg.max(1, keepdims=True)
    lse = np.log(np.exp(z).sum(1))
    lab = y.cpu().numpy()
    ref_loss = float(np.mean(lse - z[np.arange(len(lab)), lab]))
    assert abs(loss.item() - ref_loss) <= 1e-4 * max(1.0, abs(ref_loss))
    pr = np.exp(z - lse[:, None])
    dlog = (pr - np.eye(K)[lab]) / len(lab)
    dfeat = (dlog @ wl)[:, None, None, :] / (feat.shape[1] * feat.shape[2]) * (feat > 0)
    assert rel(m.dact[-1].float().cpu().numpy(), dfeat) <= TOL
    g = m.grads
    assert rel(g[m.head_w:m.head_w + K * C].view(K, C).cpu().numpy(), dlog.T @ gap) <= 1e-4
    assert rel(g[m.head_b:m.head_b + K].cpu().numpy(), dlog.sum(0)) <= 1e-4


def test_c5_backward_data_layers(run, oracle):
    m, x, _, w_used, _, _ = run
    for l in range(m.L - 1, 0, -1):
        dy = nchw(m.dact[l], IMGS)
        w = used_weight(m, w_used, l)
        xin = nchw(m.layer_input(l, x), IMGS)
        dx, _, _ = oracle.conv2d_bwd(xin, w, dy, n=m.ns[l], need=("dx",))
        prev = l - 1
        if prev in m.pool_geo:
            masked = dx * (nchw(m.pooled[prev], IMGS) > 0)
            assert rel(nchw(m.dpool[prev], IMGS), masked) <= TOL, f"conv{l + 1} dgrad"
            # pool bwd on the GPU's own pooled gradient
            h, w_, _, _ = m.pool_geo[prev]
            am = m.argmax[prev][IMGS].permute(0, 3, 1, 2).cpu().numpy()
            ref = oracle.pool2d_bwd(nchw(m.dpool[prev], IMGS), am, h, w_, n=1, s=2, mode="max")
            assert rel(nchw(m.dact[prev], IMGS), ref) <= TOL, f"pool{prev + 1} bwd"
        else:
            masked = dx * (nchw(m.act[prev], IMGS) > 0)
            assert rel(nchw(m.dact[prev], IMGS), masked) <= TOL, f"conv{l + 1} dgrad"


def test_c5_weight_gradients_full_batch(run, oracle):
    m, x, _, _, _, _ = run
    rng = np.random.default_rng(3)
    for l in range(m.L):
        ci, co, T = m.channels[l], m.channels[l + 1], m.weight(l).shape[2]
        pts = np.stack([rng.integers(0, co, 24), rng.integers(0, ci, 24), rng.integers(0, T, 24)], 1)
        xin = m.layer_input(l, x).contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        dy = m.dact[l].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        ref = oracle.conv2d_bwd_weight_at(xin, dy, pts, n=m.ns[l], layout="NHWC")
        wo, wn, bo, bn = m.seg[l]
        got = m.grads[wo:wo + wn].view(co, ci, T).cpu().numpy()[pts[:, 0], pts[:, 1], pts[:, 2]]
        scale = max(np.abs(ref).max(), 1e-30)
        assert np.abs(got - ref).max() / scale <= 1e-3, f"conv{l + 1} wgrad"
        dyf = m.dact[l].float().cpu().numpy().astype(np.float64)
        db_ref = dyf.sum(axis=(0, 1, 2))
        db = m.grads[bo:bo + bn].cpu().numpy()
        assert rel(db, db_ref) <= 1e-3, f"conv{l + 1} dbias"


def test_c5_paths(run):
    # layers 2-6 run on the tcgen05 kernels in every pass; layer 1 (Cin = 1) on the stencil path
    import ctypes
    from paper_1903_01814_b200 import _abi as A
    m = run[0]
    for l in range(m.L):
        for pass_id in (0, 1, 2):
            a = ctypes.c_int32()
            A.check(A.lib().hex_conv2d_algo(ctypes.byref(m.desc[l]), pass_id, ctypes.byref(a)), "algo")
            assert a.value == (0 if l == 0 else 1), (l, pass_id)


def test_graphed_step_matches_eager():
    # HexCNN.graphed_step (bench.py's e2e leg): a CUDA-graph replay of the step gives bit-identical
    # parameters to the eager step (same kernels, deterministic reductions)
    import synth
    from paper_1903_01814_b200.hexcnn import HexCNN
    B = 8
    x = torch.from_numpy(np.ascontiguousarray(synth.shower_images(B, 96, 96, 47, 11).transpose(0, 2, 3, 1))
                         ).cuda().to(torch.bfloat16)
    y = torch.from_numpy(synth.labels(B, 12)).cuda()
    a, b = HexCNN(batch=B, seed=3), HexCNN(batch=B, seed=3)
    a.step(x, y)
    la = a.step(x, y).clone()
    g, lb = b.graphed_step(x, y)   # one real (warm-up) step
    g.replay()                     # the second step
    torch.cuda.synchronize()
    assert torch.equal(a.params, b.params)
    assert torch.equal(a.mom, b.mom)
    assert la.item() == lb.item()


def test_training_loss_stays_finite():
    # 30 SGD-momentum steps on the bench's synthetic shower batches (raw amplitudes up to ~5000, the
    # default lr 1e-3): the loss stays finite and settles near ln 2 for random labels
    import bench
    from paper_1903_01814_b200.hexcnn import HexCNN
    xs_np, ys_np = bench.make_batches(2, 64, 96, 96, 47, seed=1000)
    xs = [torch.from_numpy(a).cuda().to(torch.bfloat16) for a in xs_np]
    ys = [torch.from_numpy(a).cuda() for a in ys_np]
    m = HexCNN(batch=64, seed=0)
    losses = [float(m.step(xs[i % 2], ys[i % 2]).item()) for i in range(30)]
    assert all(np.isfinite(losses)), losses
    assert abs(np.mean(losses[-5:]) - np.log(2)) < 0.5, losses


def test_bench_line_contract():
    # `python bench.py` (short run, no secondary configs) prints the JSON line the driver parses, with the keys
    # and value ranges its contract requires
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "3", "--warmup", "3",
                          "--no-secondary", "--no-cpu-baseline", "--sustain-s", "0"],
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["unit"] == "images/s"
    assert d["value"] > 1000 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["scaling"] == "weak" and d["data"] == "synthetic" and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] <= 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["clocks"]["sm_mhz"] > 0 and "reasons" in d["clocks"]
