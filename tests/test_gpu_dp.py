"""Data-parallel training step of config 5 with the real model.

* Two ranks (processes) share the one GPU over gloo (collectives on CUDA tensors are host-side copies in
  gloo, so no kernel waits on another rank's kernel).  Each rank steps HexCNN on its half of a 16-image
  batch; the per-layer GradBucketReducer sums the weight gradients.  Checked:
    - the DP-summed gradients (x 1/world, as the optimizer applies them) equal the single-process
      16-image step's gradients to fp32 reduction-order tolerance;
    - sampled conv weight gradients equal the fp64 oracle's point evaluation over all 16 images, fed
      both ranks' own layer inputs and upstream gradients (reading A17);
    - parameters and momenta are bitwise equal across ranks after SGD.
* A one-rank NCCL group with reduce_grads=True: the captured CUDA graph of the step (per-layer NCCL
  allreduces inside the capture, as bench.py replays it under torchrun) gives bit-identical parameters
  to the eager step.
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

B_FULL, WORLD = 16, 2
CHECK_LAYERS = (1, 2, 5)     # 0-based conv layers whose weight gradients are point-evaluated


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch():
    import synth
    x = np.ascontiguousarray(synth.shower_images(B_FULL, 96, 96, 47, 21).transpose(0, 2, 3, 1))
    y = synth.labels(B_FULL, 22)
    return x, y


def _u16(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _dp_worker(rank, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        from paper_1903_01814_b200.hexcnn import HexCNN
        x, y = _batch()
        h = B_FULL // WORLD
        xd = torch.from_numpy(x[rank * h:(rank + 1) * h]).cuda().to(torch.bfloat16)
        yd = torch.from_numpy(y[rank * h:(rank + 1) * h]).cuda()
        m = HexCNN(batch=h, seed=4)
        assert m.world == WORLD and m.reduce_grads
        loss = m.step(xd, yd)
        torch.cuda.synchronize()
        out = {"rank": rank, "loss": float(loss.item()), "grads": m.grads.cpu().numpy(),
               "params": m.params.cpu().numpy(), "mom": m.mom.cpu().numpy(),
               "xin": {l: _u16(m.layer_input(l, xd)) for l in CHECK_LAYERS},
               "dy": {l: _u16(m.dact[l]) for l in CHECK_LAYERS}}
        q.put(out)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # surface the failure instead of hanging the parent on q.get
        import traceback
        q.put({"rank": rank, "error": traceback.format_exc() + repr(ex)})


@pytest.fixture(scope="module")
def dp_run():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_dp_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        r = q.get(timeout=600)
        assert "error" not in r, r.get("error")
        res[r["rank"]] = r
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the single-process step on the full 16-image batch, same initial parameters
    from paper_1903_01814_b200.hexcnn import HexCNN
    x, y = _batch()
    m = HexCNN(batch=B_FULL, seed=4)
    loss = m.step(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(y).cuda())
    torch.cuda.synchronize()
    return res, m, float(loss.item())


def _rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


def test_dp_params_identical_across_ranks(dp_run):
    res, _, _ = dp_run
    assert np.array_equal(res[0]["grads"], res[1]["grads"])
    assert np.array_equal(res[0]["params"], res[1]["params"])
    assert np.array_equal(res[0]["mom"], res[1]["mom"])


def test_dp_grads_match_single_process(dp_run):
    res, m, loss_full = dp_run
    # each rank's loss is the mean over its half batch; their mean is the full-batch loss
    assert abs(0.5 * (res[0]["loss"] + res[1]["loss"]) - loss_full) <= 1e-5 * max(1.0, abs(loss_full))
    g_dp = res[0]["grads"].astype(np.float64) / WORLD
    g_sp = m.grads.cpu().numpy().astype(np.float64)
    for l in range(m.L):
        wo, wn, bo, bn = m.seg[l]
        assert _rel(g_dp[wo:wo + wn], g_sp[wo:wo + wn]) <= 1e-4, f"conv{l + 1} dw"
        assert _rel(g_dp[bo:bo + bn], g_sp[bo:bo + bn]) <= 1e-4, f"conv{l + 1} dbias"
    hw = slice(m.head_w, m.nparams)
    assert _rel(g_dp[hw], g_sp[hw]) <= 1e-5, "head"
    # and the SGD update applied the averaged gradient: params agree with the single-process step
    assert _rel(res[0]["params"], m.params.cpu().numpy().astype(np.float64)) <= 1e-6


def test_dp_weight_grads_vs_oracle(dp_run, oracle):
    res, m, _ = dp_run
    rng = np.random.default_rng(7)
    for l in CHECK_LAYERS:
        ci, co, T = m.channels[l], m.channels[l + 1], m.weight(l).shape[2]
        pts = np.stack([rng.integers(0, co, 16), rng.integers(0, ci, 16), rng.integers(0, T, 16)], 1)
        xin = np.concatenate([res[r]["xin"][l] for r in range(WORLD)], 0)
        dy = np.concatenate([res[r]["dy"][l] for r in range(WORLD)], 0)
        ref = oracle.conv2d_bwd_weight_at(xin, dy, pts, n=m.ns[l], layout="NHWC")
        wo, wn, _, _ = m.seg[l]
        got = res[0]["grads"][wo:wo + wn].reshape(co, ci, T)[pts[:, 0], pts[:, 1], pts[:, 2]]
        assert np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30) <= 1e-3, f"conv{l + 1} DP wgrad"


def _nccl_graph_worker(port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        from paper_1903_01814_b200.hexcnn import HexCNN
        x, y = _batch()
        xd = torch.from_numpy(x[:8]).cuda().to(torch.bfloat16)
        yd = torch.from_numpy(y[:8]).cuda()
        a = HexCNN(batch=8, seed=5, reduce_grads=True)
        b = HexCNN(batch=8, seed=5, reduce_grads=True)
        a.step(xd, yd)
        la = a.step(xd, yd).clone()
        g, lb = b.graphed_step(xd, yd)   # one real (warm-up) step, then capture
        g.replay()
        torch.cuda.synchronize()
        q.put({"ok": bool(torch.equal(a.params, b.params) and torch.equal(a.mom, b.mom)
                          and la.item() == lb.item())})
        dist.destroy_process_group()
    except Exception as ex:
        import traceback
        q.put({"error": traceback.format_exc() + repr(ex)})


def test_dp_graphed_step_nccl_capture():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_graph_worker, args=(_free_port(), q))
    p.start()
    r = q.get(timeout=600)
    p.join(timeout=120)
    assert "error" not in r, r.get("error")
    assert r["ok"]
