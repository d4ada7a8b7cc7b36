"""World-size-2 data-parallel path on CPU (gloo): the per-layer gradient bucket
reducer that HexCNN.step uses over NCCL, and the weak-scaling invariant that
the DP-summed gradient of two half batches equals the single-process
gradient of the full batch (the per-image gradients are summed either way)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # import only the reducer: it needs torch.distributed, not the CUDA library
        import importlib.util
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        src = open(os.path.join(root, "paper_1903_01814_b200", "hexcnn.py")).read()
        start = src.index("class GradBucketReducer")
        end = src.index("class HexCNN")
        ns = {"dist": dist}
        exec(src[start:end], ns)
        Reducer = ns["GradBucketReducer"]

        g = torch.Generator().manual_seed(0)
        full_x = torch.randn(8, 5, generator=g, dtype=torch.float64)
        w = torch.randn(5, 3, generator=g, dtype=torch.float64)
        # local half batch -> local gradient of sum_i ||x_i w||^2 / 2 = x^T x w
        xl = full_x[rank * 4:(rank + 1) * 4]
        grads = torch.zeros(3 * 64, dtype=torch.float64)
        gl = xl.T @ (xl @ w)               # [5,3]
        grads[:15] = gl.flatten()
        grads[64:64 + 3] = xl.sum(0)[:3]
        red = Reducer(None)
        # reverse-order buckets, as HexCNN.backward issues them
        red.launch(grads[64:128])
        red.launch(grads[0:64])
        red.wait_all()
        ref = torch.zeros_like(grads)
        ref[:15] = (full_x.T @ (full_x @ w)).flatten()
        ref[64:67] = full_x.sum(0)[:3]
        q.put((rank, torch.allclose(grads, ref, atol=1e-12)))
    finally:
        dist.destroy_process_group()


def test_dp_bucket_allreduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]
