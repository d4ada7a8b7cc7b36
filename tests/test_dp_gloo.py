"""World-size-2 data-parallel path on CPU (gloo): the per-layer gradient bucket
reducer that HexCNN.step uses over NCCL (imported from the product module, not
re-implemented), and the weak-scaling invariant of the method's only exchange
step: the DP sum of the hex-conv weight / bias gradients of two
half batches equals the weight gradient of the full batch (the per-image
gradients are summed either way).  The per-rank gradients come from the fp64
oracle (test infrastructure), laid out in the flat [W, b] segments HexCNN uses
and reduced in reverse layer order as HexCNN.backward issues them."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

LAYERS = ((3, 4, 1), (4, 2, 2))   # (Cin, Cout, n) of a two-layer toy hex net


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _grads(oracle, xs, gs, ws):
    """Flat [dW0 | db0 | dW1 | db1] of the given images (fp64 oracle adjoint)."""
    parts = []
    for (ci, co, n), x, g, w in zip(LAYERS, xs, gs, ws):
        _, dw, db = oracle.conv2d_bwd(x, w, g, n=n, need=("dw", "db"))
        parts += [dw.ravel(), db.ravel()]
    return np.concatenate(parts)


def _inputs(oracle):
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal((4, ci, 7, 9)) for ci, _, _ in LAYERS]
    gs = [rng.standard_normal((4, co, 7, 9)) for _, co, _ in LAYERS]
    ws = [rng.standard_normal((co, ci, oracle.num_taps(n))) for ci, co, n in LAYERS]
    return xs, gs, ws


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1903_01814_b200.hexcnn import GradBucketReducer
        xs, gs, ws = _inputs(oracle)
        h = slice(rank * 2, rank * 2 + 2)       # this rank's half of the 4-image batch
        flat = torch.from_numpy(_grads(oracle, [x[h] for x in xs], [g[h] for g in gs], ws))
        # segment boundaries of the flat vector, one bucket per layer
        bounds, off = [], 0
        for ci, co, n in LAYERS:
            sz = co * ci * oracle.num_taps(n) + co
            bounds.append((off, off + sz))
            off += sz
        red = GradBucketReducer(None)
        for a, b in reversed(bounds):
            red.launch(flat[a:b])
        red.wait_all()
        full = _grads(oracle, xs, gs, ws)
        q.put((rank, float(np.abs(flat.numpy() - full).max() / np.abs(full).max())))
    except Exception as ex:
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def test_dp_bucket_allreduce_world2(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [r for r, _ in res] == [0, 1]
    for _, err in res:
        assert isinstance(err, float) and err <= 1e-12, err
