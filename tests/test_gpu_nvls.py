"""NVLS gradient sum (include/hexconv.h "NVLS gradient sum", csrc/nvls.cu) on one GPU.

The run has one GPU.  Where it can create a multicast object, the object spans that one device; where it
cannot (this pool's lease, profiles/r02/nvls_probe.txt), the region is the single-rank local mode
(hex_nvls_open_local: plain device memory, ordinary loads / stores / red in place of the multimem ones).
Either way the sum over the replicas is the identity and every counter wait completes on this rank's own
arrival, and the kernel's whole control path runs: the arrivals, the acquire waits with device-resident
epochs, the per-CTA partition and the vector / scalar (ragged tail) element loop.  Pinned: the bucket comes
back bitwise unchanged, elements outside the bucket are untouched, repeated and graph-replayed calls keep
their epochs in step, and a HexCNN step whose gradients go through the NVLS path gives bit-identical
parameters to the plain step.  The sum over several ranks is the hardware's multimem.ld_reduce; the
partition that makes each element summed exactly once is pinned on CPU (tests/test_nvls_host.py)."""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["multicast", "local"])
def nv(request):
    from paper_1903_01814_b200 import nvls
    if request.param == "multicast" and not nvls.supported():
        pytest.skip("device without usable multicast objects (profiles/r02/nvls_probe.txt)")
    buf = nvls.NvlsBuffer(4 * 3_000_000, local=request.param == "local")
    yield buf
    buf.close()


BUCKETS = [(0, 1), (4, 3), (8, 5), (64, 4099), (4160, 123_457), (200_000, 1_245_440), (1_445_440, 1_554_560)]


def test_nvls_bucket_sum_single_rank(nv):
    t = nv.tensor(3_000_000)
    g = torch.Generator(device="cuda").manual_seed(5)
    ref = torch.randn(3_000_000, device="cuda", generator=g)
    t.copy_(ref)
    for slot, (off, n) in enumerate(BUCKETS):
        nv.allreduce(off, n, slot)
    for slot, (off, n) in enumerate(BUCKETS):
        nv.allreduce(off, n, slot)  # second epoch of every slot
    torch.cuda.synchronize()
    assert torch.equal(t.view(torch.int32), ref.view(torch.int32))


def test_nvls_graph_replay(nv):
    t = nv.tensor(3_000_000)
    ref = torch.arange(3_000_000, device="cuda", dtype=torch.float32) * 0.5 - 7.0
    t.copy_(ref)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            for slot, (off, n) in enumerate(BUCKETS):
                nv.allreduce(off, n, 10 + slot)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(t.view(torch.int32), ref.view(torch.int32))


def test_nvls_rejects_bad_buckets(nv):
    from paper_1903_01814_b200 import _abi as A
    L = A.lib()
    assert L.hex_nvls_allreduce_f32(nv.h, 2, 8, 0, None) == 6            # offset not a multiple of 4
    assert L.hex_nvls_allreduce_f32(nv.h, 0, nv.nbytes // 4 + 1, 0, None) == 2
    assert L.hex_nvls_allreduce_f32(nv.h, 0, 8, 64, None) == 1           # slot out of range
    assert L.hex_nvls_allreduce_f32(nv.h, -4, 8, 0, None) == 2


def test_hexcnn_step_through_nvls_is_bit_identical():
    # one rank: the multicast region where the GPU can create one, else the local mode (HexCNN picks)
    import synth
    from paper_1903_01814_b200.hexcnn import HexCNN
    B = 8
    x = np.ascontiguousarray(synth.shower_images(B, 96, 96, 47, 31).transpose(0, 2, 3, 1))
    y = synth.labels(B, 32)
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    yd = torch.from_numpy(y).cuda()
    plain = HexCNN(batch=B, seed=6)
    viaNv = HexCNN(batch=B, seed=6, reduce_grads=True, nvls=True)
    assert viaNv._nv is not None and plain._nv is None
    for _ in range(2):
        plain.step(xd, yd)
        viaNv.step(xd, yd)
    torch.cuda.synchronize()
    assert torch.equal(plain.params.view(torch.int32), viaNv.params.view(torch.int32))
    assert torch.equal(plain.grads.view(torch.int32), viaNv.grads.view(torch.int32))
    # the captured step (NVLS kernels inside the graph) continues bit-identically
    graph, _ = viaNv.graphed_step(xd, yd)   # its warm-up performs one real step
    plain.step(xd, yd)
    graph.replay()
    plain.step(xd, yd)
    torch.cuda.synchronize()
    assert torch.equal(plain.params.view(torch.int32), viaNv.params.view(torch.int32))
    viaNv._nv.close()
