"""Host logic of the NVLS gradient sum (include/hexconv.h "NVLS gradient sum", csrc/nvls.cu, nvls.py),
no GPU: the work partition every rank's kernel uses (hex_nvls_plan: each element of a bucket is summed by
exactly one (rank, CTA), in 16-byte-aligned quads, the same chunking on every rank), the argument checks of
the setup calls, and the descriptor hand-off from rank 0 to the other ranks (world 2, gloo, SCM_RIGHTS)."""
import ctypes
import os
import socket
import tempfile

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_01814_b200 import _abi as A
from paper_1903_01814_b200 import nvls


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("count", [0, 1, 3, 4, 5, 7, 4099, 57_472 + 128, 1_245_440, 2_304_770])
def test_plan_tiles_the_bucket_once(world, count):
    grid, _, _ = nvls.plan(count, world, 0)
    assert 1 <= grid <= 148
    for r in range(world):
        assert nvls.plan(count, world, r)[0] == grid  # same chunking on every rank
    covered = 0
    prev_end = 0
    for c in range(grid):
        for r in range(world):
            g, b, e = nvls.plan(count, world, r, c)
            assert g == grid
            assert b == prev_end, (c, r, b, prev_end)  # contiguous, rank slices in order inside a chunk
            assert b <= e <= count
            assert b % 4 == 0  # vector (quad) boundaries
            covered += e - b
            prev_end = e
    assert covered == count and prev_end == count


def test_plan_balances_large_buckets():
    count = 2_304_770  # the config-5 gradient vector
    grid, _, _ = nvls.plan(count, 8, 0)
    assert grid == 148
    sizes = [nvls.plan(count, 8, r, c)[2] - nvls.plan(count, 8, r, c)[1] for c in range(grid) for r in range(8)]
    assert max(sizes) - min(sizes) <= 8


def test_setup_argument_checks_without_gpu():
    L = A.lib()
    h = ctypes.c_void_p()
    fd = ctypes.c_int32()
    assert L.hex_nvls_open(0, 0, 0, 1024, -1, ctypes.byref(fd), ctypes.byref(h)) == 1      # world < 1
    assert L.hex_nvls_open(2, 2, 0, 1024, -1, ctypes.byref(fd), ctypes.byref(h)) == 1      # rank >= world
    assert L.hex_nvls_open(2, 0, 0, 1024, -1, None, ctypes.byref(h)) == 1                  # no fd_out on rank 0
    assert L.hex_nvls_open(2, 1, 0, 1024, -1, None, ctypes.byref(h)) == 1                  # no fd_in on rank 1
    assert L.hex_nvls_open(1, 0, 0, 0, -1, None, ctypes.byref(h)) == 1                     # empty region
    assert L.hex_nvls_open_local(0, 0, ctypes.byref(h)) == 1                                # empty region
    assert L.hex_nvls_open_local(0, 1024, None) == 1
    if not __import__("torch").cuda.is_available():
        assert L.hex_nvls_open_local(0, 1024, ctypes.byref(h)) == 1                         # no device
    assert L.hex_nvls_allreduce_f32(None, 0, 4, 0, None) == 1
    assert L.hex_nvls_close(None) == 1
    g = ctypes.c_int32()
    b, e = ctypes.c_int64(), ctypes.c_int64()
    assert L.hex_nvls_plan(-1, 1, 0, 0, ctypes.byref(g), ctypes.byref(b), ctypes.byref(e)) == 2
    assert L.hex_nvls_plan(16, 2, 2, 0, ctypes.byref(g), ctypes.byref(b), ctypes.byref(e)) == 1
    assert L.hex_nvls_plan(16, 2, 0, 5, ctypes.byref(g), ctypes.byref(b), ctypes.byref(e)) == 1  # cta >= grid
    s = ctypes.c_int32(7)
    assert L.hex_nvls_supported(0, ctypes.byref(s)) == 0
    if not __import__("torch").cuda.is_available():
        assert s.value == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fd_worker(rank, world, port, path, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fd = os.open(path, os.O_RDONLY) if rank == 0 else None
        got = nvls.share_fd(fd, None)
        data = os.pread(got, 64, 0)
        st = os.fstat(got)
        os.close(got)
        q.put((rank, data, st.st_ino, got != fd or rank == 0))
    except Exception as ex:  # pragma: no cover - reported through the queue
        q.put((rank, repr(ex), None, False))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_share_fd_over_process_group(world):
    with tempfile.NamedTemporaryFile(delete=False) as f:
        f.write(b"multicast handle stand-in")
        path = f.name
    try:
        ino = os.stat(path).st_ino
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        ps = [ctx.Process(target=_fd_worker, args=(r, world, port, path, q)) for r in range(world)]
        for p in ps:
            p.start()
        res = sorted((q.get(timeout=300) for _ in ps), key=lambda t: t[0])
        for p in ps:
            p.join(timeout=60)
        for rank, data, st_ino, ok in res:
            assert data == b"multicast handle stand-in", (rank, data)
            assert st_ino == ino and ok
    finally:
        os.unlink(path)
