"""NVLS gradient sum (include/hexconv.h "NVLS gradient sum"; csrc/nvls.cu) -- host plumbing only.

The method's only exchange step in data-parallel training is the sum over ranks of the flat fp32 gradient
vector.  `NvlsBuffer` allocates that vector in device memory bound to a CUDA
multicast object spanning one GPU per rank, so that `allreduce(offset, count, slot, stream)` -- one library
kernel -- sums a bucket inside the NVSwitch (multimem.ld_reduce / multimem.st).  This module only moves the
multicast object's POSIX file descriptor from rank 0 to the other ranks (SCM_RIGHTS over a Unix socket whose
abstract name travels through the process group) and places the barriers the setup protocol needs.
"""
from __future__ import annotations

import ctypes
import os
import socket
import uuid

import torch
import torch.distributed as dist

from . import _abi as A


def _cuda_device(device):
    dev = torch.device(device) if device is not None else torch.device("cuda")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def _dist_on(group):
    return dist.is_available() and dist.is_initialized()


def world_rank(group=None):
    if _dist_on(group):
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def share_fd(fd, group=None, timeout_s: float = 60.0) -> int:
    """Rank 0's file descriptor `fd`, duplicated into every rank of `group` (collective).  Rank 0 gets `fd`
    back; the others get a new descriptor of the same open file (the caller closes it)."""
    world, rank = world_rank(group)
    if world == 1:
        return fd
    if rank == 0:
        name = "\0hexconv-nvls-" + uuid.uuid4().hex
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name)
        srv.listen(world)
        srv.settimeout(timeout_s)
        obj = [name]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        try:
            for _ in range(world - 1):
                conn, _ = srv.accept()
                with conn:
                    socket.send_fds(conn, [b"fd"], [fd])
                    conn.recv(1)  # the receiver's ack: it holds its own descriptor now
        finally:
            srv.close()
        return fd
    obj = [None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    cli.settimeout(timeout_s)
    try:
        cli.connect(obj[0])
        _, fds, _, _ = socket.recv_fds(cli, 16, 1)
        cli.sendall(b"k")
    finally:
        cli.close()
    if len(fds) != 1:
        raise RuntimeError("share_fd: no descriptor received")
    return fds[0]


def _barrier(group):
    if _dist_on(group) and dist.get_world_size(group) > 1:
        dist.barrier(group=group)


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (torch.as_tensor wraps it without a copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}


class NvlsBuffer:
    """fp32 region of `nbytes` bound to a multicast object over the ranks of `group` (collective setup).
    local=True (one rank only): plain device memory, the same kernel protocol with ordinary memory operations
    (hex_nvls_open_local) -- for one GPU, and for GPUs that cannot create multicast objects."""

    def __init__(self, nbytes: int, group=None, device=None, local: bool = False):
        self.group = group
        self.world, self.rank = world_rank(group)
        dev = _cuda_device(device)
        self.device = dev
        self.local = bool(local)
        L = A.lib()
        h = ctypes.c_void_p()
        fd_out = ctypes.c_int32(-1)
        if self.local:
            if self.world != 1:
                raise ValueError("NvlsBuffer(local=True) is single-rank")
            A.check(L.hex_nvls_open_local(dev.index, nbytes, ctypes.byref(h)), "hex_nvls_open_local")
        elif self.rank == 0:
            A.check(L.hex_nvls_open(self.world, 0, dev.index, nbytes, -1, ctypes.byref(fd_out), ctypes.byref(h)),
                    "hex_nvls_open")
            fd = share_fd(fd_out.value, group)
            if fd >= 0:
                os.close(fd)
        else:
            fd = share_fd(None, group)
            try:
                A.check(L.hex_nvls_open(self.world, self.rank, dev.index, nbytes, fd, None, ctypes.byref(h)),
                        "hex_nvls_open")
            finally:
                os.close(fd)
        self.h = h
        _barrier(group)  # every device attached before any memory is bound
        uc, mc, sz = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_size_t()
        A.check(L.hex_nvls_map(h, ctypes.byref(uc), ctypes.byref(mc), ctypes.byref(sz)), "hex_nvls_map")
        self.uc, self.mc, self.nbytes = uc.value, mc.value, sz.value
        _barrier(group)  # every rank's counters are zero before anyone arrives

    def tensor(self, n: int) -> torch.Tensor:
        """The first n floats of the local (unicast) view as a torch tensor (no copy; valid until close())."""
        if 4 * n > self.nbytes:
            raise ValueError("tensor larger than the NVLS region")
        return torch.as_tensor(_CudaArray(self.uc, n), device=self.device)

    def allreduce(self, offset: int, count: int, slot: int, stream=None):
        """Sum elements [offset, offset + count) over the ranks, on `stream` (default: the current stream)."""
        if stream is None:
            stream = ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        A.check(A.lib().hex_nvls_allreduce_f32(self.h, offset, count, slot, stream), "hex_nvls_allreduce_f32")

    def close(self):
        if self.h is not None and self.h.value:
            A.check(A.lib().hex_nvls_close(self.h), "hex_nvls_close")
        self.h = None


def supported(device=None) -> bool:
    dev = _cuda_device(device)
    s = ctypes.c_int32(0)
    A.check(A.lib().hex_nvls_supported(dev.index, ctypes.byref(s)), "hex_nvls_supported")
    return bool(s.value)


def plan(count: int, world: int, rank: int, cta: int = -1):
    """(grid, begin, end) of hex_nvls_plan: the element range (rank, cta) sums (host only)."""
    g, b, e = ctypes.c_int32(), ctypes.c_int64(-1), ctypes.c_int64(-1)
    A.check(A.lib().hex_nvls_plan(count, world, rank, cta, ctypes.byref(g), ctypes.byref(b), ctypes.byref(e)),
            "hex_nvls_plan")
    return g.value, b.value, e.value
