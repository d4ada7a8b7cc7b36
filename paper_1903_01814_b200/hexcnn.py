"""Data-parallel training step of the BASELINE config-5 hexagonal CNN.

Network (BASELINE.json configs[4]): 96x96 offset-column
grid, 1 input channel, six hex convolutions with channels
1->64->128->128->256->256->256 and kernel sizes n = 2,1,2,1,2,1 (stride 1,
ReLU), hex max-pool n=1 stride 2 after layers 2 and 4, global average pool,
linear head to 2 logits, softmax cross-entropy.  bf16 NHWC activations,
fp32 master weights, SGD with momentum 0.9; data parallel over the batch with
the weight-gradient sum over NCCL (torch.distributed) -- the only exchange
step of the method -- or, with nvls=True, inside the
NVSwitch by the library's multimem kernel (nvls.py, csrc/nvls.cu).

Every tensor operation is a call into libhexconv (include/hexconv.h) on
buffers allocated once here; torch provides device memory, the stream and
the process group only.  The ReLU backward of a layer is fused into the
epilogue of the next layer's backward-data kernel (relu_y argument); for the
pooled layers the mask is taken on the pooled tensor, which is exact for max
pooling because the routed gradient reaches the argmax cell, whose value is
the pooled value.
"""
from __future__ import annotations

import ctypes
import os
import math

import numpy as np
import torch
import torch.distributed as dist

from . import _abi as A

_BF16 = A.BF16
_NHWC = A.NHWC


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _align(n, a=64):
    return (n + a - 1) // a * a


class GradBucketReducer:
    """Per-layer gradient buckets summed over the data-parallel ranks as soon
    as each layer's weight gradient is enqueued (reverse layer order), so the
    NCCL allreduce of layer l overlaps the backward of layers < l.  The 1/N
    average is folded into the optimizer's grad_scale.  Works with any
    torch.distributed backend (NCCL on GPUs; gloo in the CPU tests)."""

    def __init__(self, process_group=None):
        self.pg = process_group
        self.works = []

    def launch(self, bucket):
        self.works.append(dist.all_reduce(bucket, op=dist.ReduceOp.SUM, group=self.pg, async_op=True))

    def wait_all(self):
        for w in self.works:
            w.wait()
        self.works.clear()


class HexCNN:
    def __init__(self, batch: int = 256, H: int = 96, W: int = 96,
                 channels=(1, 64, 128, 128, 256, 256, 256), ns=(2, 1, 2, 1, 2, 1), pool_after=(2, 4),
                 num_classes: int = 2, lr: float = 1e-3, momentum: float = 0.9, seed: int = 0,
                 device="cuda", process_group=None, reduce_grads=None, nvls=None):
        self.B, self.H, self.W = batch, H, W
        self.channels, self.ns, self.pool_after = tuple(channels), tuple(ns), tuple(pool_after)
        self.K = num_classes
        self.lr, self.mu = lr, momentum
        self.dev = torch.device(device)
        self.pg = process_group
        self.world = dist.get_world_size(process_group) if (dist.is_available() and dist.is_initialized()) else 1
        # the per-layer gradient allreduce runs whenever there is more than one rank; reduce_grads=True
        # forces it at world size 1 too (tests: a one-rank NCCL group captured in a CUDA graph)
        self.reduce_grads = (self.world > 1) if reduce_grads is None else bool(reduce_grads)
        self.L = len(ns)
        # gradient sum inside the NVSwitch (nvls.py, csrc/nvls.cu) instead of NCCL buckets: HEXCNN_NVLS=1 or
        # nvls=True; the gradient vector then lives in multicast-bound memory
        self.nvls = bool(os.environ.get("HEXCNN_NVLS")) if nvls is None else bool(nvls)
        self._nv = None
        self.timer = None  # optional list: (kind, layer, start_event, end_event) around conv calls
        # weight gradients on a side stream (HEXCNN_SIDE_BWD=1): measured no faster than one stream once the
        # training data is finite (3.52 vs 3.47 ms per step), and it blurs the per-family event timings
        self._side = torch.cuda.Stream(device=device) \
            if (os.environ.get("HEXCNN_SIDE_BWD") and torch.cuda.is_available()) else None
        self._layout()
        self._init_params(seed)
        self._alloc()

    # ------------------------------------------------------------------ geometry & buffers
    def _layout(self):
        self.geo = []   # per layer: (H, W) of its input/output grid (stride 1 convs)
        h, w = self.H, self.W
        self.pool_geo = {}
        for l in range(self.L):
            self.geo.append((h, w))
            if (l + 1) in self.pool_after:
                ho, wo, po = A.output_shape(h, w, 2, 0)
                assert po == 0
                self.pool_geo[l] = (h, w, ho, wo)
                h, w = ho, wo
        self.feat_hw = (h, w)
        # flat parameter layout: per layer [W (Co*Ci*T), b (Co)], then head [wl (K*C), bl (K)]
        self.seg = []
        off = 0
        for l in range(self.L):
            ci, co, T = self.channels[l], self.channels[l + 1], A.num_taps(self.ns[l])
            wo_ = off
            off = _align(off + co * ci * T)
            bo = off
            off = _align(off + co)
            self.seg.append((wo_, co * ci * T, bo, co))
        C = self.channels[-1]
        self.head_w = off
        off = _align(off + self.K * C)
        self.head_b = off
        off = _align(off + self.K)
        self.nparams = off
        self.param_count = sum(a[1] + a[3] for a in self.seg) + self.K * C + self.K

    def _init_params(self, seed):
        rng = np.random.default_rng(seed)
        flat = np.zeros(self.nparams, dtype=np.float32)
        for l, (wo, wn, bo, bn) in enumerate(self.seg):
            ci, co, T = self.channels[l], self.channels[l + 1], A.num_taps(self.ns[l])
            lim = math.sqrt(6.0 / (ci * T))  # He-uniform, fan_in = Cin * T (A19)
            flat[wo:wo + wn] = rng.uniform(-lim, lim, size=wn)
        C = self.channels[-1]
        lim = 1.0 / math.sqrt(C)
        flat[self.head_w:self.head_w + self.K * C] = rng.uniform(-lim, lim, size=self.K * C)
        self.params = torch.from_numpy(flat).to(self.dev)
        self.params_bf16 = self.params.to(torch.bfloat16)
        self.grads = torch.zeros_like(self.params)
        if self.nvls and self.reduce_grads:
            from . import nvls as nv
            # one rank on a GPU that cannot create multicast objects: the same kernel on plain memory
            local = self.world == 1 and not nv.supported(self.dev)
            self._nv = nv.NvlsBuffer(4 * self.nparams, self.pg, self.dev, local=local)
            self._nv_side = torch.cuda.Stream(device=self.dev)  # the bucket sums overlap the backward
            g = self._nv.tensor(self.nparams)
            g.zero_()
            self.grads = g
        self.mom = torch.zeros_like(self.params)

    def weight(self, l, bf16=True):
        wo, wn, _, _ = self.seg[l]
        ci, co, T = self.channels[l], self.channels[l + 1], A.num_taps(self.ns[l])
        src = self.params_bf16 if bf16 else self.params
        return src[wo:wo + wn].view(co, ci, T)

    def bias(self, l):
        _, _, bo, bn = self.seg[l]
        return self.params[bo:bo + bn]

    def _alloc(self):
        B, dev, bf = self.B, self.dev, torch.bfloat16
        L_ = A.lib()
        self.act = []       # conv outputs (post-ReLU), NHWC
        self.pooled = {}    # pool outputs
        self.argmax = {}
        self.dact = []      # gradient wrt conv pre-activation outputs (masked), NHWC
        self.dpool = {}
        self.desc = []
        self.ws = []
        for l in range(self.L):
            h, w = self.geo[l]
            ci, co = self.channels[l], self.channels[l + 1]
            d = A.ConvDesc(B, ci, co, h, w, self.ns[l], 1, 0, _BF16, _NHWC)
            self.desc.append(d)
            self.act.append(torch.empty(B, h, w, co, dtype=bf, device=dev))
            self.dact.append(torch.empty(B, h, w, co, dtype=bf, device=dev))
            sizes = []
            for pass_id in (0, 1, 2):
                sz = ctypes.c_size_t()
                A.check(A.lib().hex_conv2d_workspace_size(ctypes.byref(d), pass_id, ctypes.byref(sz)), "ws")
                sizes.append(sz.value)
            self.ws.append([torch.empty(max(s, 1), dtype=torch.uint8, device=dev) for s in sizes])
            self.ws_sizes = getattr(self, "ws_sizes", []) + [sizes]
            if l in self.pool_geo:
                hh, ww, ho, wo = self.pool_geo[l]
                self.pooled[l] = torch.empty(B, ho, wo, co, dtype=bf, device=dev)
                self.argmax[l] = torch.empty(B, ho, wo, co, dtype=torch.uint8, device=dev)
                self.dpool[l] = torch.empty(B, ho, wo, co, dtype=bf, device=dev)
        # fused conv + ReLU + max pool (hex_conv2d_fwd_maxpool) where supported; HEXCNN_NO_FUSED_POOL=1
        # restores the separate conv and pool calls
        self.fused_pool = {l: bool(L_.hex_conv2d_fwd_maxpool_supported(ctypes.byref(self.desc[l])))
                           and not os.environ.get("HEXCNN_NO_FUSED_POOL") for l in self.pool_geo}
        self.pdesc = {l: A.PoolDesc(B, self.channels[l + 1], *self.pool_geo[l][:2], 1, 2, 0, _BF16, _NHWC,
                                    A.POOL_MAX) for l in self.pool_geo}
        # tensor-core layers read their weights pre-packed (hex_conv2d_pack_weights: every layer's fwd and
        # bwd-data packing in one launch per step instead of one per call); HEXCNN_NO_PREPACK=1 packs per call
        entries = []
        self.packed = set()  # (layer, pass)
        if not os.environ.get("HEXCNN_NO_PREPACK"):
            for l in range(self.L):
                for pass_id in (0, 1):
                    if pass_id == 1 and l == 0:
                        continue  # no bwd-data into the network input
                    algo = ctypes.c_int32()
                    A.check(L_.hex_conv2d_algo(ctypes.byref(self.desc[l]), pass_id, ctypes.byref(algo)), "algo")
                    if algo.value != 1 or self.desc[l].stride != 1:
                        continue
                    entries.append((self.desc[l], pass_id, self.weight(l).data_ptr(), self.ws[l][pass_id].data_ptr(),
                                    self.ws_sizes[l][pass_id]))
                    self.packed.add((l, pass_id))
        self.pack_args = A.PackArgs(entries) if entries else None
        C = self.channels[-1]
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        hw = self.feat_hw[0] * self.feat_hw[1]
        self.head_ws_bytes = A.lib().hex_head_workspace_size(B, self.K, C)
        self.head_ws = torch.empty(self.head_ws_bytes, dtype=torch.uint8, device=dev)
        self.head_hw = hw

    def layer_input(self, l, x):
        if l == 0:
            return x
        return self.pooled[l - 1] if (l - 1) in self.pool_geo else self.act[l - 1]

    # ------------------------------------------------------------------ one training step
    def _tic(self):
        if self.timer is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def _toc(self, kind, l, e0):
        if e0 is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.timer.append((kind, l, e0, e))

    def _w(self, l, pass_id):
        """Weight pointer of a conv call: None (NULL) where the packed copy in the pass workspace is current."""
        return None if (l, pass_id) in self.packed else _p(self.weight(l))

    def forward(self, x, stream):
        L = A.lib()
        if self.pack_args is not None:
            self.pack_args.run(stream)
        for l in range(self.L):
            xin = self.layer_input(l, x)
            ws = self.ws[l][0]
            if l in self.pool_geo and self.fused_pool[l]:
                # conv -> ReLU -> max pool in one kernel: act[l] is never written (the backward needs
                # only the pooled tensor and the argmax, see backward())
                e0 = self._tic()
                A.check(L.hex_conv2d_fwd_maxpool(ctypes.byref(self.desc[l]), _p(xin), self._w(l, 0),
                                                 _p(self.bias(l)), 1, _p(self.pooled[l]), _p(self.argmax[l]),
                                                 _p(ws), self.ws_sizes[l][0], stream), f"conv{l + 1} fwd+pool")
                self._toc("fwd_pool", l, e0)
                continue
            e0 = self._tic()
            A.check(L.hex_conv2d_fwd(ctypes.byref(self.desc[l]), _p(xin), self._w(l, 0), _p(self.bias(l)), 1,
                                     _p(self.act[l]), _p(ws), self.ws_sizes[l][0], stream), f"conv{l + 1} fwd")
            self._toc("fwd", l, e0)
            if l in self.pool_geo:
                e0 = self._tic()
                A.check(L.hex_pool2d_fwd(ctypes.byref(self.pdesc[l]), _p(self.act[l]), _p(self.pooled[l]),
                                         _p(self.argmax[l]), stream), f"pool{l + 1} fwd")
                self._toc("pool_fwd", l, e0)

    def backward(self, x, labels, stream, hooks=None):
        """Head + backward of every layer.  `hooks(l)` is called after layer l's
        weight gradient is complete (used for the per-layer gradient allreduce)."""
        L = A.lib()
        C = self.channels[-1]
        g = self.grads
        A.check(L.hex_head_fwd_bwd(self.B, self.head_hw, C, self.K, _p(self.act[-1]),
                                   _p(self.params[self.head_w:]), _p(self.params[self.head_b:]), _p(labels),
                                   _p(self.loss), _p(self.dact[-1]), _p(g[self.head_w:]), _p(g[self.head_b:]),
                                   _p(self.head_ws), self.head_ws_bytes, stream), "head")
        if hooks:
            hooks(self.L)
        # The weight gradient of layer l and the backward-data chain (dgrad l, pool bwd, ...) are independent;
        # with HEXCNN_SIDE_BWD=1 the weight gradients run on a side stream that joins before the optimizer.
        main = torch.cuda.current_stream()
        side = self._side if self._side is not None else main
        side_h = ctypes.c_void_p(side.cuda_stream) if side is not main else stream
        for l in reversed(range(self.L)):
            wo, wn, bo, bn = self.seg[l]
            xin = self.layer_input(l, x)
            dy = self.dact[l]
            if side is not main:
                side.wait_stream(main)  # dy of layer l is complete
            with torch.cuda.stream(side):
                e0 = self._tic()
                A.check(L.hex_conv2d_bwd_weight(ctypes.byref(self.desc[l]), _p(xin), _p(dy), _p(g[wo:]), _p(g[bo:]),
                                                0, _p(self.ws[l][2]), self.ws_sizes[l][2], side_h),
                        f"conv{l + 1} wgrad")
                self._toc("wgrad", l, e0)
                if hooks:
                    hooks(l)  # the allreduce of layer l's bucket is ordered after it (current stream = side)
            if l == 0:
                break
            prev = l - 1
            e0 = self._tic()
            if prev in self.pool_geo:
                # dgrad into the pooled tensor, masked by pooled > 0 (== ReLU mask at the argmax cell)
                A.check(L.hex_conv2d_bwd_data(ctypes.byref(self.desc[l]), _p(dy), self._w(l, 1),
                                              _p(self.pooled[prev]), _p(self.dpool[prev]), _p(self.ws[l][1]),
                                              self.ws_sizes[l][1], stream), f"conv{l + 1} dgrad")
                self._toc("dgrad", l, e0)
                e0 = self._tic()
                A.check(L.hex_pool2d_bwd(ctypes.byref(self.pdesc[prev]), _p(self.dpool[prev]),
                                         _p(self.argmax[prev]), _p(self.dact[prev]), stream), f"pool{prev + 1} bwd")
                self._toc("pool_bwd", prev, e0)
            else:
                A.check(L.hex_conv2d_bwd_data(ctypes.byref(self.desc[l]), _p(dy), self._w(l, 1),
                                              _p(self.act[prev]), _p(self.dact[prev]), _p(self.ws[l][1]),
                                              self.ws_sizes[l][1], stream), f"conv{l + 1} dgrad")
                self._toc("dgrad", l, e0)
        if side is not main:
            main.wait_stream(side)

    def _segment_range(self, l):
        if l == self.L:
            return self.head_w, self.nparams - self.head_w
        wo, wn, bo, bn = self.seg[l]
        return wo, bo + bn - wo

    def _segment(self, l):
        off, n = self._segment_range(l)
        return self.grads[off:off + n]

    def _nvls_reduce(self, l):
        # layer l's bucket is summed on a side stream as soon as its weight gradient is written (an event on
        # the current stream), so the sum overlaps the backward of the earlier layers
        off, n = self._segment_range(l)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._nv_side.wait_event(ev)
        with torch.cuda.stream(self._nv_side):
            self._nv.allreduce(off, n, slot=l)

    def step(self, x, labels):
        """One SGD step on the batch (x: bf16 [B,H,W,1] NHWC, labels: int32 [B]).
        Returns the device loss tensor (mean CE of this rank's batch)."""
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        self.forward(x, stream)
        if self.reduce_grads and self._nv is not None:
            self.backward(x, labels, stream, self._nvls_reduce)
            torch.cuda.current_stream().wait_stream(self._nv_side)  # SGD reads the summed gradients
        elif self.reduce_grads:
            red = GradBucketReducer(self.pg)
            self.backward(x, labels, stream, lambda l: red.launch(self._segment(l)))
            red.wait_all()
        else:
            self.backward(x, labels, stream)
        A.check(A.lib().hex_sgd_momentum(self.nparams, _p(self.params), _p(self.grads), _p(self.mom),
                                         self.lr, self.mu, 1.0 / self.world, _p(self.params_bf16), stream), "sgd")
        return self.loss

    def graphed_step(self, x, labels):
        """Capture one training step on the static buffers (x, labels) in a CUDA graph and return
        (graph, loss): graph.replay() runs the whole step (every kernel of every layer, head, the
        per-layer NCCL or NVLS gradient sums when data parallel, and SGD) as one launch, without per-call
        host dispatch; refill x / labels in place between replays.  The warm-up call performs one real
        step (it also creates the NCCL communicator before capture).  Data parallel capture needs the
        NCCL backend (gloo collectives run on the host and cannot be captured) unless the sums run in the
        NVLS kernel."""
        if self.reduce_grads and self._nv is None and dist.get_backend(self.pg) != "nccl":
            raise RuntimeError("graphed_step: data-parallel capture needs the NCCL backend")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step(x, labels)  # first-call work (function attributes, allocator) outside the capture
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            loss = self.step(x, labels)
        return graph, loss

    # ------------------------------------------------------------------ accounting
    def pool_bytes(self, l, kind):
        """Algorithmic HBM bytes of one pool call after layer l (read inputs + write outputs once)."""
        h, w, ho, wo = self.pool_geo[l]
        C = self.channels[l + 1]
        full, pooled = self.B * h * w * C * 2, self.B * ho * wo * C * 2
        am = self.B * ho * wo * C
        return full + pooled + am  # fwd: read x, write y + argmax; bwd: read dy + argmax, write dx

    def l1_bytes(self, kind):
        """Algorithmic HBM bytes of a layer-1 (Cin = 1) call: fwd reads x and writes y;
        wgrad reads x and dy (the weight gradient itself is 5 KB)."""
        h, w = self.geo[0]
        px = self.B * h * w
        return px * 2 + px * self.channels[1] * 2

    def flops_per_image(self):
        """Algorithmic FLOPs per image of fwd + dgrad (L2..L6) + wgrad, counting
        in-grid taps only (valid taps)."""
        from .functional import gather_map
        total = 0.0
        per_layer = []
        for l in range(self.L):
            h, w = self.geo[l]
            vt = int((gather_map(h, w, self.ns[l], device=self.dev) >= 0).sum().item())
            f = 2.0 * vt * self.channels[l] * self.channels[l + 1]
            passes = 3 if l > 0 else 2
            per_layer.append((f, passes))
            total += f * passes
        return total, per_layer
