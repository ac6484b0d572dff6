"""Pre-allocated execution plans for the packed hot path (serving / bench).

A plan binds one packed layer to one input geometry, owns every device
buffer the step needs (packed activations, output, flag word, pinned host
staging) and issues only the sm_100a kernels of libbnn_b200.so -- no
allocation, no host sync -- so a step can be timed, replayed or captured in
a CUDA graph.  ``run_host`` is the end-to-end call a user makes with host
memory: H2D copy, sign+pack, xnor kernel, D2H copy, one synchronize, and the
reference's ValueError on non-finite input (bitpack.py:37-38).
"""

from __future__ import annotations


import time

import torch

from . import _lib
from .bitpack import words_per_bits
from .layers import QConv2d, QDense


class _Plan:
    launches_per_step = 2

    def _alloc_common(self):
        self.flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.flags_host = torch.zeros(1, dtype=torch.int32).pin_memory()

    def check_flags(self):
        """Raise the reference's ValueError for what the steps since the last check saw,
        then clear the flag word (the pack kernels only ever OR into it)."""
        f = int(self.flags.item())
        self.flags.zero_()
        if f & _lib.FLAG_NONFINITE:
            raise ValueError("binarize requires finite inputs")
        if f & _lib.FLAG_NOTSIGN:
            raise ValueError("matrix entries must all be -1 or +1")

    # batch slices the end-to-end call is pipelined over (H2D of slice i+1, compute of
    # slice i and D2H of slice i-1 overlap; PCIe is full duplex); 1 = no pipelining
    # "auto" (default): the first run_host call on a pinned buffer pair times 1 / 2 / 4 / 8
    # slices once and keeps the fastest (LeNet at batch 1024: 1 slice, 0.31 vs 0.43 ms with 4;
    # ResNet-18 at batch 256: 8 slices, 3.19 vs 3.31 ms; results are identical for any count)
    host_chunks = "auto"
    host_chunk_candidates = (1, 2, 4, 8)
    host_taper = None  # optional relative slice sizes overriding the equal split

    def run_host(self, x_host: torch.Tensor, y_host: torch.Tensor) -> torch.Tensor:
        """End to end from pinned host memory: H2D, pack, kernel, D2H, one sync.

        Plans whose leading dimension is a batch of independent items (ConvPlan,
        DensePlan) pipeline the copies against the compute over ``host_chunks``
        batch slices on three streams; the result is identical to one pass.  With
        pinned host buffers the whole schedule is captured once per (x_host,
        y_host) pair into a CUDA graph and replayed, so a call costs one launch.
        """
        pinned = x_host.is_pinned() and y_host.is_pinned()
        if self.host_chunks == "auto" and not self.host_taper:
            self.host_chunks = self._tune_host_chunks(x_host, y_host) if pinned else 4
        g = self._host_graph(x_host, y_host) if pinned else None
        cur = torch.cuda.current_stream()
        if g is not None:
            g.replay()
        else:
            self._host_schedule(x_host, y_host)
        cur.synchronize()
        f = int(self.flags_host[0])
        if f & _lib.FLAG_NONFINITE:
            raise ValueError("binarize requires finite inputs")
        return y_host

    def _host_graph(self, x_host: torch.Tensor, y_host: torch.Tensor):
        """The captured schedule of this (x_host, y_host, slicing); None if capture failed."""
        key = (x_host.data_ptr(), y_host.data_ptr(), self.host_chunks, tuple(self.host_taper or ()))
        graphs = self.__dict__.setdefault("_host_graphs", {})
        if key not in graphs:
            self._host_schedule(x_host, y_host)  # warm-up outside capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g):
                    self._host_schedule(x_host, y_host)
            except RuntimeError:
                g = None
            # the entry keeps the host buffers alive: the graph's copy nodes hold their
            # addresses, and a freed pinned block can come back at the same address
            graphs[key] = (g, x_host, y_host)
            while len(graphs) > 16:  # bounded: the oldest schedule (and its buffers) goes first
                graphs.pop(next(iter(graphs)))
        return graphs[key][0]

    def _tune_host_chunks(self, x_host: torch.Tensor, y_host: torch.Tensor) -> int:
        """Time the end-to-end schedule per slice count (host clock around replay + sync)."""
        if not hasattr(self, "run_device_range"):
            return 1
        cands = [c for c in self.host_chunk_candidates if c <= self.b]
        times = {}
        for _ in range(2):  # two passes: the first candidate is not the only one timed on cold clocks
            for c in cands:
                self.host_chunks = c
                g = self._host_graph(x_host, y_host)
                run = g.replay if g is not None else (lambda: self._host_schedule(x_host, y_host))
                run()
                torch.cuda.synchronize()
                for _ in range(5):  # one call at a time on the host clock, as run_host is used:
                    t0 = time.perf_counter()  # the launch cost of a many-node graph counts too
                    run()
                    torch.cuda.current_stream().synchronize()
                    t = (time.perf_counter() - t0) * 1e3
                    times[c] = min(t, times.get(c, t))
        best, best_ms = 1, None
        for c in cands:  # (more slices must win by 3% to be taken)
            if best_ms is None or times[c] < 0.97 * best_ms:
                best, best_ms = c, times[c]
        graphs = self.__dict__.get("_host_graphs", {})
        for c in self.host_chunk_candidates:  # drop the losing candidates' graphs
            if c != best:
                graphs.pop((x_host.data_ptr(), y_host.data_ptr(), c, ()), None)
        return best

    def _host_schedule(self, x_host: torch.Tensor, y_host: torch.Tensor):
        hc = 4 if self.host_chunks == "auto" else self.host_chunks
        chunks = min(len(self.host_taper) if self.host_taper else hc, self.b) \
            if hasattr(self, "run_device_range") else 1
        cur = torch.cuda.current_stream()
        self.flags.zero_()  # this call's flags only (a memset node inside the graph)
        if chunks <= 1:
            self.x.copy_(x_host, non_blocking=True)
            self.run_device()
            y_host.copy_(self.y, non_blocking=True)
        else:
            if not hasattr(self, "_streams"):
                self._streams = (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream())
            h2d, comp, d2h = self._streams
            for st in self._streams:
                st.wait_stream(cur)
            bounds = [self.b * i // chunks for i in range(chunks + 1)]
            if self.host_taper:  # relative slice sizes, e.g. (4, 2, 1): a short last slice = a short drain
                tot, acc, bounds = sum(self.host_taper), 0, [0]
                for wgt in self.host_taper:
                    acc += wgt
                    bounds.append(max(bounds[-1] + 1, self.b * acc // tot) if acc < tot else self.b)
                bounds = [min(v, self.b) for v in bounds]
            for i0, i1 in zip(bounds[:-1], bounds[1:]):
                with torch.cuda.stream(h2d):
                    self.x[i0:i1].copy_(x_host[i0:i1], non_blocking=True)
                comp.wait_stream(h2d)
                with torch.cuda.stream(comp):
                    self.run_device_range(i0, i1, comp.cuda_stream)
                d2h.wait_stream(comp)
                with torch.cuda.stream(d2h):
                    y_host[i0:i1].copy_(self.y[i0:i1], non_blocking=True)
            for st in self._streams:
                cur.wait_stream(st)
        self.flags_host.copy_(self.flags, non_blocking=True)

    @property
    def h2d_bytes(self) -> int:
        return self.x.numel() * self.x.element_size()

    @property
    def d2h_bytes(self) -> int:
        return self.y.numel() * self.y.element_size()


class ConvPlan(_Plan):
    """sign+pack (bnn_pack_nchw_f32) -> implicit-im2col conv (bnn_bconv2d)."""

    def __init__(self, layer: QConv2d, batch: int, h: int, w: int, strict: bool = False):
        self.layer = layer
        self.b, self.h, self.w = batch, h, w
        self.oh, self.ow = layer.output_hw(h, w)
        c = layer.in_channels
        self.x = torch.empty((batch, c, h, w), dtype=torch.float32, device="cuda")
        self.xw = torch.empty((batch, h, w, words_per_bits(c)), dtype=torch.uint64, device="cuda")
        self.y = torch.empty((batch, layer.filters, self.oh, self.ow), dtype=torch.float32,
                             device="cuda")
        self.wd = layer.device_weights()
        self.mode = _lib.PACK_STRICT if strict else _lib.PACK_SIGN
        self.algo = _lib.ALGOS[layer.algo] if isinstance(layer.algo, str) else layer.algo
        self._alloc_common()
        self.lib = _lib.load()
        kh, kw = layer.kernel
        self.m, self.n, self.k = layer.filters, batch * self.oh * self.ow, c * kh * kw
        # C % 256 == 0: scratch of the pre-expanded conv engine (its own buffer: run_host slices
        # run on several streams); the expansion pass is part of kernel()
        self.ws = None
        need = int(self.lib.bnn_bconv2d_ws_bytes(batch, c, h, w, layer.filters, kh, kw, layer.stride[0],
                                                 layer.stride[1], layer.pad[0], layer.pad[1]))
        if need > 0 and (self.algo == _lib.ALGO_UMMA_XP or (self.algo == _lib.ALGO_AUTO and c >= 256)):
            self.ws = torch.empty(need, dtype=torch.uint8, device="cuda")
            self.ws_slices = {}
            from .layers import make_epilogue
            self.ep = make_epilogue(layer.domain)
            self.launches_per_step = 3  # pack, expand, conv

    @property
    def binary_ops(self) -> int:
        return 2 * self.m * self.n * self.k

    def pack(self, stream: int | None = None):
        s = _lib.stream_ptr() if stream is None else stream
        L = self.layer
        _lib.check(self.lib.bnn_pack_nchw_f32(self.x.data_ptr(), self.b, L.in_channels, self.h,
                                              self.w, self.xw.data_ptr(), self.mode,
                                              self.flags.data_ptr(), s), "pack")

    def kernel(self, stream: int | None = None):
        s = _lib.stream_ptr() if stream is None else stream
        L = self.layer
        kh, kw = L.kernel
        if self.ws is not None:
            import ctypes
            _lib.check(self.lib.bnn_bconv2d_ws(self.xw.data_ptr(), self.b, L.in_channels, self.h,
                                               self.w, self.wd.data_ptr(), L.filters, kh, kw,
                                               L.stride[0], L.stride[1], L.pad[0], L.pad[1],
                                               self.y.data_ptr(), ctypes.byref(self.ep), self.algo,
                                               self.ws.data_ptr(), self.ws.numel(), s), "bconv2d_ws")
            return
        _lib.check(self.lib.bnn_bconv2d(self.xw.data_ptr(), self.b, L.in_channels, self.h,
                                        self.w, self.wd.data_ptr(), L.filters, kh, kw,
                                        L.stride[0], L.stride[1], L.pad[0], L.pad[1],
                                        self.y.data_ptr(), L.domain, None, None, self.algo, s),
                   "bconv2d")

    def run_device(self):
        self.pack()
        self.kernel()
        return self.y

    def run_device_range(self, i0: int, i1: int, stream: int):
        """pack + conv of images [i0, i1) only (images are independent)."""
        L = self.layer
        kh, kw = L.kernel
        nb = i1 - i0
        x = self.x[i0:i1]
        xw = self.xw[i0:i1]
        y = self.y[i0:i1]
        _lib.check(self.lib.bnn_pack_nchw_f32(x.data_ptr(), nb, L.in_channels, self.h, self.w,
                                              xw.data_ptr(), self.mode, self.flags.data_ptr(),
                                              stream), "pack")
        if self.ws is not None:
            import ctypes
            # one scratch per image range: the slices of a pipelined run overlap on streams
            ws = self.ws_slices.get((i0, i1))
            if ws is None:
                ws = torch.empty(int(self.lib.bnn_bconv2d_ws_bytes(
                    nb, L.in_channels, self.h, self.w, L.filters, kh, kw, L.stride[0], L.stride[1],
                    L.pad[0], L.pad[1])), dtype=torch.uint8, device="cuda")
                self.ws_slices[(i0, i1)] = ws
            _lib.check(self.lib.bnn_bconv2d_ws(xw.data_ptr(), nb, L.in_channels, self.h, self.w,
                                               self.wd.data_ptr(), L.filters, kh, kw, L.stride[0],
                                               L.stride[1], L.pad[0], L.pad[1], y.data_ptr(),
                                               ctypes.byref(self.ep), self.algo, ws.data_ptr(),
                                               ws.numel(), stream), "bconv2d_ws")
            return
        _lib.check(self.lib.bnn_bconv2d(xw.data_ptr(), nb, L.in_channels, self.h, self.w,
                                        self.wd.data_ptr(), L.filters, kh, kw, L.stride[0],
                                        L.stride[1], L.pad[0], L.pad[1], y.data_ptr(), L.domain,
                                        None, None, self.algo, stream), "bconv2d")


class DensePlan(_Plan):
    """sign+pack rows (bnn_pack_rows_f32) -> xnor GEMM (bnn_xnor_gemm), out [B, units]."""

    def __init__(self, layer: QDense, batch: int, strict: bool = False,
                 host_splitk: int | None = None):
        self.layer = layer
        self.b = batch
        k = layer.in_features
        self.x = torch.empty((batch, k), dtype=torch.float32, device="cuda")
        self.xw = torch.empty((batch, words_per_bits(k)), dtype=torch.uint64, device="cuda")
        self.y = torch.empty((batch, layer.units), dtype=torch.float32, device="cuda")
        layer._require_packed()
        self.wa = layer.packed.words
        self.mode = _lib.PACK_STRICT if strict else _lib.PACK_SIGN
        self.algo = _lib.ALGOS[layer.algo] if isinstance(layer.algo, str) else layer.algo
        self._alloc_common()
        self.lib = _lib.load()
        self.m, self.n, self.k = layer.units, batch, k
        self.chunks = self._k_chunks(host_splitk) if self.algo == _lib.ALGOS["auto"] \
            else [(0, self.k)]
        if len(self.chunks) > 1:
            self.part = torch.empty((len(self.chunks), batch, layer.units), dtype=torch.float32,
                                    device="cuda")
            self._kstreams = [torch.cuda.Stream() for _ in self.chunks]
            self.launches_per_step = 2 + len(self.chunks)

    def _k_chunks(self, splits):
        """Host split-K (opt-in, ``host_splitk=<ranges>``): word-aligned K ranges of
        >= 512 bits run as popcount-domain GEMMs on forked streams and
        bnn_sum_partials_f32 adds the exact integer counts (bit-identical to one
        launch).  Meant for GEMMs with too few output tiles to fill the SMs
        (config 1: 16 tiles of 128 x 128 on 148 SMs), but measured slower there
        (tools/splitk_diag.py, profiles/r01/splitk_c1.txt): a K=512 launch costs
        8.3 us against 16.4 us for all of K=4096 -- the per-launch fixed latency
        dominates -- and the engine already spreads config 1 over 128 CTAs
        (128 x 16 tiles), so the forked launches cannot overlap.  Off by default."""
        words = words_per_bits(self.k)
        if splits is None:
            return [(0, self.k)]
        splits = min(int(splits), words // 4)
        if splits < 2:
            return [(0, self.k)]
        step = -(-words // splits)
        step = -(-step // 4) * 4  # whole 256-bit superstages per range
        return [(64 * w0, min(self.k, 64 * (w0 + step))) for w0 in range(0, words, step)]

    @property
    def binary_ops(self) -> int:
        return 2 * self.m * self.n * self.k

    def pack(self, stream: int | None = None):
        s = _lib.stream_ptr() if stream is None else stream
        _lib.check(self.lib.bnn_pack_rows_f32(self.x.data_ptr(), self.b, self.k, self.k,
                                              self.xw.data_ptr(), self.xw.shape[1], 0, self.mode,
                                              None, self.flags.data_ptr(), s), "pack")

    def kernel(self, stream: int | None = None):
        s = _lib.stream_ptr() if stream is None else stream
        if len(self.chunks) > 1 and stream is None:
            return self._kernel_split()
        _lib.check(self.lib.bnn_xnor_gemm(self.wa.data_ptr(), self.wa.shape[1], self.xw.data_ptr(),
                                          self.xw.shape[1], self.m, self.n, self.k, 0, 0,
                                          self.y.data_ptr(), 1, self.m, self.layer.domain, None,
                                          None, self.algo, s), "xnor_gemm")

    def _kernel_split(self):
        cur = torch.cuda.current_stream()
        for i, ((k0, k1), st) in enumerate(zip(self.chunks, self._kstreams)):
            st.wait_stream(cur)
            w0 = k0 // 64
            _lib.check(self.lib.bnn_xnor_gemm(
                self.wa.data_ptr() + 8 * w0, self.wa.shape[1], self.xw.data_ptr() + 8 * w0,
                self.xw.shape[1], self.m, self.n, k1 - k0, 0, 0, self.part[i].data_ptr(), 1,
                self.m, _lib.POPCOUNT, None, None, self.algo, st.cuda_stream), "xnor_gemm")
        for st in self._kstreams:
            cur.wait_stream(st)
        _lib.check(self.lib.bnn_sum_partials_f32(self.part.data_ptr(), len(self.chunks),
                                                 self.y.numel(), self.y.numel(), self.layer.domain,
                                                 self.k, self.y.data_ptr(), cur.cuda_stream),
                   "sum_partials")

    def run_device(self):
        self.pack()
        self.kernel()
        return self.y

    def run_device_range(self, i0: int, i1: int, stream: int):
        """sign+pack and GEMM of batch rows [i0, i1) (rows are independent)."""
        nb = i1 - i0
        x, xw, y = self.x[i0:i1], self.xw[i0:i1], self.y[i0:i1]
        _lib.check(self.lib.bnn_pack_rows_f32(x.data_ptr(), nb, self.k, self.k, xw.data_ptr(),
                                              self.xw.shape[1], 0, self.mode, None,
                                              self.flags.data_ptr(), stream), "pack")
        _lib.check(self.lib.bnn_xnor_gemm(self.wa.data_ptr(), self.wa.shape[1], xw.data_ptr(),
                                          self.xw.shape[1], self.m, nb, self.k, 0, 0,
                                          y.data_ptr(), 1, self.m, self.layer.domain, None,
                                          None, self.algo, stream), "xnor_gemm")


class GemmPlan(_Plan):
    """Square / long-K binary GEMM on pre-packed operands (config 5): one kernel."""

    launches_per_step = 1

    def __init__(self, a_rows: torch.Tensor, b_rows: torch.Tensor, k: int, algo="auto",
                 domain: int = _lib.POPCOUNT):
        self.a, self.bw = a_rows, b_rows
        self.m, self.n, self.k = a_rows.shape[0], b_rows.shape[0], k
        self.x = b_rows  # the per-step input is the packed activation matrix
        self.y = torch.empty((self.m, self.n), dtype=torch.float32, device="cuda")
        self.algo = _lib.ALGOS[algo] if isinstance(algo, str) else algo
        self.domain = domain
        self._alloc_common()
        self.lib = _lib.load()
        # large shapes: scratch for the pre-expanded engine (bnn_xnor_gemm_ws); both the
        # expansion pass and the GEMM run inside every step
        self.ws = None
        from .gemm import xp_eligible
        if self.algo == _lib.ALGO_UMMA_XP or (self.algo == _lib.ALGO_AUTO and
                                              xp_eligible(self.m, self.n, self.k)):
            self.ws = torch.empty(int(self.lib.bnn_xnor_gemm_ws_bytes(self.m, self.n, self.k)),
                                  dtype=torch.uint8, device="cuda")
            self.launches_per_step = 2

    @property
    def binary_ops(self) -> int:
        return 2 * self.m * self.n * self.k

    def pack(self, stream=None):
        pass

    def kernel(self, stream: int | None = None):
        s = _lib.stream_ptr() if stream is None else stream
        if self.ws is not None:
            _lib.check(self.lib.bnn_xnor_gemm_ws(self.a.data_ptr(), self.a.stride(0),
                                                 self.bw.data_ptr(), self.bw.stride(0), self.m,
                                                 self.n, self.k, 0, 0, self.y.data_ptr(), self.n, 1,
                                                 self.domain, self.algo, self.ws.data_ptr(),
                                                 self.ws.numel(), s), "xnor_gemm_ws")
            return
        _lib.check(self.lib.bnn_xnor_gemm(self.a.data_ptr(), self.a.stride(0), self.bw.data_ptr(),
                                          self.bw.stride(0), self.m, self.n, self.k, 0, 0,
                                          self.y.data_ptr(), self.n, 1, self.domain, None, None,
                                          self.algo, s), "xnor_gemm")

    def run_device(self):
        self.kernel()
        return self.y


class BitplanePlan(_Plan):
    """Multi-bit (act_bit = weight_bit = 2) GEMM on pre-packed bit planes (config 5)."""

    launches_per_step = 1

    def __init__(self, a_planes: torch.Tensor, b_planes: torch.Tensor, k: int,
                 a_grid: str = "unsigned", b_grid: str = "unsigned"):
        self.a, self.bw = a_planes, b_planes
        self.bits, self.m, _ = a_planes.shape
        self.n, self.k = b_planes.shape[1], k
        self.x = b_planes
        self.y = torch.empty((self.m, self.n), dtype=torch.float32, device="cuda")
        self.grids = (a_grid, b_grid)
        self._alloc_common()
        from .gemm import xp_eligible
        self.ws = None  # large shapes: scratch of the pre-expanded engine (bnn_bitplane_gemm_ws)
        if xp_eligible(self.m, self.n, self.k):
            self.ws = torch.empty(int(_lib.load().bnn_xnor_gemm_ws_bytes(self.m, self.n, self.k)),
                                  dtype=torch.uint8, device="cuda")
            self.launches_per_step = 2

    @property
    def binary_ops(self) -> int:
        return 2 * self.m * self.n * self.k  # logical 2MNK (plane ops = x bits^2)

    def pack(self, stream=None):
        pass

    def kernel(self, stream=None):
        from .gemm import bitplane_gemm
        bitplane_gemm(self.a, self.bw, self.k, a_grid=self.grids[0], b_grid=self.grids[1],
                      out=self.y, workspace_in=self.ws)

    def run_device(self):
        self.kernel()
        return self.y


def _count_lib_launches(fn) -> int:
    from . import _lib
    n = [0]
    real_call, real_status = _lib.call, _lib.call_status
    quiet = ("bnn_set_", "bnn_debug_set", "bnn_last_error", "bnn_status_string", "bnn_abi_version",
             "bnn_conv_channel_words", "bnn_device_sm_count")

    kernels_per_call = {"bnn_avgpool_fc_f32": 2}  # entry points launching > 1 kernel

    def counted(f):
        def wrap(name, *args):
            if not name.startswith(quiet):
                n[0] += kernels_per_call.get(name, 1)
            return f(name, *args)
        return wrap

    _lib.call, _lib.call_status = counted(real_call), counted(real_status)
    try:
        fn()
    finally:
        _lib.call, _lib.call_status = real_call, real_status
    return n[0]


class NetPlan(_Plan):
    """Whole-network inference step (LeNet C3 / ResNet-18 C4) on a resident batch.

    Binary layers run without per-layer host syncs (sync_checks = False) and
    share one flag word, read once by check_flags / run_host.
    """

    def __init__(self, net, batch: int, chw):
        from .layers import INFER_PACKED
        from .nets import binary_ops_per_image
        self.net, self.b, self.chw = net, batch, tuple(chw)
        self.mode = INFER_PACKED
        self._alloc_common()
        for layer in net.binary_layers():
            layer.sync_checks = False
            layer.flags = self.flags
        # zeros, not empty: the warm-up forward below must not see NaN bit patterns
        self.x = torch.zeros((batch,) + self.chw, dtype=torch.float32, device="cuda")
        self.ops_per_image = binary_ops_per_image(net, self.chw)
        self.y = net.forward(self.x, self.mode)  # (first call: weight re-layouts, probes)
        # this library's kernel launches per step: every C-ABI compute call of a warm
        # forward launches one kernel (the float layers' torch kernels are not counted)
        self.launches_per_step = _count_lib_launches(lambda: net.forward(self.x, self.mode))

    @property
    def binary_ops(self) -> int:
        return self.b * self.ops_per_image

    def pack(self, stream=None):
        pass

    def kernel(self, stream=None):
        out = self.net.forward(self.x, self.mode)
        self.y.copy_(out)
        return self.y

    def run_device(self):
        return self.kernel()

    # end to end: the batch is pipelined over slices (images are independent; the
    # classifier head's per-image order makes every slice's logits equal the full
    # batch's), H2D of slice i+1 under the forward of slice i; the slice count is tuned on
    # the first call (_Plan.host_chunks = "auto")

    def run_device_range(self, i0: int, i1: int, stream: int):
        """Forward of images [i0, i1) on the current stream (the caller's context)."""
        out = self.net.forward(self.x[i0:i1], self.mode)
        self.y[i0:i1].copy_(out)

    def kernel_breakdown(self):
        """One forward with CUDA events around every C-ABI compute call, measured on the
        launching stream while a leading sleep kernel holds the GPU until the whole
        forward is queued (so no host launch gap lands inside an interval).  Returns
        [(entry point, ms, binary ops)]; binary ops for the GEMM / conv calls (2MNK),
        0 otherwise."""
        from . import _lib
        recs = []
        real_call, real_status = _lib.call, _lib.call_status
        quiet = ("bnn_set_", "bnn_debug_set", "bnn_last_error", "bnn_status_string",
                 "bnn_abi_version", "bnn_conv_channel_words", "bnn_device_sm_count")

        def ops_of(name, a):
            if name.startswith("bnn_bconv2d"):
                B, C, H, W, F, kh, kw, sh, sw, ph, pw = a[1:5] + a[6:13]
                oh, ow = (H + 2 * ph - kh) // sh + 1, (W + 2 * pw - kw) // sw + 1
                return 2 * F * B * oh * ow * C * kh * kw
            if name.startswith("bnn_xnor_gemm"):
                return 2 * a[4] * a[5] * a[6]
            return 0

        def timed(f):
            def wrap(name, *a):
                if name.startswith(quiet):
                    return f(name, *a)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                r = f(name, *a)
                e.record()
                recs.append((name, s, e, ops_of(name, a)))
                return r
            return wrap

        torch.cuda.synchronize()
        torch.cuda._sleep(200_000_000)  # ~0.1 s at ~2 GHz: the forward queues behind it
        _lib.call, _lib.call_status = timed(real_call), timed(real_status)
        try:
            self.net.forward(self.x, self.mode)
        finally:
            _lib.call, _lib.call_status = real_call, real_status
        torch.cuda.synchronize()
        return [(n, s.elapsed_time(e), ops) for n, s, e, ops in recs]


class NsplitGemmPlan(_Plan):
    """Config-5 GEMM on N GPUs: this rank's N shard of the packed
    activations, one tcgen05 GEMM into its N-major [shard, M] output, then one
    all-gather of the shards into the full [N, M] result on every rank
    (parallel.NsplitGemm).  Bit-identical to the one-GPU GEMM for any world size."""

    launches_per_step = 1
    graph_ok = False  # the step contains a collective: replayed eagerly

    def __init__(self, a_rows: torch.Tensor, b_shard: torch.Tensor, k: int, n_total: int,
                 algo="auto", group=None):
        from .parallel import NsplitGemm
        self.ns = NsplitGemm(a_rows, b_shard, k, n_total, group=group, algo=algo)
        self.m, self.n, self.k = self.ns.m, n_total, k
        self.x = b_shard
        self.y = self.ns.full[:n_total]
        self.b = b_shard.shape[-2]
        self._alloc_common()
        self.gather_ms = []

    @property
    def binary_ops(self) -> int:
        return 2 * self.m * self.n * self.k  # whole-job work (all shards)

    @property
    def local_ops(self) -> int:
        return 2 * self.m * (self.ns.n1 - self.ns.n0) * self.k

    def pack(self, stream=None):
        pass

    def kernel(self, stream=None):
        self.ns.compute()

    def run_device(self):
        self.ns.compute()
        return self.ns.gather()

    def run_host(self, x_host: torch.Tensor, y_host: torch.Tensor) -> torch.Tensor:
        """H2D of this rank's packed B shard, GEMM, all-gather, D2H of the full [N, M]
        result; eager (no graph around the collective)."""
        self.x.copy_(x_host, non_blocking=True)
        self.run_device()
        y_host.copy_(self.y[: self.n], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return y_host
