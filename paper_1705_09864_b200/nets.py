"""Whole-network inference runners built on the packed hot path.

* ``lenet_c3`` -- BASELINE configs[2]: full-precision conv5x5(1->64, pad 2) +
  tanh + maxpool, QActivation + QConvolution5x5(64->64, pad 2, 1 bit) + BN +
  maxpool, QFullyConnected(3136->1000, 1 bit) + BN, full-precision FC(1000->10).
* ``resnet18_c4`` -- BASELINE configs[3]: binary ResNet-18; the stem conv and
  the classifier are full precision, every other conv (3x3 and the 1x1
  downsamples) is a 1-bit QConvolution preceded by the sign activation and
  followed by BatchNorm; basic block  out = BN(QConv(sign(BN(QConv(sign(x)))))) + shortcut.

Float layers mirror the reference's inference semantics (layers.py:81-141,
422-659): convolutions/dense in float32 with TF32 off, BatchNorm with running
statistics in the reference's op order  gamma * ((x - mean) * inv_std) + beta
(layers.py:596-602).  They run as torch ops -- they are not the hot path;
every binary layer runs the sm_100a kernels in ``infer_packed`` mode and the
float-path equivalent in ``infer_float`` mode, so the two modes must agree
exactly at every binary layer (the reference's cross-mode property,
test_layers.py:181-220).  Weights are random-init with NumPy generators
(layers._uniform_init rule) -- there is no network access for checkpoints.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib
from .layers import (INFER_FLOAT, INFER_PACKED, PackedNHWC, QConvolution, QFullyConnected,
                     _check_mode, _float_matmul, _uniform_init)

BN_EPS = 1e-5  # layers.py:36


def _t(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


class _Lazy:
    """Host (NumPy) parameters, uploaded to the GPU on first use (the CPU
    reference can build the same network without a device)."""

    def _dev(self, name):
        cache = self.__dict__.setdefault("_dev_cache", {})
        if name not in cache:
            a = getattr(self, name)
            cache[name] = None if a is None else _t(a)
        return cache[name]


class Conv2d(_Lazy):
    """Full-precision convolution (layers.py:81-141), NCHW f32.

    ``k``, ``stride`` and ``pad`` are ints or (h, w) pairs, like the reference's
    ``Conv2d(cin, cout, (kh, kw), stride=(sh, sw), pad=(ph, pw))``.
    ``engine="tc"`` (default where supported: 64 filters, C*kh*kw <= 320 -- the
    ResNet-18 and LeNet stems): ``bnn_conv2d_f32_tc``, tcgen05 kind::tf32 with a
    three-term hi/lo split (f32 accuracy).  ``engine="cudnn"``: cuDNN f32 with
    TF32 off.  Both modes of a network use the same engine, so the cross-mode
    exactness of the binary layers is unaffected.
    """

    engine = "tc"

    def __init__(self, cin, cout, k, stride=1, pad=0, bias=True, rng=None):
        self.cin, self.cout = cin, cout
        self.kh, self.kw = _pair(k)
        self.stride, self.pad = stride, pad
        fan_in, fan_out = cin * self.kh * self.kw, cout * self.kh * self.kw
        shape = (cout, cin, self.kh, self.kw)
        self.weight = _uniform_init(rng, shape, fan_in, fan_out) if rng is not None \
            else np.zeros(shape, np.float32)
        self.bias = np.zeros(cout, np.float32) if bias else None

    # (stride / pad may be re-assigned as ints or pairs, e.g. by the .bmx reader)
    @property
    def sh(self):
        return _pair(self.stride)[0]

    @property
    def sw(self):
        return _pair(self.stride)[1]

    @property
    def ph(self):
        return _pair(self.pad)[0]

    @property
    def pw(self):
        return _pair(self.pad)[1]

    def output_hw(self, h, w):
        return ((h + 2 * self.ph - self.kh) // self.sh + 1,
                (w + 2 * self.pw - self.kw) // self.sw + 1)

    def geometry(self):
        """(kh, kw, sh, sw, ph, pw) in the C ABI's argument order."""
        return self.kh, self.kw, self.sh, self.sw, self.ph, self.pw

    def tc_supported(self) -> bool:
        return self.cout == 64 and self.cin * self.kh * self.kw <= 320

    def forward(self, x, mode=INFER_FLOAT):
        if self.engine == "tc" and self.tc_supported():
            x = x.contiguous()
            b, c, h, w = x.shape
            oh, ow = self.output_hw(h, w)
            y = torch.empty((b, self.cout, oh, ow), dtype=torch.float32, device=x.device)
            _lib.call("bnn_conv2d_f32_tc", _lib.ptr(x), b, c, h, w, _lib.ptr(self._dev("weight")),
                      _lib.ptr(self._dev("bias")), self.cout, *self.geometry(), _lib.ptr(y),
                      _lib.stream_ptr())
            return y
        prev = torch.backends.cudnn.allow_tf32
        torch.backends.cudnn.allow_tf32 = False
        torch.backends.cudnn.benchmark = True  # fastest exact-fp32 algorithm for the shape
        try:
            return F.conv2d(x, self._dev("weight"), self._dev("bias"), stride=(self.sh, self.sw),
                            padding=(self.ph, self.pw))
        finally:
            torch.backends.cudnn.allow_tf32 = prev


def _pair(v):
    if isinstance(v, (tuple, list)):
        if len(v) != 2:
            raise ValueError(f"expected an int or an (h, w) pair, got {v!r}")
        return int(v[0]), int(v[1])
    return int(v), int(v)


class Dense(_Lazy):
    """Full-precision linear layer y = x W^T + b (layers.py:266-317)."""

    def __init__(self, fin, fout, bias=True, rng=None):
        self.weight = _uniform_init(rng, (fout, fin), fin, fout) if rng is not None else \
            np.zeros((fout, fin), np.float32)
        self.bias = np.zeros(fout, np.float32) if bias else None

    def forward(self, x, mode=INFER_FLOAT):
        y = _float_matmul(x, self._dev("weight").T)
        b = self._dev("bias")
        return y + b if b is not None else y


class BatchNorm(_Lazy):
    """Inference BatchNorm in the reference op order (layers.py:587-602)."""

    def __init__(self, channels, rng=None):
        if rng is not None:  # randomised running stats as gen_golden.py:46-52 does
            self.gamma = (0.5 + rng.random(channels)).astype(np.float32)
            self.beta = (rng.standard_normal(channels) * 0.1).astype(np.float32)
            self.mean = (rng.standard_normal(channels) * 0.05).astype(np.float32)
            self.var = (0.5 + rng.random(channels)).astype(np.float32)
        else:
            self.gamma = np.ones(channels, np.float32)
            self.beta = np.zeros(channels, np.float32)
            self.mean = np.zeros(channels, np.float32)
            self.var = np.ones(channels, np.float32)
        self.inv_std = (1.0 / np.sqrt(self.var + np.float32(BN_EPS))).astype(np.float32)

    def device_params(self):
        """(mean, inv_std, gamma, beta) CUDA tensors for the fused conv / GEMM epilogue."""
        return self._dev("mean"), self._dev("inv_std"), self._dev("gamma"), self._dev("beta")

    def forward(self, x, mode=INFER_FLOAT):
        shape = (1, -1, 1, 1) if x.dim() == 4 else (1, -1)
        xhat = (x - self._dev("mean").view(shape)) * self._dev("inv_std").view(shape)
        return self._dev("gamma").view(shape) * xhat + self._dev("beta").view(shape)


class Tanh:
    def forward(self, x, mode=INFER_FLOAT):
        return torch.tanh(x)


class ReLU:
    def forward(self, x, mode=INFER_FLOAT):
        return torch.relu(x)


class MaxPool2d:
    def __init__(self, k, stride=None, pad=0):
        self.k, self.stride, self.pad = k, stride or k, pad

    def forward(self, x, mode=INFER_FLOAT):
        return F.max_pool2d(x, self.k, self.stride, self.pad)


class Flatten:
    def forward(self, x, mode=INFER_FLOAT):
        return x.reshape(x.shape[0], -1)  # NCHW flatten order (layers.py:459)


class GlobalAvgPool:
    def forward(self, x, mode=INFER_FLOAT):
        return x.mean(dim=(2, 3))


def avgpool_dense(x: torch.Tensor, dense: "Dense") -> torch.Tensor:
    """GlobalAvgPool -> Dense as one kernel (bnn_avgpool_fc_f32), used in both modes:
    each image's logits are summed in an order of their own, so batch shards of a
    network (multi-GPU batch sharding) reproduce the one-GPU logits bit for bit."""
    x = x.contiguous()
    b, c, h, w = x.shape
    wt = dense._dev("weight")
    y = torch.empty((b, wt.shape[0]), dtype=torch.float32, device=x.device)
    pooled = torch.empty((b, c), dtype=torch.float32, device=x.device)
    _lib.call("bnn_avgpool_fc_f32", _lib.ptr(x), b, c, h * w, _lib.ptr(wt),
              _lib.ptr(dense._dev("bias")), wt.shape[0], _lib.ptr(y), _lib.ptr(pooled),
              _lib.stream_ptr())
    return y


class StemPost:
    """BatchNorm -> ReLU -> MaxPool of a full-precision stem as one kernel in
    ``infer_packed`` mode (bnn_bn_relu_maxpool_f32, bit-identical); the three
    torch ops in ``infer_float`` mode."""

    def __init__(self, channels, rng, k=3, stride=2, pad=1):
        self.bn, self.relu, self.pool = BatchNorm(channels, rng), ReLU(), MaxPool2d(k, stride, pad)

    def fusable(self, conv: "Conv2d") -> bool:
        """The fused conv + post-op kernel covers the tensor-core conv with a 3x3/2/1
        pool (ResNet-18's stem)."""
        p = self.pool
        return (conv.engine == "tc" and conv.tc_supported() and conv.bias is None and
                (p.k, p.stride, p.pad) == (3, 2, 1))

    def forward_fused_conv(self, conv: "Conv2d", x: torch.Tensor, pack: bool = False,
                           flags: torch.Tensor | None = None):
        """maxpool(relu(BN(conv(x)))) in one kernel (bnn_conv_bn_relu_maxpool_f32_tc):
        the pool runs on sign-adjusted conv outputs before the BatchNorm, which is
        exact because the rounded BN + ReLU is monotone per channel."""
        x = x.contiguous()
        b, c, h, w = x.shape
        oh, ow = conv.output_hw(h, w)
        ph, pw = (oh - 1) // 2 + 1, (ow - 1) // 2 + 1
        y = torch.empty((b, conv.cout, ph, pw), dtype=torch.float32, device=x.device)
        mean, inv, gamma, beta = self.bn.device_params()
        args = (_lib.ptr(x), b, c, h, w, _lib.ptr(conv._dev("weight")), conv.cout,
                *conv.geometry(), _lib.ptr(mean),
                _lib.ptr(inv), _lib.ptr(gamma), _lib.ptr(beta), 1, _lib.ptr(y))
        if pack and conv.cout == 64:  # + the sign-packed words of y for the first block
            words = torch.empty((b, ph, pw, 1), dtype=torch.uint64, device=x.device)
            st = _lib.call_status("bnn_conv_bn_relu_maxpool_pack_f32_tc", *args, _lib.ptr(words),
                                  _lib.ptr(flags), _lib.stream_ptr())
            if st == _lib.OK:
                return PackedNHWC(words, y.shape, y)
        else:
            st = _lib.call_status("bnn_conv_bn_relu_maxpool_f32_tc", *args, _lib.stream_ptr())
        if st == _lib.EUNSUP:  # shape outside the fused kernel: two kernels
            return self.forward(conv.forward(x), INFER_PACKED)
        _lib.check(st, "bnn_conv_bn_relu_maxpool_f32_tc")
        return y

    def forward(self, x, mode=INFER_FLOAT):
        if mode != INFER_PACKED:
            return self.pool.forward(self.relu.forward(self.bn.forward(x)))
        x = x.contiguous()
        b, c, h, w = x.shape
        p = self.pool
        oh, ow = (h + 2 * p.pad - p.k) // p.stride + 1, (w + 2 * p.pad - p.k) // p.stride + 1
        y = torch.empty((b, c, oh, ow), dtype=torch.float32, device=x.device)
        mean, inv, gamma, beta = self.bn.device_params()
        _lib.call("bnn_bn_relu_maxpool_f32", _lib.ptr(x), b, c, h, w, _lib.ptr(mean),
                  _lib.ptr(inv), _lib.ptr(gamma), _lib.ptr(beta), 1, p.k, p.stride, p.pad,
                  _lib.ptr(y), _lib.stream_ptr())
        return y


class Sequential:
    def __init__(self, layers):
        self.layers = list(layers)

    fuse_bn = True  # infer_packed: a binary layer's following BatchNorm runs in its epilogue
    fuse_stem = True  # infer_packed: float stem conv + StemPost as one tensor-core kernel
    # opt-in: LeNet's fused stem pools before the tanh where the device's tanhf probes monotone
    # (1.2 s exhaustive probe once per process; stem 130 -> 112 us; this pool's B200 / CUDA 12.9
    # tanhf probes NOT monotone, so the switch then changes nothing)
    pool_first = False

    def forward(self, x, mode=INFER_FLOAT, capture=None):
        if capture is not None:  # per-layer capture reads every block's f32 output
            saved = [(l, l.needs_f32_out) for l in self.layers if isinstance(l, BinaryBasicBlock)]
            for l, _ in saved:
                l.needs_f32_out = True
            try:
                return self._forward(x, mode, capture)
            finally:
                for l, v in saved:
                    l.needs_f32_out = v
        return self._forward(x, mode, capture)

    def _forward(self, x, mode=INFER_FLOAT, capture=None):
        i, n = 0, len(self.layers)
        while i < n:
            layer = self.layers[i]
            nxt = self.layers[i + 1] if i + 1 < n else None
            if isinstance(x, PackedNHWC) and not isinstance(layer, BinaryBasicBlock) and not (
                    mode == INFER_PACKED and self.fuse_bn and _binary_pool_fc(self.layers[i:i + 6])):
                x = x.float()  # a float consumer of a packed activation
            if isinstance(layer, GlobalAvgPool) and isinstance(nxt, Dense) and x.dim() == 4:
                x = avgpool_dense(x, nxt)  # classifier head, one kernel (both modes)
                if capture is not None:
                    capture += [None, x]
                i += 2
                continue
            if mode == INFER_PACKED and self.fuse_stem and _lenet_stem(self.layers[i:i + 3]):
                # conv + tanh + maxpool, one kernel; a binary conv behind it reads only the sign
                # bits, which the same kernel packs (no f32 tensor, no pack pass)
                nb = self.fuse_bn and _binary_pool_fc(self.layers[i + 3:i + 9])
                x = _lenet_stem_forward(self.layers[i], x, pool_first=self.pool_first and _pool_first_ok(),
                                        pack=nb,
                                        f32_out=capture is not None,
                                        flags=self.layers[i + 3]._flags() if nb else None)
                if capture is not None:
                    capture += [None, None, x.f32 if isinstance(x, PackedNHWC) else x]
                i += 3
                continue
            if mode == INFER_PACKED and self.fuse_bn and _binary_pool_fc(self.layers[i:i + 6]):
                # QConv -> BN -> maxpool -> flatten -> QFC -> BN with 1-bit activations
                # between the two binary layers (sign-pack epilogue, packed OR-pool)
                x = _binary_pool_fc_forward(self.layers[i:i + 6], x)
                if capture is not None:
                    capture += [None] * 5 + [x]
                i += 6
                continue
            if (mode == INFER_PACKED and self.fuse_stem and isinstance(layer, Conv2d)
                    and isinstance(nxt, StemPost) and nxt.fusable(layer)):
                after = self.layers[i + 2] if i + 2 < n else None
                pack = isinstance(after, BinaryBasicBlock) and after.fused and after.packed_io
                # conv + BN + ReLU + maxpool (+ the first block's sign-pack), one kernel
                x = nxt.forward_fused_conv(layer, x, pack=pack,
                                           flags=after.conv1._flags() if pack else None)
                if capture is not None:
                    capture.append(None)
                    capture.append(x.float() if isinstance(x, PackedNHWC) else x)
                i += 2
                continue
            if (mode == INFER_PACKED and self.fuse_bn and isinstance(nxt, BatchNorm)
                    and isinstance(layer, (QConvolution, QFullyConnected)) and layer.bits == 1):
                x = layer.forward_fused(x, nxt)
                if capture is not None:  # keep per-layer capture indices aligned
                    capture.append(None)
                    capture.append(x)
                i += 2
                continue
            x = layer.forward(x, mode)
            if capture is not None:
                capture.append(x.float() if isinstance(x, PackedNHWC) else x)
            i += 1
        return x.float() if isinstance(x, PackedNHWC) else x

    def binary_layers(self):
        out = []
        for l in self.layers:
            if isinstance(l, (QConvolution, QFullyConnected)):
                out.append(l)
            elif hasattr(l, "binary_layers"):
                out.extend(l.binary_layers())
        return out

    def pack_for_inference(self):
        for l in self.binary_layers():
            l.pack()


def _lenet_stem(ls) -> bool:
    """Conv2d (tensor-core engine) -> Tanh -> MaxPool2d(2, 2, 0)."""
    return (len(ls) == 3 and isinstance(ls[0], Conv2d) and isinstance(ls[1], Tanh) and
            isinstance(ls[2], MaxPool2d) and (ls[2].k, ls[2].stride, ls[2].pad) == (2, 2, 0) and
            ls[0].engine == "tc" and ls[0].tc_supported())


_TANH_MONOTONE = None


def tanh_is_monotone() -> bool:
    """Exhaustive device check (once per process) that the f32 tanh is monotone, which
    makes maxpool(tanh(v)) == tanh(maxpool(v)) exact (the fused LeNet stem's ``pool_first``
    argument: one tanh per pooled output instead of four, stem 130 -> 112 us at batch 1024)."""
    global _TANH_MONOTONE
    if _TANH_MONOTONE is None:
        v = torch.zeros(1, dtype=torch.int64, device="cuda")
        _lib.call("bnn_probe_tanh_monotone", _lib.ptr(v), _lib.stream_ptr())
        _TANH_MONOTONE = int(v.item()) == 0
    return _TANH_MONOTONE


def _pool_first_ok() -> bool:
    """Pool before the tanh when the device's tanhf was probed monotone (exact then).  The probe
    synchronises, so inside a CUDA-graph capture only a cached answer is used."""
    if _TANH_MONOTONE is None and torch.cuda.is_current_stream_capturing():
        return False
    return tanh_is_monotone()


def _lenet_stem_forward(conv: "Conv2d", x: torch.Tensor, pool_first: bool = False, pack: bool = False,
                        f32_out: bool = True, flags: torch.Tensor | None = None):
    """maxpool2x2(tanh(conv(x) + b)) in one kernel (bnn_conv_tanh_maxpool2_f32_tc): the
    same per-element f32 ops as the three torch calls, the conv output never written.
    ``pack``: the kernel also writes the sign-packed NHWC words for a following binary conv
    (its QActivation + pack fused) and a ``PackedNHWC`` is returned; with ``f32_out`` False
    the f32 tensor is never written either."""
    x = x.contiguous()
    b, c, h, w = x.shape
    oh, ow = conv.output_hw(h, w)
    if pack and conv.cout % 64 == 0:
        shape = (b, conv.cout, oh // 2, ow // 2)
        y = torch.empty(shape, dtype=torch.float32, device=x.device) if f32_out else None
        words = torch.empty((b, oh // 2, ow // 2, conv.cout // 64), dtype=torch.uint64, device=x.device)
        st = _lib.call_status("bnn_conv_tanh_maxpool2_pack_f32_tc", _lib.ptr(x), b, c, h, w,
                              _lib.ptr(conv._dev("weight")), _lib.ptr(conv._dev("bias")), conv.cout,
                              *conv.geometry(), int(pool_first), _lib.ptr(y), _lib.ptr(words),
                              _lib.ptr(flags), _lib.stream_ptr())
        if st != _lib.EUNSUP:
            _lib.check(st, "bnn_conv_tanh_maxpool2_pack_f32_tc")
            return PackedNHWC(words, shape, y)
    y = torch.empty((b, conv.cout, oh // 2, ow // 2), dtype=torch.float32, device=x.device)
    st = _lib.call_status("bnn_conv_tanh_maxpool2_f32_tc", _lib.ptr(x), b, c, h, w,
                          _lib.ptr(conv._dev("weight")), _lib.ptr(conv._dev("bias")), conv.cout,
                          *conv.geometry(), int(pool_first), _lib.ptr(y), _lib.stream_ptr())
    if st == _lib.EUNSUP:
        return MaxPool2d(2).forward(torch.tanh(conv.forward(x)))
    _lib.check(st, "bnn_conv_tanh_maxpool2_f32_tc")
    return y


_SMS = []


def _sm_count() -> int:
    if not _SMS:
        _SMS.append(torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count)
    return _SMS[0]


def _binary_pool_fc(ls) -> bool:
    """QConvolution -> BatchNorm -> MaxPool2d(k, k, 0) -> Flatten -> QFullyConnected ->
    BatchNorm, 1-bit, the conv's filters a multiple of 64 (whole channel words)."""
    return (len(ls) == 6 and isinstance(ls[0], QConvolution) and isinstance(ls[1], BatchNorm) and
            isinstance(ls[2], MaxPool2d) and ls[2].pad == 0 and ls[2].stride == ls[2].k and
            isinstance(ls[3], Flatten) and isinstance(ls[4], QFullyConnected) and
            isinstance(ls[5], BatchNorm) and ls[0].bits == 1 and ls[4].bits == 1 and
            ls[0].filters % 64 == 0)


def _binary_pool_fc_forward(ls, x) -> torch.Tensor:
    """sign(maxpool(BN(conv))) == OR-pool of sign(BN(conv)): the conv epilogue writes only
    the packed sign words, bnn_maxpool_packed ORs the windows, and the FC reads the pooled
    NHWC words as its K-contiguous rows -- its weights permuted once from the reference's
    (c, h, w) flatten order (layers.py:459) to (h, w, c) (popcounts are permutation
    invariant, the outputs are unchanged)."""
    conv, bn1, pool, _, fc, bn2 = ls
    t = x.contiguous() if not isinstance(x, PackedNHWC) else x
    h = conv.forward_fused(t, bn1, pack_out=True, f32_out=False)
    b, c, hh, ww = h.shape
    oh, ow = (hh - pool.k) // pool.k + 1, (ww - pool.k) // pool.k + 1
    cw = h.words.shape[-1]
    # an even row pitch (16-byte aligned rows) lets the FC run its TMA-fed kind::mxf4 route
    # (LeNet: 49 words per image -> pitch 50, 19.3 -> 15.2 us); the pad word is never read
    rw = oh * ow * cw
    pitch = rw + (rw & 1)
    pooled = torch.empty((b, pitch), dtype=torch.uint64, device="cuda")
    _lib.call("bnn_maxpool_packed_ld", _lib.ptr(h.words), b, hh, ww, cw, pool.k, pool.k,
              _lib.ptr(pooled), pitch, _lib.stream_ptr())
    if fc.in_features != c * oh * ow:
        raise ValueError(f"expected {fc.in_features} features, got {c * oh * ow}")
    return fc.forward_packed_hwc(pooled[:, :rw], (c, oh, ow), bn2)


class BinaryBasicBlock:
    """out = BN2(QConv3x3(sign(BN1(QConv3x3(sign(x), stride))))) + shortcut(x)."""

    def __init__(self, cin, cout, stride, rng):
        self.conv1 = QConvolution(cin, cout, (3, 3), (stride, stride), (1, 1), rng=rng, domain="dot")
        self.bn1 = BatchNorm(cout, rng)
        self.conv2 = QConvolution(cout, cout, (3, 3), (1, 1), (1, 1), rng=rng, domain="dot")
        self.bn2 = BatchNorm(cout, rng)
        self.down = None
        if stride != 1 or cin != cout:
            self.down = QConvolution(cin, cout, (1, 1), (stride, stride), (0, 0), rng=rng,
                                     domain="dot")
            self.bnd = BatchNorm(cout, rng)

    def binary_layers(self):
        return [self.conv1, self.conv2] + ([self.down] if self.down else [])

    fused = True  # infer_packed: BN and the shortcut add run in the conv epilogues
    # infer_packed: activations stay sign-packed between the binary convs -- conv1
    # writes only the packed sign of BN1's output (its f32 has no other consumer),
    # conv2 writes the f32 block output (next shortcut) and its packed sign (next
    # block's convs), so no standalone pack pass runs inside the network
    packed_io = True
    emit_packed = True  # False for the last block (a float layer consumes it)
    # False when no consumer reads the f32 block output: the next block has a
    # downsample shortcut (it reads the packed words only) -- conv2's epilogue then
    # computes BN + shortcut for the sign and writes the packed words alone
    needs_f32_out = True
    split_shortcut = True  # conv2 epilogue without the add + one add/sign-pack pass
    # (for the convs the shifted-window kernel runs -- C, F <= 128 -- and the pre-expanded conv
    # engine -- C % 256 == 0 -- the shortcut add stays in conv2's epilogue, whose residual reads
    # are coalesced there)

    def _fused_shortcut(self, h) -> bool:
        c, f = self.conv2.in_channels, self.conv2.filters
        if not self.split_shortcut or (c in (64, 128) and f in (64, 128)):
            return True
        if c >= 256 and c % 256 == 0 and f % 64 == 0 and f <= 1024 and \
                self.conv2.algo in ("auto", "xp", _lib.ALGO_AUTO, _lib.ALGO_UMMA_XP):
            # the pre-expanded conv engine (bnn_bconv2d_ws, rows = pixels): for every filter a
            # warp reads / writes 32 consecutive pixels, so the shortcut add and the sign-pack
            # stay in conv2's epilogue (no f32 round trip, no add / sign-pack pass)
            return True
        if c == 256 and f == 256:
            # the shifted-window kernel takes C = 256 when a CTA owns >= 5 tiles of 128 padded
            # positions (launch_wconv, bnn_wconv.cu); below that the general engine runs and
            # the split add / sign-pack pass is faster
            b, _, hh, ww = h.shape
            tiles = -(-(b * (hh + 2) * (ww + 2)) // 128)
            ranges = max(1, _sm_count() // 2)
            return tiles >= 5 * min(ranges, tiles)
        return False

    def forward(self, x, mode=INFER_FLOAT):
        if mode == INFER_PACKED and self.fused and self.packed_io:
            if not isinstance(x, PackedNHWC):
                x = PackedNHWC.from_f32(x, self.conv1._flags())
            h = self.conv1.forward_fused(x, self.bn1, pack_out=True, f32_out=False)
            sc = x.float() if self.down is None else self.down.forward_fused(x, self.bnd)
            fused_sc = self._fused_shortcut(h)
            if self.emit_packed and not self.needs_f32_out and fused_sc:
                return self.conv2.forward_fused(h, self.bn2, residual=sc, pack_out=True,
                                                f32_out=False)
            if not fused_sc:
                # the conv epilogue without the shortcut is faster on the general engine's
                # shapes (profiles/r01/resnet_layer_epilogues.txt: f32 vs pack+f32+res), so
                # the add and the sign-pack run as one streaming pass (bit-identical)
                y = self.conv2.forward_fused(h, self.bn2)
                b, f, oh, ow = y.shape
                words = torch.empty((b, oh, ow, (f + 63) // 64), dtype=torch.uint64,
                                    device=y.device)
                _lib.call("bnn_add_pack_nchw_f32", _lib.ptr(y), _lib.ptr(sc.contiguous()), b, f,
                          oh, ow, _lib.ptr(y), _lib.ptr(words), _lib.ptr(self.conv2._flags()),
                          _lib.stream_ptr())
                return PackedNHWC(words, y.shape, y) if self.emit_packed else y
            return self.conv2.forward_fused(h, self.bn2, residual=sc, pack_out=self.emit_packed)
        if isinstance(x, PackedNHWC):
            x = x.float()
        if mode == INFER_PACKED and self.fused:
            h = self.conv1.forward_fused(x, self.bn1)
            sc = x if self.down is None else self.down.forward_fused(x, self.bnd)
            return self.conv2.forward_fused(h, self.bn2, residual=sc)
        h = self.bn1.forward(self.conv1.forward(x, mode))
        h = self.bn2.forward(self.conv2.forward(h, mode))
        sc = x if self.down is None else self.bnd.forward(self.down.forward(x, mode))
        return h + sc


def lenet_c3(seed: int = 0) -> Sequential:
    """BASELINE configs[2] topology, random init."""
    rng = np.random.default_rng(seed)
    return Sequential([
        Conv2d(1, 64, 5, pad=2, rng=rng), Tanh(), MaxPool2d(2),
        QConvolution(64, 64, (5, 5), (1, 1), (2, 2), rng=rng),  # sign of the input fused
        BatchNorm(64, rng), MaxPool2d(2), Flatten(),
        QFullyConnected(64 * 7 * 7, 1000, rng=rng), BatchNorm(1000, rng),
        Dense(1000, 10, rng=rng),
    ])


def resnet18_c4(seed: int = 0, num_classes: int = 1000) -> Sequential:
    """BASELINE configs[3]: binary ResNet-18 (stem and classifier full precision)."""
    rng = np.random.default_rng(seed)
    layers = [Conv2d(3, 64, 7, stride=2, pad=3, bias=False, rng=rng), StemPost(64, rng, 3, 2, 1)]
    cin = 64
    for cout, stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
        layers.append(BinaryBasicBlock(cin, cout, stride, rng))
        layers.append(BinaryBasicBlock(cout, cout, 1, rng))
        cin = cout
    layers[-1].emit_packed = False  # the average pool reads the f32 output
    blocks = [l for l in layers if isinstance(l, BinaryBasicBlock)]
    for blk, nxt in zip(blocks[:-1], blocks[1:]):
        blk.needs_f32_out = nxt.down is None  # identity shortcuts read the f32 output
    layers += [GlobalAvgPool(), Dense(512, num_classes, rng=rng)]
    return Sequential(layers)


def binary_ops_per_image(net: Sequential, chw) -> int:
    """2*M*N*K summed over the binary layers for one image."""
    c, h, w = chw
    total = 0

    def conv(layer, c, h, w):
        oh, ow = layer.output_hw(h, w)
        return layer.filters, oh, ow, 2 * layer.filters * oh * ow * layer.k_reduce

    for layer in net.layers:
        if isinstance(layer, Conv2d):
            h, w = layer.output_hw(h, w)
            c = layer.cout
        elif isinstance(layer, (MaxPool2d, StemPost)):
            pl = layer if isinstance(layer, MaxPool2d) else layer.pool
            h = (h + 2 * pl.pad - pl.k) // pl.stride + 1
            w = (w + 2 * pl.pad - pl.k) // pl.stride + 1
        elif isinstance(layer, QConvolution):
            c, h, w, ops = conv(layer, c, h, w)
            total += ops
        elif isinstance(layer, BinaryBasicBlock):
            c1, h1, w1, o1 = conv(layer.conv1, c, h, w)
            _, _, _, o2 = conv(layer.conv2, c1, h1, w1)
            total += o1 + o2
            if layer.down is not None:
                total += conv(layer.down, c, h, w)[3]
            c, h, w = c1, h1, w1
        elif isinstance(layer, (Flatten, GlobalAvgPool)):
            c, h, w = (c * h * w if isinstance(layer, Flatten) else c), 1, 1
        elif isinstance(layer, QFullyConnected):
            total += 2 * layer.units * layer.in_features
            c = layer.units
    return total
