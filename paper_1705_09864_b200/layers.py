"""Quantized layers with a bit-packed xnor-popcount inference path on the B200.

Drop-in for the hot-path layers of the reference ``bitnn.layers``
(``/root/reference/pkg/src/bitnn/layers.py``): ``QActivation`` (:392-419),
``QConv2d`` (:159-263) and ``QDense`` (:320-389), with the same constructor
arguments, modes (``train_float`` / ``infer_float`` / ``infer_packed``,
:31-34), ``ModeError`` rules and popcount-domain outputs.  ``infer_packed``
runs the sm_100a kernels (fused sign+pack, implicit-im2col conv, xnor GEMM);
``infer_float`` keeps the reference's float semantics on the GPU (used as the
in-framework equivalence check, as in the reference).  Training/backward is
out of scope (OUT OF SCOPE) and raises ModeError.

BMXNet names: ``QConvolution`` / ``QFullyConnected`` take ``act_bit`` /
``weight_bit`` and fuse the preceding sign activation
into the pack kernel; ``QConvolution`` accepts spatial padding with the
reference-composition semantics "zero-pad, then binarize" (pad = +1, G2).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib, qmath
from .bitpack import (BitMatrix, pack_matrix_a, pack_nchw, pack_planes_device, pack_rows_device,
                      raise_on_flags, to_device_f32, to_device_words, words_per_bits)
from .gemm import bitplane_gemm, xnor_rows_gemm

TRAIN_FLOAT = "train_float"
INFER_FLOAT = "infer_float"
INFER_PACKED = "infer_packed"
MODES = (TRAIN_FLOAT, INFER_FLOAT, INFER_PACKED)
BN_EPS = 1e-5  # layers.py:36


class ModeError(RuntimeError):
    """A layer was asked to run in a mode its current state cannot serve (layers.py:40-41)."""


def _check_mode(mode):
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}; choose from {MODES}")
    if mode == TRAIN_FLOAT:
        raise ModeError("training is out of scope for the B200 inference path")


def _uniform_init(rng, shape, fan_in, fan_out):
    """layers._uniform_init (layers.py:49-51), NumPy RNG for seed parity."""
    bound = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-bound, bound, size=shape).astype(np.float32)


def _ret(t: torch.Tensor, was_np: bool):
    return t.cpu().numpy() if was_np else t


def _float_matmul(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return a @ b
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _float_conv(x, w, stride):
    """im2col (unfold, rows (c, i, j) like tensor.im2col) + f32 matmul, TF32 off.

    Exact for +-1 operands (integer sums < 2^24); cuDNN's Winograd/FFT
    algorithms would round.  This is the reference float path (layers.py:240-242).
    """
    b = x.shape[0]
    f, c, kh, kw = w.shape
    oh = (x.shape[2] - kh) // stride[0] + 1
    ow = (x.shape[3] - kw) // stride[1] + 1
    cols = F.unfold(x, (kh, kw), stride=stride)  # [B, C*kh*kw, oh*ow]
    out = _float_matmul(w.reshape(f, -1), cols)  # [B, F, oh*ow]
    return out.reshape(b, f, oh, ow)


class QActivation:
    """Quantize activations to ``bits`` (sign at 1 bit) -- layers.py:392-419."""

    kind = "qactivation"

    def __init__(self, bits=1):
        self.bits = int(bits)
        qmath.QuantSpec(self.bits)

    def spec(self):
        return {"kind": self.kind, "bits": self.bits}

    def forward(self, x, mode=INFER_FLOAT):
        _check_mode(mode)
        t, was_np = to_device_f32(x)
        if self.bits == 1:
            # binarize(clip(x)) == binarize(x); one fused sign kernel
            out = torch.empty_like(t)
            flags = torch.zeros(1, dtype=torch.int32, device=t.device)
            _lib.call("bnn_binarize_f32", _lib.ptr(t), t.numel(), _lib.ptr(out), _lib.ptr(flags),
                      _lib.stream_ptr())
            raise_on_flags(flags, "quantize_signed requires finite inputs")
            return _ret(out, was_np)
        return _ret(qmath.quantize_signed(t, self.bits), was_np)


class _QLayer:
    """Shared packed-weight state of the quantized conv / dense layers.

    ``sync_checks`` (default True) reads the pack kernel's flag word after
    every packed forward to raise the reference's ValueError on non-finite /
    non-sign input; network runners and CUDA-graph capture set it False and
    read ``flags`` once at the end instead (no host sync per layer).
    """

    sync_checks = True
    flags = None

    def _flags(self):
        if self.flags is None:
            self.flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        return self.flags

    def _finish(self, flags, msg="binarize requires finite inputs"):
        if self.sync_checks:
            raise_on_flags(flags, msg)

    def _set_packed(self, bm: BitMatrix):
        self.packed = bm
        self._dev_words = None

    def pack(self):
        """Freeze sign(weight) into packed words for ``infer_packed`` (layers.py:215-223)."""
        if self.bits != 1:
            raise ModeError("packed inference supports 1-bit weights only")
        if self.weight is None:
            raise ModeError("no float weights to pack")
        w = torch.from_numpy(np.ascontiguousarray(self._flat_weight_np())).cuda()
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        words = pack_rows_device(w, 0, strict=False, flags=flags)
        raise_on_flags(flags)
        self._set_packed(BitMatrix(words=words, vectors=w.shape[0], n_bits=w.shape[1],
                                   layout="a", pad_fill=0))
        return self.packed

    def load_packed(self, words, n_bits=None):
        """Install layout-'a' words from storage (``.bmx`` payload, modelio.py:221-237)."""
        k = self.k_reduce if n_bits is None else n_bits
        w = to_device_words(words)
        self._set_packed(BitMatrix(words=w, vectors=w.shape[0], n_bits=k, layout="a",
                                   pad_fill=0))

    def _require_packed(self):
        if self.bits != 1:
            raise ModeError("packed inference supports 1-bit weights only")
        if self.packed is None:
            raise ModeError("layer has no packed weights; pack() or load a converted model")


class PackedNHWC:
    """A sign-binarised activation kept packed between binary layers.

    ``words``: u64 [B, H, W, ceil(C/64)] -- channel c at bit c % 64 of word
    c // 64, bit 1 = (x >= 0) (binarize, bitpack.py:30-42), channel tail 0: the
    layout ``pack_nchw`` writes and ``bnn_bconv2d`` reads.  ``f32`` is the same
    activation before the sign in NCHW f32 when a consumer needs it (a residual
    shortcut, a float layer), else None.  The packed words are written by the
    producing conv's epilogue, so no standalone pack pass runs.
    """

    __slots__ = ("words", "shape", "f32")

    def __init__(self, words: torch.Tensor, shape, f32: torch.Tensor | None = None):
        self.words, self.shape, self.f32 = words, tuple(int(v) for v in shape), f32

    @classmethod
    def from_f32(cls, x: torch.Tensor, flags: torch.Tensor | None = None) -> "PackedNHWC":
        x = x.contiguous()
        return cls(pack_nchw(x, strict=False, flags=flags), x.shape, x)

    def float(self) -> torch.Tensor:
        if self.f32 is None:
            raise ValueError("this packed activation kept no f32 copy")
        return self.f32


def make_epilogue(domain: int, bn=None, residual: torch.Tensor | None = None,
                  scale: torch.Tensor | None = None, shift: torch.Tensor | None = None,
                  pack_out: torch.Tensor | None = None, pack_flags: torch.Tensor | None = None):
    """ctypes ``bnn_epilogue`` for the fused GEMM / conv epilogue.

    ``bn`` is any object with ``device_params() -> (mean, inv_std, gamma, beta)``
    CUDA f32 tensors (e.g. ``nets.BatchNorm``); the kernel applies it in the
    reference's op order (layers.py:598-602), bit-identical to an unfused BN.
    """
    e = _lib.Epilogue()
    e.domain = domain
    e.scale, e.shift = _lib.ptr(scale), _lib.ptr(shift)
    keep = [scale, shift, residual]
    if bn is not None:
        mean, inv, gamma, beta = bn.device_params()
        e.bn_mean, e.bn_inv_std, e.bn_gamma, e.bn_beta = (_lib.ptr(t) for t in (mean, inv, gamma, beta))
        keep += [mean, inv, gamma, beta]
    if residual is not None:
        e.residual = _lib.ptr(residual)
    if pack_out is not None:  # sign-pack of the final value, [cols, pack_ld] u64
        e.pack_out, e.pack_ld = _lib.ptr(pack_out), pack_out.shape[-1]
        e.pack_flags = _lib.ptr(pack_flags)
        keep += [pack_out, pack_flags]
    e._keep = keep  # keep tensors alive with the struct
    return e


class QConv2d(_QLayer):
    """Binary convolution -- layers.py:159-263 (popcount-domain outputs).

    ``infer_packed`` requires +-1 inputs (the reference validates them in
    pack_matrix_b, bitpack.py:69-75) and, like the reference, rejects padding.
    """

    kind = "qconv"
    _allow_pad = False
    _fuse_sign = False  # the reference QConv2d consumes QActivation's output as-is

    def __init__(self, in_channels, filters, kernel, stride=(1, 1), pad=(0, 0), bits=1,
                 rng=None):
        self.in_channels = in_channels
        self.filters = filters
        self.kernel = tuple(kernel)
        self.stride = tuple(stride)
        self.pad = tuple(pad)
        if self.pad != (0, 0) and not self._allow_pad:
            raise ValueError("quantized convolution does not support padding")
        self.bits = int(bits)
        qmath.QuantSpec(self.bits)
        kh, kw = self.kernel
        self.k_reduce = in_channels * kh * kw
        if rng is not None:
            self.weight = _uniform_init(rng, (filters, in_channels, kh, kw), self.k_reduce,
                                        filters * kh * kw)
        else:
            self.weight = None
        self.packed = None
        self._dev_words = None
        self.domain = _lib.POPCOUNT
        self.algo = "auto"

    def spec(self):
        return {"kind": self.kind, "in_channels": self.in_channels, "filters": self.filters,
                "kernel": list(self.kernel), "stride": list(self.stride), "pad": list(self.pad),
                "bits": self.bits}

    def _flat_weight_np(self):
        return np.asarray(self.weight, np.float32).reshape(self.filters, self.k_reduce)

    def device_weights(self) -> torch.Tensor:
        """Tap-major re-layout of the packed words (load-time, cached)."""
        self._require_packed()
        if self._dev_words is None:
            kh, kw = self.kernel
            cw = words_per_bits(self.in_channels)
            out = torch.empty((self.filters, kh * kw * cw), dtype=torch.uint64, device="cuda")
            _lib.call("bnn_conv_weights_reorder", _lib.ptr(self.packed.words), self.filters,
                      self.in_channels, kh, kw, _lib.ptr(out), _lib.stream_ptr())
            self._dev_words = out
        return self._dev_words

    def output_hw(self, h, w):
        kh, kw = self.kernel
        oh = (h + 2 * self.pad[0] - kh) // self.stride[0] + 1
        ow = (w + 2 * self.pad[1] - kw) // self.stride[1] + 1
        if min(h, w) < 1 or oh < 1 or ow < 1 or h + 2 * self.pad[0] < kh or \
                w + 2 * self.pad[1] < kw:
            raise ValueError(f"kernel {kh}x{kw} does not fit input {h}x{w} with pad "
                             f"{self.pad[0]},{self.pad[1]}")
        return oh, ow

    def conv_workspace(self, b: int, h: int, w: int, algo: int):
        """Scratch of the pre-expanded conv engine (bnn_bconv2d_ws) for this geometry, or None
        when the engine does not take it (C % 256 != 0, ...) or another engine was asked for.
        One buffer per (device, stream), shared by all layers: calls on a stream are ordered."""
        if algo not in (_lib.ALGO_AUTO, _lib.ALGO_UMMA_XP):
            return None
        if algo == _lib.ALGO_AUTO and self.in_channels < 256:  # (mirrors bconv2d_impl in bnn_capi.cu)
            return None
        kh, kw = self.kernel
        need = int(_lib.load().bnn_bconv2d_ws_bytes(b, self.in_channels, h, w, self.filters, kh, kw,
                                                    self.stride[0], self.stride[1], self.pad[0],
                                                    self.pad[1]))
        if need <= 0:
            return None
        from .gemm import scratch
        return scratch(need, "cuda")

    def forward_packed_words(self, x_words: torch.Tensor, b: int, h: int, w: int,
                             out: torch.Tensor | None = None, scale=None, shift=None):
        """Conv on already-packed NHWC words -> f32 NCHW (no host sync)."""
        import ctypes
        kh, kw = self.kernel
        oh, ow = self.output_hw(h, w)
        if out is None:
            out = torch.empty((b, self.filters, oh, ow), dtype=torch.float32, device="cuda")
        wd = self.device_weights()
        algo = _lib.ALGOS[self.algo] if isinstance(self.algo, str) else self.algo
        ws = self.conv_workspace(b, h, w, algo)
        if ws is not None:
            e = make_epilogue(self.domain, scale=scale, shift=shift)
            _lib.call("bnn_bconv2d_ws", _lib.ptr(x_words), b, self.in_channels, h, w, _lib.ptr(wd),
                      self.filters, kh, kw, self.stride[0], self.stride[1], self.pad[0], self.pad[1],
                      _lib.ptr(out), ctypes.byref(e), algo, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
            return out
        _lib.call("bnn_bconv2d", _lib.ptr(x_words), b, self.in_channels, h, w, _lib.ptr(wd),
                  self.filters, kh, kw, self.stride[0], self.stride[1], self.pad[0], self.pad[1],
                  _lib.ptr(out), self.domain, _lib.ptr(scale), _lib.ptr(shift), algo,
                  _lib.stream_ptr())
        return out

    def _strict_input(self) -> bool:
        return True

    def forward_fused(self, x, bn=None, residual: torch.Tensor | None = None,
                      out: torch.Tensor | None = None, pack_out: bool = False,
                      f32_out: bool = True):
        """``infer_packed`` conv with BatchNorm (+ residual add) fused into the epilogue.

        ``x``: f32 NCHW (packed here, sign fused) or a ``PackedNHWC`` from a
        previous layer's epilogue (no pack pass).  ``pack_out``: also emit the
        sign-packed output for the next binary layer (the next QActivation and
        pack fused into this epilogue) and return a ``PackedNHWC`` whose ``f32``
        is the f32 output (None when ``f32_out`` is False).
        """
        import ctypes
        self._require_packed()
        flags = torch.zeros(1, dtype=torch.int32, device="cuda") if self.sync_checks \
            else self._flags()
        if isinstance(x, PackedNHWC):
            b, c, h, w = x.shape
            if c != self.in_channels:
                raise ValueError(f"expected {self.in_channels} channels, got {c}")
            xw = x.words
        else:
            t = x.contiguous()
            b, c, h, w = t.shape
            xw = pack_nchw(t, strict=self._strict_input(), flags=flags)
        kh, kw = self.kernel
        oh, ow = self.output_hw(h, w)
        if not (f32_out or pack_out):
            raise ValueError("nothing to compute: f32_out and pack_out are both False")
        if out is None and f32_out:
            out = torch.empty((b, self.filters, oh, ow), dtype=torch.float32, device="cuda")
        if not f32_out:
            out = None
        pw_out = torch.empty((b, oh, ow, words_per_bits(self.filters)), dtype=torch.uint64,
                             device="cuda") if pack_out else None
        if residual is not None:
            residual = residual.contiguous()
            if tuple(residual.shape) != (b, self.filters, oh, ow):
                raise ValueError("residual must match the conv output shape")
        e = make_epilogue(self.domain, bn, residual, pack_out=pw_out,
                          pack_flags=flags if pack_out else None)
        wd = self.device_weights()
        algo = _lib.ALGOS[self.algo] if isinstance(self.algo, str) else self.algo
        ws = self.conv_workspace(b, h, w, algo)
        if ws is not None:
            _lib.call("bnn_bconv2d_ws", _lib.ptr(xw), b, self.in_channels, h, w, _lib.ptr(wd),
                      self.filters, kh, kw, self.stride[0], self.stride[1], self.pad[0], self.pad[1],
                      _lib.ptr(out), ctypes.byref(e), algo, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        else:
            _lib.call("bnn_bconv2d_ex", _lib.ptr(xw), b, self.in_channels, h, w, _lib.ptr(wd),
                      self.filters, kh, kw, self.stride[0], self.stride[1], self.pad[0], self.pad[1],
                      _lib.ptr(out), ctypes.byref(e), algo, _lib.stream_ptr())
        self._finish(flags)
        if pack_out:
            return PackedNHWC(pw_out, (b, self.filters, oh, ow), out)
        return out

    def forward(self, x, mode=INFER_FLOAT):
        _check_mode(mode)
        t, was_np = to_device_f32(x)
        if t.dim() != 4:
            raise ValueError(f"expected [B, C, H, W] input, got ndim={t.dim()}")
        b, c, h, w = t.shape
        self.output_hw(h, w)
        if mode == INFER_PACKED:
            self._require_packed()
            flags = torch.zeros(1, dtype=torch.int32, device="cuda") if self.sync_checks \
                else self._flags()
            xw = pack_nchw(t, strict=self._strict_input(), flags=flags)
            y = self.forward_packed_words(xw, b, h, w)
            self._finish(flags)
            return _ret(y, was_np)
        if self.weight is None:
            raise ModeError("layer holds packed weights only; float modes unavailable")
        wq = qmath.quantize_signed(torch.from_numpy(np.asarray(self.weight, np.float32)).cuda(),
                                   self.bits)
        if self.pad != (0, 0):
            # G2: the reference composition zero-pads, then binarizes
            t = F.pad(t, (self.pad[1], self.pad[1], self.pad[0], self.pad[0]))
        if self._fuse_sign:
            t = qmath.quantize_signed(t, self.act_bit)
        dot = _float_conv(t, wq, self.stride)
        if self.bits == 1 and self.domain == _lib.POPCOUNT:
            return _ret((dot + self.k_reduce) * 0.5, was_np)
        return _ret(dot, was_np)


class QDense(_QLayer):
    """Binary fully connected layer -- layers.py:320-389 (popcount domain)."""

    kind = "qfc"
    _fuse_sign = False

    def __init__(self, in_features, units, bits=1, rng=None):
        self.in_features = in_features
        self.units = units
        self.bits = int(bits)
        qmath.QuantSpec(self.bits)
        self.k_reduce = in_features
        if rng is not None:
            self.weight = _uniform_init(rng, (units, in_features), in_features, units)
        else:
            self.weight = None
        self.packed = None
        self._dev_words = None
        self.domain = _lib.POPCOUNT
        self.algo = "auto"

    def spec(self):
        return {"kind": self.kind, "in_features": self.in_features, "units": self.units,
                "bits": self.bits}

    def _flat_weight_np(self):
        return np.asarray(self.weight, np.float32)

    def _strict_input(self) -> bool:
        return True

    def forward_fused(self, x: torch.Tensor, bn=None, out: torch.Tensor | None = None):
        """``infer_packed`` dense layer with BatchNorm fused into the epilogue ([B, units])."""
        import ctypes
        self._require_packed()
        t = x.contiguous()
        flags = torch.zeros(1, dtype=torch.int32, device="cuda") if self.sync_checks \
            else self._flags()
        xw = pack_rows_device(t, 0, strict=self._strict_input(), flags=flags)
        if out is None:
            out = torch.empty((t.shape[0], self.units), dtype=torch.float32, device="cuda")
        e = make_epilogue(self.domain, bn)
        algo = _lib.ALGOS[self.algo] if isinstance(self.algo, str) else self.algo
        a = self.packed.words
        _lib.call("bnn_xnor_gemm_ex", _lib.ptr(a), a.stride(0), _lib.ptr(xw), xw.stride(0),
                  self.units, t.shape[0], self.in_features, 0, 0, _lib.ptr(out), 1, out.stride(0),
                  ctypes.byref(e), algo, _lib.stream_ptr())
        self._finish(flags)
        return out

    def device_words_hwc(self, chw) -> torch.Tensor:
        """Packed weights with K re-ordered from the reference's NCHW flatten order
        (c, h, w) (layers.py:459) to (h, w, c): the order of pooled packed NHWC words.
        Load-time permutation, cached; popcounts are permutation invariant."""
        self._require_packed()
        cache = self.__dict__.setdefault("_hwc_cache", {})
        key = tuple(chw)
        if key not in cache:
            c, h, w = key
            if c * h * w != self.in_features or c % 64:
                raise ValueError("(h, w, c) re-order needs whole 64-channel words")
            words = self.packed.words.cpu().numpy().view(np.uint8)
            bits = np.unpackbits(words, axis=1, bitorder="little")[:, :self.in_features]
            bits = bits.reshape(self.units, c, h, w).transpose(0, 2, 3, 1).reshape(self.units, -1)
            packed = np.packbits(bits, axis=1, bitorder="little").view(np.uint64)
            rw = packed.shape[1]
            padded = np.zeros((self.units, rw + (rw & 1)), np.uint64)  # even pitch: 16-byte rows
            padded[:, :rw] = packed
            cache[key] = torch.from_numpy(padded).cuda()[:, :rw]
        return cache[key]

    def forward_packed_hwc(self, x_words: torch.Tensor, chw, bn=None) -> torch.Tensor:
        """[B, in_features / 64] packed activation rows in (h, w, c) order (pooled packed
        NHWC words) -> f32 [B, units] with the fused BatchNorm epilogue."""
        import ctypes
        a = self.device_words_hwc(chw)
        n = x_words.shape[0]
        out = torch.empty((n, self.units), dtype=torch.float32, device="cuda")
        e = make_epilogue(self.domain, bn)
        algo = _lib.ALGOS[self.algo] if isinstance(self.algo, str) else self.algo
        _lib.call("bnn_xnor_gemm_ex", _lib.ptr(a), a.stride(0), _lib.ptr(x_words),
                  x_words.stride(0), self.units, n, self.in_features, 0, 0, _lib.ptr(out), 1,
                  out.stride(0), ctypes.byref(e), algo, _lib.stream_ptr())
        return out

    def forward_packed_rows(self, x_words: torch.Tensor, out=None, scale=None, shift=None):
        """[B, W] packed activations (tail 0) -> f32 [B, units] (no host sync)."""
        self._require_packed()
        return xnor_rows_gemm(self.packed.words, x_words, self.in_features, a_pad=0, b_pad=0,
                              domain=self.domain, out=out, transpose_out=True, scale=scale,
                              shift=shift, algo=self.algo)

    def forward(self, x, mode=INFER_FLOAT):
        _check_mode(mode)
        t, was_np = to_device_f32(x)
        if mode == INFER_PACKED:
            self._require_packed()
            if t.dim() != 2 or t.shape[1] != self.in_features:
                raise ValueError(f"expected [B, {self.in_features}] input")
            flags = torch.zeros(1, dtype=torch.int32, device="cuda") if self.sync_checks \
                else self._flags()
            xw = pack_rows_device(t, 0, strict=self._strict_input(), flags=flags)
            y = self.forward_packed_rows(xw)
            self._finish(flags)
            return _ret(y, was_np)
        if self.weight is None:
            raise ModeError("layer holds packed weights only; float modes unavailable")
        wq = qmath.quantize_signed(torch.from_numpy(np.asarray(self.weight, np.float32)).cuda(),
                                   self.bits)
        if self._fuse_sign:
            t = qmath.quantize_signed(t, self.act_bit)
        dot = _float_matmul(t, wq.T)
        if self.bits == 1 and self.domain == _lib.DOT:
            return _ret(dot, was_np)
        y = (dot + self.in_features) * 0.5 if self.bits == 1 else dot
        return _ret(y, was_np)


# ----------------------------------------------------------------- BMXNet names
class QConvolution(QConv2d):
    """BMXNet ``QConvolution`` (act_bit / weight_bit), sign of the input fused.

    Accepts raw float input: the sign activation (QActivation(act_bit=1)) is
    folded into the pack kernel.  Spatial padding is allowed and means
    "zero-pad then binarize" (pad positions are +1).
    """

    kind = "qconvolution"
    _allow_pad = True
    _fuse_sign = True

    def __init__(self, in_channels, num_filter, kernel, stride=(1, 1), pad=(0, 0), act_bit=1,
                 weight_bit=1, rng=None, domain="popcount"):
        if int(act_bit) != int(weight_bit):
            raise ValueError("act_bit != weight_bit has no reference packed path (G4)")
        super().__init__(in_channels, num_filter, kernel, stride, pad, bits=weight_bit, rng=rng)
        self.act_bit = int(act_bit)
        self.weight_bit = int(weight_bit)
        self.domain = _lib.DOT if domain == "dot" else _lib.POPCOUNT
        self.planes = None

    def _strict_input(self) -> bool:
        return False

    # ---- act_bit = weight_bit = 2: bit planes over the same engine (north star; the reference
    # has a float path only for bits > 1, layers.py:237-244 -- this is its packed counterpart:
    # zero-pad, quantize_signed (qmath.py), im2col (tensor.py:60-78), sum_k v_w v_x)
    def pack(self):
        if self.bits == 1:
            return super().pack()
        if self.bits != 2:
            raise ModeError("packed multi-bit inference supports act_bit = weight_bit = 2")
        if self.weight is None:
            raise ModeError("no float weights to pack")
        w = torch.from_numpy(np.ascontiguousarray(self._flat_weight_np())).cuda()
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.planes = pack_planes_device(w, self.bits, "signed", flags)
        raise_on_flags(flags, "quantize_signed requires finite inputs")
        self.packed = self.planes  # marks the layer as packed
        return self.planes

    def _require_packed(self):
        if self.bits == 1:
            return super()._require_packed()
        if self.packed is None:
            raise ModeError("layer has no packed weights; pack() or load a converted model")

    def forward(self, x, mode=INFER_FLOAT):
        if self.bits == 1 or mode != INFER_PACKED:
            return super().forward(x, mode)
        _check_mode(mode)
        self._require_packed()
        t, was_np = to_device_f32(x)
        if t.dim() != 4 or t.shape[1] != self.in_channels:
            raise ValueError(f"expected [B, {self.in_channels}, H, W] input")
        b, _, h, w = t.shape
        oh, ow = self.output_hw(h, w)
        if self.pad != (0, 0):  # G2 generalised: zero-pad, then quantize (0 -> its grid value)
            t = F.pad(t, (self.pad[1], self.pad[1], self.pad[0], self.pad[0]))
        # im2col rows [B * OH * OW, C * kh * kw] in the reference's (c, ky, kx) order
        cols = F.unfold(t, self.kernel, stride=self.stride)
        rows = cols.transpose(1, 2).reshape(b * oh * ow, self.k_reduce).contiguous()
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        xp = pack_planes_device(rows, self.bits, "signed", flags)
        y = bitplane_gemm(self.planes, xp, self.k_reduce, a_grid="signed", b_grid="signed",
                          transpose_out=True)  # [B * OH * OW, F]
        raise_on_flags(flags, "quantize_signed requires finite inputs")
        y = y.view(b, oh, ow, self.filters).permute(0, 3, 1, 2).contiguous()
        return _ret(y, was_np)


class QFullyConnected(QDense):
    """BMXNet ``QFullyConnected`` (act_bit / weight_bit), sign of the input fused."""

    kind = "qfullyconnected"
    _fuse_sign = True

    def __init__(self, in_features, num_hidden, act_bit=1, weight_bit=1, rng=None,
                 domain="popcount", act_grid="signed", weight_grid="signed"):
        if int(act_bit) != int(weight_bit):
            raise ValueError("act_bit != weight_bit has no reference packed path (G4)")
        if int(weight_bit) not in (1, 2):
            raise ValueError("packed multi-bit path supports act_bit = weight_bit in {1, 2}")
        super().__init__(in_features, num_hidden, bits=weight_bit, rng=rng)
        self.act_bit = int(act_bit)
        self.weight_bit = int(weight_bit)
        self.domain = _lib.DOT if domain == "dot" else _lib.POPCOUNT
        # multi-bit grids: "signed" = quantize_signed (the reference layers'),
        # "unsigned" = quantize on [0, 1] (config 5's U[0,1] operands)
        self.act_grid, self.weight_grid = act_grid, weight_grid

    def pack(self):
        if self.bits == 1:
            return super().pack()
        if self.weight is None:
            raise ModeError("no float weights to pack")
        w = torch.from_numpy(np.ascontiguousarray(self._flat_weight_np())).cuda()
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.planes = pack_planes_device(w, self.bits, self.weight_grid, flags)
        raise_on_flags(flags, "quantize_signed requires finite inputs")
        self.packed = self.planes  # marks the layer as packed
        return self.planes

    def _require_packed(self):
        if self.packed is None:
            raise ModeError("layer has no packed weights; pack() or load a converted model")

    def forward(self, x, mode=INFER_FLOAT):
        if self.bits == 1 or mode != INFER_PACKED:
            if self.bits != 1 and mode == INFER_FLOAT and self.act_grid == "unsigned":
                _check_mode(mode)
                t, was_np = to_device_f32(x)
                xq = qmath.quantize(t, self.act_bit)
                wq = qmath.quantize(torch.from_numpy(np.asarray(self.weight, np.float32)).cuda(),
                                    self.weight_bit) if self.weight_grid == "unsigned" else \
                    qmath.quantize_signed(torch.from_numpy(np.asarray(self.weight, np.float32)).cuda(),
                                          self.weight_bit)
                return _ret(_float_matmul(xq, wq.T), was_np)
            return super().forward(x, mode)
        _check_mode(mode)
        self._require_packed()
        t, was_np = to_device_f32(x)
        if t.dim() != 2 or t.shape[1] != self.in_features:
            raise ValueError(f"expected [B, {self.in_features}] input")
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        xp = pack_planes_device(t, self.bits, self.act_grid, flags)
        y = bitplane_gemm(self.planes, xp, self.in_features, a_grid=self.weight_grid,
                          b_grid=self.act_grid, transpose_out=True)
        raise_on_flags(flags, "quantize_signed requires finite inputs")
        return _ret(y, was_np)

    def _strict_input(self) -> bool:
        return False
