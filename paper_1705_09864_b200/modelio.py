"""``.bmx`` model container -> B200 network.

Reader for the reference's BMX1 format (``pkg/docs/format.md``; writer
modelio.py:109-135, reader :161-247): magic "BMX1", u32 version 1, u32-length
arch JSON, u32 tensor count, then per tensor (u16 name length, name
"layer<i>.<field>", u8 dtype 0 = f32 / 1 = packed 1-bit, u8 ndim, u64 dims,
payload).  Packed payloads are layout-'a' u64 words, LSB-first, 0-filled
tails -- installed on the GPU verbatim (``load_packed``) after the padding
audit (bitpack.py:197-215); any device re-layout happens at load time.  The
same validation rules and ``ModelFormatError`` messages as the reference.
"""

from __future__ import annotations

import json
import struct

import numpy as np
import torch

from . import nets
from .bitpack import words_per_bits
from .layers import (INFER_FLOAT, INFER_PACKED, QActivation, QConv2d, QDense, _check_mode)

MAGIC = b"BMX1"
VERSION = 1
DTYPE_F32 = 0
DTYPE_PACKED1 = 1


class ModelFormatError(Exception):
    """The bytes on disk do not form a valid model file (modelio.py:45-46)."""


class _Conv2d(nets.Conv2d):
    def __init__(self, spec):
        kh, kw = spec["kernel"]
        super().__init__(spec["in_channels"], spec["filters"], kh, bias=spec["bias"])
        self.weight = np.zeros((spec["filters"], spec["in_channels"], kh, kw), np.float32)
        self.stride, self.pad = tuple(spec["stride"]), tuple(spec["pad"])


class _Dense(nets.Dense):
    def __init__(self, spec):
        super().__init__(spec["in_features"], spec["units"], bias=spec["bias"])


class _MaxPool(nets.MaxPool2d):
    def __init__(self, spec):
        if list(spec["kernel"]) != list(spec["stride"]):
            raise ModelFormatError("pooling windows must tile the input (kernel == stride)")
        super().__init__(tuple(spec["kernel"]), tuple(spec["stride"]))


class _BatchNorm(nets.BatchNorm):
    def __init__(self, spec):
        super().__init__(spec["channels"])
        self.eps = spec.get("eps", 1e-5)

    def finalize(self):
        self.inv_std = (1.0 / np.sqrt(self.var + np.float32(self.eps))).astype(np.float32)
        self.__dict__.pop("_dev_cache", None)


class SoftmaxOutput:
    """layers.SoftmaxOutput.forward (layers.py:631-637) in float32."""

    def forward(self, logits, mode=INFER_FLOAT):
        shifted = logits - logits.max(dim=1, keepdim=True).values
        log_probs = shifted - torch.log(torch.exp(shifted).sum(dim=1, keepdim=True))
        return torch.exp(log_probs)


def _layer_from_spec(spec):
    kind = spec.get("kind")
    if kind == "conv":
        return _Conv2d(spec)
    if kind == "qconv":
        return QConv2d(spec["in_channels"], spec["filters"], spec["kernel"], spec["stride"],
                       spec["pad"], spec["bits"])
    if kind == "fc":
        return _Dense(spec)
    if kind == "qfc":
        return QDense(spec["in_features"], spec["units"], spec["bits"])
    if kind == "qactivation":
        return QActivation(spec["bits"])
    if kind == "tanh":
        return nets.Tanh()
    if kind == "flatten":
        return nets.Flatten()
    if kind == "maxpool":
        return _MaxPool(spec)
    if kind == "batchnorm":
        return _BatchNorm(spec)
    raise ModelFormatError(f"unknown layer kind {kind!r}")


def _expected_fields(layer):
    """field -> (allows_packed, float shape) (modelio.py:64-81)."""
    if isinstance(layer, _Conv2d):
        f = {"weight": (False, layer.weight.shape)}
        if layer.bias is not None:
            f["bias"] = (False, (layer.weight.shape[0],))
        return f
    if isinstance(layer, _Dense):
        f = {"weight": (False, layer.weight.shape)}
        if layer.bias is not None:
            f["bias"] = (False, (layer.weight.shape[0],))
        return f
    if isinstance(layer, QConv2d):
        kh, kw = layer.kernel
        return {"weight": (True, (layer.filters, layer.in_channels, kh, kw))}
    if isinstance(layer, QDense):
        return {"weight": (True, (layer.units, layer.in_features))}
    if isinstance(layer, _BatchNorm):
        c = layer.gamma.shape[0]
        return {n: (False, (c,)) for n in ("gamma", "beta", "running_mean", "running_var")}
    return {}


def _packed_dims(layer):
    return (layer.filters, layer.k_reduce) if isinstance(layer, QConv2d) else \
        (layer.units, layer.in_features)


class Network(nets.Sequential):
    """Feed-forward stack + softmax head (layers.py:664-686) on the GPU."""

    def __init__(self, layers, input_shape):
        super().__init__(layers)
        self.input_shape = tuple(input_shape)
        self.head = SoftmaxOutput()
        self.fuse_bn = False  # reference layer order: keep BN separate

    def forward(self, x, mode=INFER_FLOAT, capture=None):
        _check_mode(mode)
        was_np = not isinstance(x, torch.Tensor)
        t = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda() if was_np else x
        for layer in self.layers:
            t = layer.forward(t, mode)
            if capture is not None:
                capture.append(t.cpu().numpy() if was_np else t)
        probs = self.head.forward(t, mode)
        return probs.cpu().numpy() if was_np else probs

    @property
    def quantized_layers(self):
        return [l for l in self.layers if isinstance(l, (QConv2d, QDense))]


def load_model(path) -> Network:
    """Parse a ``.bmx`` file into a GPU network, validating like modelio.load_model."""
    buf = open(path, "rb").read()
    off = 0

    def take(n):
        nonlocal off
        if off + n > len(buf):
            raise ModelFormatError(f"truncated file: wanted {n} bytes at offset {off}, "
                                   f"have {len(buf) - off}")
        out = buf[off:off + n]
        off += n
        return out

    def unpack(fmt):
        return struct.unpack(fmt, take(struct.calcsize(fmt)))

    if take(4) != MAGIC:
        raise ModelFormatError(f"bad magic; not a {MAGIC.decode()} model file")
    (version,) = unpack("<I")
    if version != VERSION:
        raise ModelFormatError(f"unsupported version {version} (expected {VERSION})")
    (arch_len,) = unpack("<I")
    try:
        arch = json.loads(take(arch_len).decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise ModelFormatError(f"arch descriptor is not valid JSON: {exc}") from None
    for key in ("input_shape", "layers"):
        if key not in arch:
            raise ModelFormatError(f"arch descriptor missing {key!r}")
    if arch.get("head", {}).get("kind", "softmax") != "softmax":
        raise ModelFormatError(f"unknown head kind {arch['head'].get('kind')!r}")
    layers = [_layer_from_spec(spec) for spec in arch["layers"]]
    expected = [_expected_fields(l) for l in layers]
    seen = set()
    (count,) = unpack("<I")
    for _ in range(count):
        (name_len,) = unpack("<H")
        name = take(name_len).decode("utf-8")
        dtype, ndim = unpack("<BB")
        dims = unpack(f"<{ndim}Q")
        prefix, _, fieldname = name.partition(".")
        try:
            idx = int(prefix[5:]) if prefix.startswith("layer") else -1
        except ValueError:
            idx = -1
        if not (0 <= idx < len(layers)) or fieldname not in expected[idx]:
            raise ModelFormatError(f"tensor {name!r} does not match the arch descriptor")
        if name in seen:
            raise ModelFormatError(f"duplicate tensor {name!r}")
        seen.add(name)
        allows_packed, want = expected[idx][fieldname]
        layer = layers[idx]
        if dtype == DTYPE_F32:
            if tuple(dims) != tuple(want):
                raise ModelFormatError(f"tensor {name!r} has dims {tuple(dims)}, arch expects "
                                       f"{tuple(want)}")
            n = int(np.prod(dims, dtype=np.int64)) if dims else 1
            arr = np.frombuffer(take(4 * n), dtype="<f4").reshape(dims).copy()
            attr = {"running_mean": "mean", "running_var": "var"}.get(fieldname, fieldname)
            setattr(layer, attr, arr)
        elif dtype == DTYPE_PACKED1:
            if not allows_packed:
                raise ModelFormatError(f"tensor {name!r} cannot be bit-packed")
            if tuple(dims) != _packed_dims(layer):
                raise ModelFormatError(f"tensor {name!r} has dims {tuple(dims)}, arch expects "
                                       f"{_packed_dims(layer)}")
            rows, cols = (int(d) for d in dims)
            words = np.frombuffer(take(8 * rows * words_per_bits(cols)), dtype="<u8")
            words = words.reshape(rows, words_per_bits(cols)).copy()
            rem = cols % 64
            if rem and np.any(words[:, -1] & np.uint64(~((1 << rem) - 1) & 0xFFFFFFFFFFFFFFFF)):
                raise ModelFormatError(f"tensor {name!r}: padding audit failed: tail bits of "
                                       "layout 'a' matrix are not all 0")
            layer.load_packed(words, cols)
        else:
            raise ModelFormatError(f"unknown tensor dtype code {dtype}")
    if off != len(buf):
        raise ModelFormatError(f"{len(buf) - off} trailing bytes after last tensor")
    for idx, fields in enumerate(expected):
        for f in fields:
            if f"layer{idx}.{f}" not in seen:
                raise ModelFormatError(f"missing tensor layer{idx}.{f}")
    for l in layers:
        if isinstance(l, _BatchNorm):
            l.finalize()
        if isinstance(l, (QConv2d, QDense)) and l.packed is None and l.weight is not None:
            l.weight = np.asarray(l.weight, np.float32)
    return Network(layers, arch["input_shape"])
