"""CPU reference forward of the network runners (TEST INFRASTRUCTURE ONLY).

Walks a ``paper_1705_09864_b200.nets.Sequential`` and recomputes it on the
host with the reference's semantics: float layers in NumPy float32 (the
reference's Conv2d / Dense / BatchNorm / MaxPool / Tanh, layers.py:81-659,
via the oracle's im2col), binary layers through the pinned oracle
composition (im2col(zero pad) -> binarize -> pack -> xnor GEMM, G2).  Used as
the CPU baseline of the network workloads and for end-to-end agreement
reports; nothing in the product imports it.
"""

from __future__ import annotations

import numpy as np

from . import oracle as orc


def _np(t):
    return t if isinstance(t, np.ndarray) or t is None else t.detach().cpu().numpy()


def _conv_f32(x, w, b, stride, pad, threads=None):
    """stride / pad: (h, w) pairs."""
    n, c, h, ww = x.shape
    f, _, kh, kw = w.shape
    oh, ow = orc.conv_output_hw(h, ww, kh, kw, stride, pad)
    cols = orc.im2col(x, kh, kw, stride, pad, threads)
    out = w.reshape(f, -1) @ cols
    if b is not None:
        out = out + b[:, None]
    return np.ascontiguousarray(out.reshape(f, n, oh, ow).transpose(1, 0, 2, 3))


def _maxpool(x, k, s, p):
    n, c, h, w = x.shape
    if p:
        x = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)), constant_values=-np.inf)
    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    out = np.full((n, c, oh, ow), -np.inf, np.float32)
    for i in range(k):
        for j in range(k):
            out = np.maximum(out, x[:, :, i:i + s * oh:s, j:j + s * ow:s])
    return out


def _bn(layer, x):
    shape = (1, -1, 1, 1) if x.ndim == 4 else (1, -1)
    inv_std = (1.0 / np.sqrt(layer.var + np.float32(1e-5))).astype(np.float32)
    xhat = (x - layer.mean.reshape(shape)) * inv_std.reshape(shape)
    return layer.gamma.reshape(shape) * xhat + layer.beta.reshape(shape)


def _qconv(layer, x, threads=None):
    p = orc.qconv_packed(x, layer.weight, layer.stride, layer.pad, threads)
    return (2 * p - layer.k_reduce).astype(np.float32) if layer.domain == 1 else p


def _qfc(layer, x, threads=None):
    p = orc.qdense_packed(orc.binarize(x), layer.weight, threads)
    return (2 * p - layer.in_features).astype(np.float32) if layer.domain == 1 else p


def forward(net, x: np.ndarray, threads=None, capture=None) -> np.ndarray:
    """``capture`` (a list) receives every top-level layer's output, like
    ``Sequential.forward(..., capture=...)``."""
    from paper_1705_09864_b200 import nets
    from paper_1705_09864_b200.layers import QConvolution, QFullyConnected

    x = np.ascontiguousarray(x, np.float32)
    for layer in net.layers:
        if isinstance(layer, nets.Conv2d):
            x = _conv_f32(x, _np(layer.weight), None if layer.bias is None else _np(layer.bias),
                          (layer.sh, layer.sw), (layer.ph, layer.pw), threads)
        elif isinstance(layer, nets.Dense):
            x = x @ _np(layer.weight).T
            if layer.bias is not None:
                x = x + _np(layer.bias)
        elif isinstance(layer, nets.BatchNorm):
            x = _bn(layer, x)
        elif isinstance(layer, nets.Tanh):
            x = np.tanh(x)
        elif isinstance(layer, nets.ReLU):
            x = np.maximum(x, np.float32(0))
        elif isinstance(layer, nets.MaxPool2d):
            x = _maxpool(x, layer.k, layer.stride, layer.pad)
        elif isinstance(layer, nets.Flatten):
            x = x.reshape(x.shape[0], -1)
        elif isinstance(layer, nets.GlobalAvgPool):
            x = x.mean(axis=(2, 3), dtype=np.float32)
        elif isinstance(layer, nets.StemPost):
            x = _maxpool(np.maximum(_bn(layer.bn, x), np.float32(0)), layer.pool.k,
                         layer.pool.stride, layer.pool.pad)
        elif isinstance(layer, QConvolution):
            x = _qconv(layer, x, threads)
        elif isinstance(layer, QFullyConnected):
            x = _qfc(layer, x, threads)
        elif isinstance(layer, nets.BinaryBasicBlock):
            h = _bn(layer.bn1, _qconv(layer.conv1, x, threads))
            h = _bn(layer.bn2, _qconv(layer.conv2, h, threads))
            sc = x if layer.down is None else _bn(layer.bnd, _qconv(layer.down, x, threads))
            x = (h + sc).astype(np.float32)
        else:
            raise TypeError(f"no reference for {type(layer).__name__}")
        x = np.ascontiguousarray(x, np.float32)
        if capture is not None:
            capture.append(x)
    return x
