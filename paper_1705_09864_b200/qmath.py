"""Quantization arithmetic (drop-in for ``bitnn.qmath``, qmath.py:1-123).

The maps and quantizers are elementwise; on this framework they run on the
GPU as torch elementwise ops in float32 with the reference's exact op order
(clip -> 0.5*x + 0.5 -> *levels -> +0.5 -> floor -> /levels -> 2*q - 1), so
results are bit-identical to the NumPy float32 reference (no FMA contraction
happens in eager torch).  NumPy inputs return NumPy outputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

MIN_BITS = 1
MAX_BITS = 31


@dataclass(frozen=True)
class QuantSpec:
    """qmath.QuantSpec (qmath.py:24-41)."""

    bits: int

    def __post_init__(self):
        if not (MIN_BITS <= self.bits <= MAX_BITS):
            raise ValueError(f"bits must be in [{MIN_BITS}, {MAX_BITS}], got {self.bits}")

    @property
    def levels(self) -> int:
        return (1 << self.bits) - 1


def _as_tensor(x):
    if isinstance(x, torch.Tensor):
        return x, False
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32))), True


def _ret(t, was_np):
    return t.cpu().numpy() if was_np else t


def quantize(x, bits: int):
    """qmath.quantize (qmath.py:50-65): i / (2**bits - 1), ties half away from zero."""
    if not (2 <= bits <= MAX_BITS):
        raise ValueError(f"bits must be in [2, {MAX_BITS}], got {bits}")
    t, was_np = _as_tensor(x)
    if not bool(torch.isfinite(t).all()):
        raise ValueError("quantize requires finite inputs")
    if bool((t < 0.0).any()) or bool((t > 1.0).any()):
        raise ValueError("quantize requires inputs in [0, 1]")
    levels = float((1 << bits) - 1)
    return _ret(torch.floor(t * levels + 0.5) / levels, was_np)


def quantize_codes(x: torch.Tensor, bits: int) -> torch.Tensor:
    """Integer grid index of quantize(x, bits) (same float32 op order), int32."""
    levels = float((1 << bits) - 1)
    return torch.floor(x * levels + 0.5).to(torch.int32)


def quantize_signed(x, bits: int):
    """qmath.quantize_signed (qmath.py:68-84); 1 bit == binarize(clip(x))."""
    if not (MIN_BITS <= bits <= MAX_BITS):
        raise ValueError(f"bits must be in [{MIN_BITS}, {MAX_BITS}], got {bits}")
    t, was_np = _as_tensor(x)
    if not bool(torch.isfinite(t).all()):
        raise ValueError("quantize_signed requires finite inputs")
    clamped = torch.clamp(t, -1.0, 1.0)
    if bits == 1:
        return _ret(torch.where(clamped >= 0, 1.0, -1.0).to(t.dtype), was_np)
    return _ret(2.0 * quantize(0.5 * clamped + 0.5, bits) - 1.0, was_np)


def map_dot_to_xnor(dot, n: int):
    """qmath.map_dot_to_xnor (qmath.py:87-99): (dot + n) / 2."""
    if n < 0:
        raise ValueError("n must be non-negative")
    if isinstance(dot, torch.Tensor):
        if bool((dot.abs() > n).any()):
            raise ValueError(f"dot product outside [-{n}, {n}]")
        return (dot + n) * 0.5
    dot = np.asarray(dot)
    if np.any(np.abs(dot) > n):
        raise ValueError(f"dot product outside [-{n}, {n}]")
    return (dot + n) * 0.5


def map_xnor_to_dot(p, n: int):
    """qmath.map_xnor_to_dot (qmath.py:102-109): 2p - n."""
    if n < 0:
        raise ValueError("n must be non-negative")
    if isinstance(p, torch.Tensor):
        if bool((p < 0).any()) or bool((p > n).any()):
            raise ValueError(f"popcount outside [0, {n}]")
        return 2.0 * p - n
    p = np.asarray(p)
    if np.any(p < 0) or np.any(p > n):
        raise ValueError(f"popcount outside [0, {n}]")
    return 2.0 * p - n
