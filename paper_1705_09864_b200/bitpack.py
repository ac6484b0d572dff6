"""Bit packing of +-1 matrices into 64-bit words, on the B200.

Drop-in for the reference ``bitnn.bitpack`` (``/root/reference/pkg/src/
bitnn/bitpack.py``): same word format (bit k of a vector is bit k % 64 of
u64 word k // 64, LSB-first, bit 1 <=> +1), the same two layouts ('a': [M,
W] rows with 0-filled tails, 'b': [W, N] columns with 1-filled tails), the
same ``BitMatrix`` container and the same ``ValueError`` cases.  Words live
in CUDA memory as ``torch.uint64`` tensors; every packing step is one of the
hand-written sm_100a kernels behind ``include/bnn_b200.h``.

Inputs may be NumPy arrays (returned results are then NumPy, as in the
reference) or torch tensors (results stay on the GPU).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

WORD_BITS = 64


def words_per_bits(n_bits: int) -> int:
    """bitpack.words_per_bits (bitpack.py:45-46)."""
    return (n_bits + WORD_BITS - 1) // WORD_BITS


# ----------------------------------------------------------------- helpers
def to_device_f32(x) -> tuple[torch.Tensor, bool]:
    """(contiguous CUDA float32 tensor, input_was_numpy)."""
    _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        was_np = False
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
        was_np = True
    if t.dtype != torch.float32:
        t = t.to(torch.float32)
    if not t.is_cuda:
        t = t.cuda(non_blocking=False)
    return t.contiguous(), was_np


def to_device_words(w) -> torch.Tensor:
    _lib.require_cuda()
    if isinstance(w, torch.Tensor):
        t = w
    else:
        a = np.asarray(w)
        if a.dtype != np.uint64:
            raise ValueError("words must be uint64")
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype not in (torch.uint64, torch.int64):
        raise ValueError("words must be uint64")
    if t.dtype == torch.int64:
        t = t.view(torch.uint64)
    return t.cuda().contiguous() if not t.is_cuda else t.contiguous()


def _new_flags() -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device="cuda")


def raise_on_flags(flags: torch.Tensor, finite_msg: str = "binarize requires finite inputs"):
    """Read the pack kernel's flag word (one device sync) and raise like the reference."""
    f = int(flags.item())
    if f & _lib.FLAG_NONFINITE:
        raise ValueError(finite_msg)
    if f & _lib.FLAG_NOTSIGN:
        raise ValueError("matrix entries must all be -1 or +1")
    if f & _lib.FLAG_RANGE:
        raise ValueError("quantize requires inputs in [0, 1]")


def _out(t: torch.Tensor, was_np: bool):
    return t.cpu().numpy() if was_np else t


# ----------------------------------------------------------------- binarize
def binarize(x):
    """bitpack.binarize (bitpack.py:30-42): sign with sign(0) = sign(-0) = +1.

    Non-finite entries raise ValueError.  Returns float32 +-1.
    """
    t, was_np = to_device_f32(x)
    out = torch.empty_like(t)
    flags = _new_flags()
    _lib.call("bnn_binarize_f32", _lib.ptr(t), t.numel(), _lib.ptr(out), _lib.ptr(flags),
              _lib.stream_ptr())
    raise_on_flags(flags)
    return _out(out, was_np)


# ----------------------------------------------------------------- BitMatrix
@dataclass
class BitMatrix:
    """A +-1 matrix packed into 64-bit words (bitpack.py:90-141).

    ``words`` is [vectors, words_per_k] for layout 'a' and [words_per_k,
    vectors] for layout 'b'; on this framework it is a CUDA uint64 tensor.
    """

    words: torch.Tensor
    vectors: int
    n_bits: int
    layout: str
    pad_fill: int

    def __post_init__(self):
        if self.layout not in ("a", "b"):
            raise ValueError(f"layout must be 'a' or 'b', got {self.layout!r}")
        if self.pad_fill not in (0, 1):
            raise ValueError(f"pad_fill must be 0 or 1, got {self.pad_fill}")
        if isinstance(self.words, np.ndarray):
            if self.words.dtype != np.uint64:
                raise ValueError("words must be uint64")
        elif not isinstance(self.words, torch.Tensor) or self.words.dtype != torch.uint64:
            raise ValueError("words must be uint64")
        expect = ((self.vectors, self.words_per_vector) if self.layout == "a"
                  else (self.words_per_vector, self.vectors))
        if tuple(self.words.shape) != expect:
            raise ValueError(f"words shape {tuple(self.words.shape)} != expected {expect}")
        if isinstance(self.words, np.ndarray):
            self.words = to_device_words(self.words)

    @property
    def words_per_vector(self) -> int:
        return words_per_bits(self.n_bits)

    @property
    def nbytes(self) -> int:
        return self.words.numel() * 8

    def vector_words(self, i: int) -> torch.Tensor:
        return self.words[i] if self.layout == "a" else self.words[:, i]

    def rows(self) -> torch.Tensor:
        """K-contiguous [vectors, W] words (layout 'b' transposed on device)."""
        if self.layout == "a":
            return self.words.contiguous()
        return words_transpose(self.words)

    def unpack(self) -> np.ndarray:
        """Reconstruct the +-1 float32 matrix in its original orientation (host)."""
        rows = self.rows().cpu().numpy()
        flat = rows.reshape(-1).view(np.uint8) if rows.size else rows.view(np.uint8)
        bits = np.unpackbits(flat, bitorder="little").reshape(
            self.vectors, self.words_per_vector * WORD_BITS)
        signs = np.where(bits[:, : self.n_bits] == 1, 1.0, -1.0).astype(np.float32)
        return signs if self.layout == "a" else signs.T


# ----------------------------------------------------------------- packing
def pack_rows_device(x: torch.Tensor, pad_fill: int = 0, strict: bool = False,
                     flags: torch.Tensor | None = None,
                     row_popc: torch.Tensor | None = None) -> torch.Tensor:
    """Fused sign + pack of a CUDA f32 [R, K] matrix into [R, ceil(K/64)] words.

    No host sync: non-finite / non-sign inputs are OR-ed into ``flags``.
    """
    if x.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={x.dim()}")
    r, k = x.shape
    ld = x.stride(0) if x.stride(1) == 1 else None
    if ld is None:
        x = x.contiguous()
        ld = k
    out = torch.empty((r, words_per_bits(k)), dtype=torch.uint64, device=x.device)
    _lib.call("bnn_pack_rows_f32", _lib.ptr(x), r, k, max(ld, k), _lib.ptr(out),
              out.shape[1], pad_fill, _lib.PACK_STRICT if strict else _lib.PACK_SIGN,
              _lib.ptr(row_popc), _lib.ptr(flags), _lib.stream_ptr())
    return out


def pack_matrix_a(mat) -> BitMatrix:
    """pack_matrix_a (bitpack.py:144-149): +-1 rows [M, K], 0-filled tails."""
    t, _ = to_device_f32(mat)
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={t.dim()}")
    flags = _new_flags()
    words = pack_rows_device(t, 0, strict=True, flags=flags)
    raise_on_flags(flags)
    m, k = t.shape
    return BitMatrix(words=words, vectors=m, n_bits=k, layout="a", pad_fill=0)


def pack_matrix_b(mat) -> BitMatrix:
    """pack_matrix_b (bitpack.py:152-169): +-1 columns of [K, N] -> [W, N], 1-filled tails."""
    t, _ = to_device_f32(mat)
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={t.dim()}")
    k, n = t.shape
    out = torch.empty((words_per_bits(k), n), dtype=torch.uint64, device=t.device)
    flags = _new_flags()
    _lib.call("bnn_pack_cols_f32", _lib.ptr(t), k, n, n, _lib.ptr(out), n, 1, _lib.PACK_STRICT,
              _lib.ptr(flags), _lib.stream_ptr())
    raise_on_flags(flags)
    return BitMatrix(words=out, vectors=n, n_bits=k, layout="b", pad_fill=1)


def pack_row(values, pad_fill: int = 0):
    """pack_row (bitpack.py:172-182): one +-1 vector -> u64 words."""
    t, was_np = to_device_f32(values)
    if t.dim() != 1:
        raise ValueError("pack_row expects a 1-D vector")
    if pad_fill not in (0, 1):
        raise ValueError(f"pad_fill must be 0 or 1, got {pad_fill}")
    if t.numel() == 0:
        out = torch.zeros(0, dtype=torch.uint64, device="cuda")
        return _out(out, was_np)
    flags = _new_flags()
    out = pack_rows_device(t[None, :], pad_fill, strict=True, flags=flags)[0]
    raise_on_flags(flags)
    return _out(out, was_np)


def unpack_row(words, n_bits: int) -> np.ndarray:
    """unpack_row (bitpack.py:184-194) (host-side inverse, for tests)."""
    w = words.cpu().numpy() if isinstance(words, torch.Tensor) else np.asarray(words)
    w = np.ascontiguousarray(w, dtype=np.uint64)
    if w.ndim != 1:
        raise ValueError("unpack_row expects a 1-D word array")
    if w.size != words_per_bits(n_bits):
        raise ValueError(f"{w.size} words cannot hold {n_bits} bits")
    if n_bits == 0:
        return np.zeros(0, dtype=np.float32)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:n_bits]
    return np.where(bits == 1, 1.0, -1.0).astype(np.float32)


def pack_nchw(x: torch.Tensor, strict: bool = False,
              flags: torch.Tensor | None = None) -> torch.Tensor:
    """NCHW f32 -> packed NHWC words [B, H, W, ceil(C/64)] (sign on the fly)."""
    if x.dim() != 4:
        raise ValueError(f"expected [B, C, H, W] input, got ndim={x.dim()}")
    x = x.contiguous()
    b, c, h, w = x.shape
    out = torch.empty((b, h, w, words_per_bits(c)), dtype=torch.uint64, device=x.device)
    _lib.call("bnn_pack_nchw_f32", _lib.ptr(x), b, c, h, w, _lib.ptr(out),
              _lib.PACK_STRICT if strict else _lib.PACK_SIGN, _lib.ptr(flags), _lib.stream_ptr())
    return out


def pack_planes_device(x: torch.Tensor, bits: int = 2, grid: str = "signed",
                       flags: torch.Tensor | None = None) -> torch.Tensor:
    """k-bit quantize + bit-plane pack of a CUDA f32 [R, K] matrix -> [bits, R, W] u64.

    Codes follow qmath.quantize / quantize_signed (qmath.py:50-84) bit for bit;
    plane p holds bit p of every code.  No host sync (flags as pack_rows_device).
    """
    if x.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={x.dim()}")
    x = x.contiguous()
    r, k = x.shape
    w = words_per_bits(k)
    out = torch.empty((bits, r, w), dtype=torch.uint64, device=x.device)
    g = _lib.GRID_SIGNED if grid == "signed" else _lib.GRID_UNSIGNED
    _lib.call("bnn_pack_planes_f32", _lib.ptr(x), r, k, k, bits, g, _lib.ptr(out), w, r * w,
              _lib.ptr(flags), _lib.stream_ptr())
    return out


def words_transpose(words: torch.Tensor) -> torch.Tensor:
    """[R, C] u64 -> [C, R] u64 on the device (layout 'b' <-> K-contiguous rows)."""
    r, c = words.shape
    out = torch.empty((c, r), dtype=torch.uint64, device=words.device)
    _lib.call("bnn_words_transpose", _lib.ptr(words), r, c, words.stride(0), _lib.ptr(out), r,
              _lib.stream_ptr())
    return out


def audit_padding(bm: BitMatrix) -> None:
    """audit_padding (bitpack.py:197-215): raise if a tail bit disagrees with the fill."""
    if bm.n_bits % WORD_BITS == 0:
        return
    bad = _new_flags()
    w = bm.words
    if bm.layout == "a":
        ld_vec, ld_word = w.stride(0), w.stride(1)
    else:
        ld_vec, ld_word = w.stride(1), w.stride(0)
    _lib.call("bnn_audit_padding", _lib.ptr(w), bm.vectors, bm.n_bits, ld_vec, ld_word,
              bm.pad_fill, _lib.ptr(bad), _lib.stream_ptr())
    if int(bad.item()):
        raise ValueError(f"padding audit failed: tail bits of layout {bm.layout!r} matrix "
                         f"are not all {bm.pad_fill}")


def _popcount64(words, soft: int):
    was_np = not isinstance(words, torch.Tensor)
    w = to_device_words(np.asarray(words, dtype=np.uint64) if was_np else words)
    out = torch.empty(w.shape, dtype=torch.uint8, device=w.device)
    _lib.call("bnn_popcount64", _lib.ptr(w), w.numel(), _lib.ptr(out), soft, _lib.stream_ptr())
    return out.cpu().numpy() if was_np else out


def popcount64(words):
    """popcount64 (bitpack.py:49-52): per-element popcount of u64 words (POPC), as u8."""
    return _popcount64(words, 0)


def popcount64_soft(words):
    """popcount64_soft (bitpack.py:55-66): the shift/mask popcount, bit-identical to
    ``popcount64`` (the reference pins the two against each other)."""
    return _popcount64(words, 1)


def dot_xnor_popcount(a_words, b_words, n_bits: int) -> int:
    """dot_xnor_popcount (bitpack.py:218-231): agreement count of two packed vectors.

    Expects the 'a'/'b' packing pair (0- and 1-filled tails), as the reference.
    """
    from .gemm import xnor_rows_gemm

    a = to_device_words(a_words)
    b = to_device_words(b_words)
    wpk = words_per_bits(n_bits)
    if tuple(a.shape) != (wpk,) or tuple(b.shape) != (wpk,):
        raise ValueError(f"expected {wpk} words per operand for n_bits={n_bits}")
    c = xnor_rows_gemm(a[None, :], b[None, :], n_bits, a_pad=0, b_pad=1)
    return int(c.item())
