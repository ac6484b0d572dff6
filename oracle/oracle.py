"""CPU oracle for the binarise -> bit-pack -> xnor-popcount path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1705_09864_b200`` imports
this module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs do, as the checker.  It is a
restatement of the reference ``bitnn`` package (``/root/reference/pkg/src/
bitnn``): the hot loops are plain C (``bnn_oracle.c``, loaded via ctypes)
and the scalar maps are NumPy.  Its parity with the reference is pinned by
``tests/test_oracle_golden.py`` against vectors produced by the reference
itself (``tests/golden/gen_golden_vectors.py``), so parity is *pinned*.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

WORD_BITS = 64  # bitpack.py:22
MAX_K_EXACT = 1 << 24  # gemm.py:43-44

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile bnn_oracle.c (gcc) into oracle/_build/liboracle.so."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.orc_binarize_f32.argtypes = [vp, i64, vp]
        L.orc_pack_rows.argtypes = [vp, i64, i64, vp, i32, i32]
        L.orc_pack_cols.argtypes = [vp, i64, i64, vp, i32, i32]
        L.orc_binarize_pack_rows.argtypes = [vp, i64, i64, vp, i32, i32]
        L.orc_xnor_gemm.argtypes = [vp, vp, i64, i64, i64, vp, i32]
        L.orc_xnor_gemm.restype = None
        L.orc_xor_popc_gemm_rowrow.argtypes = [vp, vp, i64, i64, i64, vp, i32]
        L.orc_xor_popc_gemm_rowrow.restype = None
        L.orc_im2col_f32.argtypes = [vp] + [i32] * 10 + [vp, i32]
        _lib = L
    return _lib


def _threads(threads):
    if threads is None:
        threads = int(os.environ.get("BMX_THREADS", os.cpu_count() or 1))
    return max(1, int(threads))


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def words_per_bits(n: int) -> int:
    """bitpack.words_per_bits (bitpack.py:45-46)."""
    return (n + WORD_BITS - 1) // WORD_BITS


# ---------------------------------------------------------------- bitpack
def binarize(x) -> np.ndarray:
    """bitpack.binarize (bitpack.py:30-42): x >= 0 -> +1; non-finite -> ValueError."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    if lib().orc_binarize_f32(_ptr(x), x.size, _ptr(out)) != 0:
        raise ValueError("binarize requires finite inputs")
    return out


def pack_rows(signs, pad_fill=0, threads=None) -> np.ndarray:
    """pack_matrix_a words (bitpack.py:144-149, _pack_last_axis :78-87)."""
    s = np.ascontiguousarray(signs, dtype=np.float32)
    if s.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={s.ndim}")
    r, k = s.shape
    out = np.zeros((r, words_per_bits(k)), dtype=np.uint64)
    rc = lib().orc_pack_rows(_ptr(s), r, k, _ptr(out), pad_fill, _threads(threads))
    if rc == -2:
        raise ValueError("matrix entries must all be -1 or +1")
    return out


def pack_cols(signs, pad_fill=1, threads=None) -> np.ndarray:
    """pack_matrix_b words [ceil(K/64), N] (bitpack.py:152-169)."""
    s = np.ascontiguousarray(signs, dtype=np.float32)
    if s.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={s.ndim}")
    k, n = s.shape
    out = np.zeros((words_per_bits(k), n), dtype=np.uint64)
    rc = lib().orc_pack_cols(_ptr(s), k, n, _ptr(out), pad_fill, _threads(threads))
    if rc == -2:
        raise ValueError("matrix entries must all be -1 or +1")
    return out


def binarize_pack_rows(x, pad_fill=0, threads=None) -> np.ndarray:
    """pack_matrix_a(binarize(x)) fused (gemm.py:406-408, layers.py:221)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    r, k = x.shape
    out = np.zeros((r, words_per_bits(k)), dtype=np.uint64)
    if lib().orc_binarize_pack_rows(_ptr(x), r, k, _ptr(out), pad_fill, _threads(threads)):
        raise ValueError("binarize requires finite inputs")
    return out


def audit_padding(words: np.ndarray, n_bits: int, layout: str, pad_fill: int) -> None:
    """bitpack.audit_padding (bitpack.py:197-215)."""
    rem = n_bits % WORD_BITS
    if rem == 0:
        return
    mask = np.uint64(~((1 << rem) - 1) & 0xFFFFFFFFFFFFFFFF)
    last = words[:, -1] if layout == "a" else words[-1, :]
    expected = mask if pad_fill == 1 else np.uint64(0)
    if not np.all((last & mask) == expected):
        raise ValueError(f"padding audit failed: tail bits of layout {layout!r} matrix "
                         f"are not all {pad_fill}")


# ---------------------------------------------------------------- gemm
def xnor_gemm(a_words: np.ndarray, b_words: np.ndarray, threads=None) -> np.ndarray:
    """xnor_gemm_parallel (gemm.py:254-284): popcount domain, int32 [M, N].

    ``a_words`` layout 'a' [M, W] (pad 0), ``b_words`` layout 'b' [W, N] (pad 1).
    """
    a = np.ascontiguousarray(a_words, dtype=np.uint64)
    b = np.ascontiguousarray(b_words, dtype=np.uint64)
    m, w = a.shape
    w2, n = b.shape
    if w != w2:
        raise ValueError("word counts differ")
    c = np.zeros((m, n), dtype=np.int32)
    lib().orc_xnor_gemm(_ptr(a), _ptr(b), m, n, w, _ptr(c), _threads(threads))
    return c


def xor_popc_rowrow(a_words: np.ndarray, b_rows: np.ndarray, threads=None) -> np.ndarray:
    """sum_w popc(a[m,w] ^ b[n,w]) with both operands K-contiguous."""
    a = np.ascontiguousarray(a_words, dtype=np.uint64)
    b = np.ascontiguousarray(b_rows, dtype=np.uint64)
    c = np.zeros((a.shape[0], b.shape[0]), dtype=np.int32)
    lib().orc_xor_popc_gemm_rowrow(_ptr(a), _ptr(b), a.shape[0], b.shape[0], a.shape[1],
                                   _ptr(c), _threads(threads))
    return c


# ---------------------------------------------------------------- qmath
def map_dot_to_xnor(dot, n: int):
    """qmath.map_dot_to_xnor (qmath.py:87-99)."""
    dot = np.asarray(dot)
    if n < 0 or np.any(np.abs(dot) > n):
        raise ValueError("dot product outside [-n, n]")
    return (dot + n) * 0.5


def map_xnor_to_dot(p, n: int):
    """qmath.map_xnor_to_dot (qmath.py:102-109)."""
    p = np.asarray(p)
    if n < 0 or np.any(p < 0) or np.any(p > n):
        raise ValueError("popcount outside [0, n]")
    return 2.0 * p - n


def quantize(x, bits: int):
    """qmath.quantize (qmath.py:50-65): floor(x*levels + 0.5)/levels, in x's dtype."""
    if not (2 <= bits <= 31):
        raise ValueError("bits must be in [2, 31]")
    x = np.asarray(x)
    if not np.all(np.isfinite(x)):
        raise ValueError("quantize requires finite inputs")
    if np.any(x < 0.0) or np.any(x > 1.0):
        raise ValueError("quantize requires inputs in [0, 1]")
    levels = (1 << bits) - 1
    return np.floor(x * levels + 0.5) / levels


def quantize_codes(x, bits: int) -> np.ndarray:
    """Integer codes i of quantize(x) = i / levels (same f32 op order)."""
    x = np.asarray(x)
    levels = (1 << bits) - 1
    return np.floor(x * levels + 0.5).astype(np.int64)


def quantize_signed(x, bits: int):
    """qmath.quantize_signed (qmath.py:68-84)."""
    x = np.asarray(x)
    if not np.all(np.isfinite(x)):
        raise ValueError("quantize_signed requires finite inputs")
    clamped = np.clip(x, -1.0, 1.0)
    if bits == 1:
        return np.where(clamped >= 0, 1.0, -1.0).astype(clamped.dtype)
    return 2.0 * quantize(0.5 * clamped + 0.5, bits) - 1.0


# ---------------------------------------------------------------- tensor
def conv_output_hw(h, w, kh, kw, stride=(1, 1), pad=(0, 0)):
    """tensor.conv_output_hw (tensor.py:15-27)."""
    sh, sw = stride
    ph, pw = pad
    if min(h, w, kh, kw) < 1 or min(sh, sw) < 1 or min(ph, pw) < 0:
        raise ValueError("invalid convolution geometry")
    oh = (h + 2 * ph - kh) // sh + 1
    ow = (w + 2 * pw - kw) // sw + 1
    if oh < 1 or ow < 1:
        raise ValueError("kernel does not fit input")
    return oh, ow


def im2col(x, kh, kw, stride=(1, 1), pad=(0, 0), threads=None) -> np.ndarray:
    """tensor.im2col (tensor.py:60-78): [B,C,H,W] -> [C*kh*kw, B*oh*ow], zero pad."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b, c, h, w = x.shape
    oh, ow = conv_output_hw(h, w, kh, kw, stride, pad)
    cols = np.empty((c * kh * kw, b * oh * ow), dtype=np.float32)
    rc = lib().orc_im2col_f32(_ptr(x), b, c, h, w, kh, kw, stride[0], stride[1], pad[0], pad[1],
                              _ptr(cols), _threads(threads))
    if rc:
        raise ValueError("invalid convolution geometry")
    return cols


# ---------------------------------------------------------------- compositions
def qdense_packed(x, weight, threads=None) -> np.ndarray:
    """QDense.forward(INFER_PACKED) (layers.py:361-369): popcount domain [B, units].

    xnor_gemm_parallel(pack_matrix_a(binarize(W)), pack_matrix_b(x.T)).T with
    x already +-1 (QActivation output).
    """
    aw = pack_rows(binarize(weight), 0, threads)
    bw = pack_cols(np.ascontiguousarray(np.asarray(x, np.float32).T), 1, threads)
    return xnor_gemm(aw, bw, threads).T.astype(np.float32)


def qfc_dot(x_f32, w_f32, threads=None) -> np.ndarray:
    """Config 1: K - 2 popc(A xor W) = map_xnor_to_dot(P, K), shape [batch, units]."""
    k = x_f32.shape[1]
    aw = binarize_pack_rows(w_f32, 0, threads)
    bw = pack_cols(binarize(np.ascontiguousarray(np.asarray(x_f32, np.float32).T)), 1, threads)
    p = xnor_gemm(aw, bw, threads).T
    return (2 * p.astype(np.int64) - k).astype(np.float32)


def qconv_packed(x, weight, stride=(1, 1), pad=(0, 0), threads=None) -> np.ndarray:
    """QConv2d.forward(INFER_PACKED) (layers.py:225-245) with the G2 padding rule.

    Composition of unmodified reference steps: im2col (zero pad) -> binarize
    (sign(0)=+1, so pad contributes +1) -> pack_matrix_b -> xnor_gemm ->
    reshape(F, B, oh, ow).transpose(1, 0, 2, 3).  Popcount domain f32 NCHW.
    """
    x = np.asarray(x, np.float32)
    weight = np.asarray(weight, np.float32)
    f, c, kh, kw = weight.shape
    b, _, h, w = x.shape
    oh, ow = conv_output_hw(h, w, kh, kw, stride, pad)
    aw = binarize_pack_rows(weight.reshape(f, c * kh * kw), 0, threads)
    cols = binarize(im2col(x, kh, kw, stride, pad, threads))
    bw = pack_cols(cols, 1, threads)
    out = xnor_gemm(aw, bw, threads).astype(np.float32)
    return np.ascontiguousarray(out.reshape(f, b, oh, ow).transpose(1, 0, 2, 3))
