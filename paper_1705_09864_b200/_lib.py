"""ctypes binding of libbnn_b200.so (the C ABI declared in include/bnn_b200.h).

The library is the product path: if it is missing or no CUDA device is
present, every op raises instead of falling back to a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BNN_LIB_PATH") or os.path.join(_PKG, "libbnn_b200.so")  # override: dev experiments

# enum values mirrored from include/bnn_b200.h
OK, EINVAL, EDIMS, EKEXACT, EPAD, EALIGN, EGEOM, EUNSUP, ECUDA = 0, -1, -2, -3, -4, -5, -6, -7, 1
POPCOUNT, DOT = 0, 1
ALGO_AUTO, ALGO_POPC, ALGO_BMMA, ALGO_UMMA = 0, 1, 2, 3
ALGO_UMMA_V0 = 16  # tcgen05 engine variant v = ALGO_UMMA_V0 + v (v in 0..4)
ALGO_UMMA_XP = 24  # bnn_xnor_gemm_ws: pre-expanded operands + 2-CTA kind::mxf4 GEMM
ALGOS = {"auto": ALGO_AUTO, "popc": ALGO_POPC, "bmma": ALGO_BMMA, "umma": ALGO_UMMA,
         "xp": ALGO_UMMA_XP, **{f"umma{v}": ALGO_UMMA_V0 + v for v in range(5)}}
# debug knobs (bnn_debug_set; process-wide, experiment scripts only)
DEBUG_UMMA_BITS, DEBUG_FP4_BN, DEBUG_PAIR_KW32, DEBUG_STEM_BITS = 1, 2, 3, 4
DEBUG_PACK_PIX, DEBUG_PACK_CH, DEBUG_STEMPOST_SIMPLE, DEBUG_GRID_CAP = 5, 6, 7, 8
WATCHDOG_WORDS = 225
FLAG_NONFINITE, FLAG_NOTSIGN, FLAG_RANGE = 1, 2, 4
GRID_UNSIGNED, GRID_SIGNED = 0, 1
PACK_SIGN, PACK_STRICT = 0, 1

# every exported symbol and its ctypes signature (restype, argtypes)
_i64, _i32, _vp, _cp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_char_p
SIGNATURES = {
    "bnn_abi_version": (_i32, []),
    "bnn_last_error": (_cp, []),
    "bnn_status_string": (_cp, [_i32]),
    "bnn_device_sm_count": (_i32, []),
    "bnn_binarize_f32": (_i32, [_vp, _i64, _vp, _vp, _vp]),
    "bnn_popcount64": (_i32, [_vp, _i64, _vp, _i32, _vp]),
    "bnn_avgpool_fc_f32": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp]),
    "bnn_pack_rows_f32": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "bnn_pack_cols_f32": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i32, _i32, _vp, _vp]),
    "bnn_pack_nchw_f32": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _i32, _vp, _vp]),
    "bnn_words_transpose": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp]),
    "bnn_audit_padding": (_i32, [_vp, _i64, _i64, _i64, _i64, _i32, _vp, _vp]),
    "bnn_xnor_gemm": (_i32, [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp, _i64,
                             _i64, _i32, _vp, _vp, _i32, _vp]),
    "bnn_xnor_gemm_ws_bytes": (_i64, [_i64, _i64, _i64]),
    "bnn_xnor_gemm_ws": (_i32, [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp, _i64,
                                _i64, _i32, _i32, _vp, _i64, _vp]),
    "bnn_bitplane_gemm_ws": (_i32, [_vp, _i64, _i64, _i32, _vp, _i64, _i64, _i32, _i32, _i64, _i64,
                                    _i64, _vp, _i64, _i64, _i32, _vp, _i64, _vp]),
    "bnn_bconv2d_ws_bytes": (_i64, [_i64] * 11),
    "bnn_bconv2d_ws": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _i64,
                              _i64, _vp, _vp, _i32, _vp, _i64, _vp]),
    "bnn_conv_channel_words": (_i64, [_i64]),
    "bnn_conv_weights_reorder": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "bnn_bconv2d": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _i64,
                           _i64, _vp, _i32, _vp, _vp, _i32, _vp]),
    "bnn_probe_pipe_peak": (_i32, [_i32, _i64, _vp, _vp, _vp]),
    "bnn_pack_planes_f32": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _vp, _i64, _i64, _vp, _vp]),
    "bnn_bitplane_gemm": (_i32, [_vp, _i64, _i64, _i32, _vp, _i64, _i64, _i32, _i32, _i64, _i64,
                                 _i64, _vp, _i64, _i64, _vp]),
    "bnn_debug_set": (_i32, [_i32, _i64]),
    "bnn_bn_relu_maxpool_f32": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _i32,
                                       _i32, _i32, _vp, _vp]),
    "bnn_conv_bn_relu_maxpool_f32_tc": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i64,
                                               _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i32,
                                               _vp, _vp]),
    "bnn_conv_bn_relu_maxpool_pack_f32_tc": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64,
                                                    _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp,
                                                    _vp, _i32, _vp, _vp, _vp, _vp]),
    "bnn_conv_tanh_maxpool2_f32_tc": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _i64,
                                             _i64, _i64, _i64, _i64, _i64, _i32, _vp, _vp]),
    "bnn_conv_tanh_maxpool2_pack_f32_tc": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _i64,
                                                  _i64, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _vp,
                                                  _vp]),
    "bnn_probe_tanh_monotone": (_i32, [_vp, _vp]),
    "bnn_sum_partials_f32": (_i32, [_vp, _i32, _i64, _i64, _i32, _i64, _vp, _vp]),
    "bnn_add_pack_nchw_f32": (_i32, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "bnn_maxpool_packed": (_i32, [_vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp, _vp]),
    "bnn_maxpool_packed_ld": (_i32, [_vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp, _i64, _vp]),
    "bnn_conv2d_f32_tc": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _i64, _i64,
                                 _i64, _i64, _i64, _vp, _vp]),
    "bnn_xnor_gemm_ex": (_i32, [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp, _i64,
                                _i64, _vp, _i32, _vp]),
    "bnn_bconv2d_ex": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64,
                              _i64, _i64, _vp, _vp, _i32, _vp]),
    "bnn_umma_trace": (_i32, [_vp]),
    "bnn_debug_stamp": (_i32, [_vp, _vp]),
    "bnn_umma_watchdog": (_i32, [_vp]),
}


class Epilogue(ctypes.Structure):
    """struct bnn_epilogue (include/bnn_b200.h)."""
    _fields_ = [("domain", ctypes.c_int), ("scale", ctypes.c_void_p), ("shift", ctypes.c_void_p),
                ("bn_mean", ctypes.c_void_p), ("bn_inv_std", ctypes.c_void_p),
                ("bn_gamma", ctypes.c_void_p), ("bn_beta", ctypes.c_void_p),
                ("residual", ctypes.c_void_p), ("pack_out", ctypes.c_void_p),
                ("pack_ld", ctypes.c_int64), ("pack_flags", ctypes.c_void_p)]


class BnnError(RuntimeError):
    """A CUDA-side failure inside libbnn_b200 (status > 0)."""


_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library and bind every symbol (no CUDA calls made)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_1705_09864_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def require_cuda(t: torch.Tensor | None = None) -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1705_09864_b200 needs a CUDA device (B200); no CPU fallback")
    if t is not None and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception types."""
    if status == OK:
        return
    msg = (_lib.bnn_last_error() or b"").decode() if _lib is not None else ""
    if status > 0:
        raise BnnError(f"{what}: {msg}")
    raise ValueError(msg or what)


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)


def call_status(name: str, *args) -> int:
    """Call without raising: the status code (callers that handle BNN_EUNSUP)."""
    return int(getattr(load(), name)(*args))
