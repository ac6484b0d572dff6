"""bitnn/gemm_b200.py -- the file a ``bitnn`` maintainer adds to register the B200
kernel.  Reference-side binding only: plain ctypes over
the C ABI of libbnn_b200.so (include/bnn_b200.h); no code of this repository's
Python package is imported.

Contract: identical to ``bitnn.gemm.xnor_gemm_base`` (gemm.py:226-230) --
``BitMatrix`` operands of layouts ('a', 'b') with complementary tail fills (0, 1),
validated by the reference's own ``_check_operands`` (gemm.py:212-223), result the
popcount domain as a new float32 NumPy array [M, N].  Negative status codes raise
``ValueError`` (each ``BNN_E*`` mirrors a reference ``ValueError`` case), positive
ones ``RuntimeError``.

In ``bitnn/gemm.py`` the maintainer then adds ``"xnor_b200"`` to ``KERNEL_IDS``
(gemm.py:294) and one branch in ``run_kernel`` (gemm.py:297-324):

    if kernel == "xnor_b200":
        from .gemm_b200 import xnor_gemm_b200
        return xnor_gemm_b200(a_bm, b_bm)
"""

import ctypes
import os

import numpy as np
import torch

_LIB_PATH = os.environ.get("BITNN_B200_LIB", "libbnn_b200.so")
_i64, _int, _vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
_L = None


def _lib():
    global _L
    if _L is None:
        lib = ctypes.CDLL(_LIB_PATH)
        lib.bnn_xnor_gemm.argtypes = [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _int, _int, _vp,
                                      _i64, _i64, _int, _vp, _vp, _int, _vp]
        lib.bnn_words_transpose.argtypes = [_vp, _i64, _i64, _i64, _vp, _i64, _vp]
        lib.bnn_last_error.restype = ctypes.c_char_p
        _L = lib
    return _L


def _raise(rc):
    msg = _lib().bnn_last_error().decode()
    raise (ValueError if rc < 0 else RuntimeError)(msg)


def xnor_gemm_b200(a, b):
    """BitMatrix('a', pad 0) x BitMatrix('b', pad 1) -> popcount-domain float32 [M, N]."""
    from .gemm import _check_operands
    _check_operands(a, b)  # the reference's validation, unchanged
    lib = _lib()
    m, n, k = a.vectors, b.vectors, a.n_bits
    w = (k + 63) // 64
    s = torch.cuda.current_stream().cuda_stream
    aw = torch.from_numpy(np.ascontiguousarray(a.words).view(np.int64)).cuda()  # [M, W]
    bw = torch.from_numpy(np.ascontiguousarray(b.words).view(np.int64)).cuda()  # [W, N]
    bt = torch.empty((n, w), dtype=torch.int64, device="cuda")                  # [N, W]
    rc = lib.bnn_words_transpose(bw.data_ptr(), w, n, n, bt.data_ptr(), w, s)
    if rc:
        _raise(rc)
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    # a_pad 0, b_pad 1 (complementary tails), C[m, n] at m * n + n, popcount domain,
    # no affine, engine AUTO
    rc = lib.bnn_xnor_gemm(aw.data_ptr(), w, bt.data_ptr(), w, m, n, k, 0, 1, c.data_ptr(), n, 1,
                           0, None, None, 0, s)
    if rc:
        _raise(rc)
    return c.cpu().numpy()
