"""B200-native binarise -> bit-pack -> xnor-popcount path (BMXNet, arXiv 1705.09864).

Drop-in for the hot path of the reference ``bitnn`` package: the packing
helpers, the xnor GEMM kernels and the quantized layers, backed by
hand-written sm_100a CUDA kernels in ``libbnn_b200.so`` (C ABI:
``include/bnn_b200.h``).  There is no CPU fallback.
"""

from . import _lib
from .bitpack import (BitMatrix, WORD_BITS, audit_padding, binarize, dot_xnor_popcount,
                      pack_matrix_a, pack_matrix_b, pack_nchw, pack_row, pack_rows_device,
                      popcount64, popcount64_soft, unpack_row, words_per_bits, words_transpose)
from .gemm import (KERNEL_IDS, BenchRecord, GemmDims, benchmark_kernel, run_kernel,
                   xnor_gemm_b200, xnor_gemm_base, xnor_gemm_base_soft, xnor_gemm_blocked,
                   xnor_gemm_parallel, xnor_gemm_unrolled, xnor_rows_gemm)
from .layers import (INFER_FLOAT, INFER_PACKED, TRAIN_FLOAT, ModeError, QActivation, QConv2d,
                     QConvolution, QDense, QFullyConnected)
from .qmath import map_dot_to_xnor, map_xnor_to_dot, quantize, quantize_signed

__version__ = "0.1.0"


def load_library():
    """Load libbnn_b200.so (raises ImportError with a build hint if absent)."""
    return _lib.load()
