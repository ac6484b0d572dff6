"""C-ABI and host-logic tests that run without a GPU.

The library must load and export every symbol include/bnn_b200.h declares;
argument validation happens before any CUDA call, so the reference's
ValueError cases can be checked here.
"""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bnn_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1705_09864_b200 import _lib, build
    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(bnn_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(lib):
    from paper_1705_09864_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 14
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(raw, s), f"{s} not exported"
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_library_is_sm100a_only():
    from paper_1705_09864_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(8\d|90)", out)


def test_status_strings(lib):
    assert lib.bnn_abi_version() == 2
    assert lib.bnn_status_string(0) == b"ok"
    assert b"float32" in lib.bnn_status_string(-3)


def _gemm(lib, **kw):
    args = dict(A=1, lda=1, B=1, ldb=1, M=1, N=1, K=1, a_pad=0, b_pad=1, C=1, ldc_m=1, ldc_n=1,
                domain=0, scale=None, shift=None, algo=0, stream=None)
    args.update(kw)
    return lib.bnn_xnor_gemm(*args.values())


def test_gemm_validation_mirrors_gemmdims(lib):
    # GemmDims (gemm.py:170-177): dims >= 1, K < 2^24; pads in {0, 1}
    for bad in (dict(M=0), dict(N=0), dict(K=0), dict(M=-1)):
        assert _gemm(lib, **bad) == -2
    assert b"must be positive" in lib.bnn_last_error()
    assert _gemm(lib, K=1 << 24, lda=1 << 18, ldb=1 << 18) == -3
    assert b"exactness" in lib.bnn_last_error()
    assert _gemm(lib, a_pad=2) == -4
    assert _gemm(lib, K=130, lda=2) == -5  # lda < ceil(K/64)
    assert _gemm(lib, domain=7) == -1
    assert _gemm(lib, algo=99) == -7
    assert _gemm(lib, algo=2, M=0) == -2  # validation precedes engine dispatch


def test_gemm_ws_validation_and_workspace_size(lib):
    # bnn_xnor_gemm_ws: the same GemmDims validation, before any dispatch; workspace =
    # 16 bytes of e2m1 codes per 32 bits of every operand row
    assert lib.bnn_xnor_gemm_ws_bytes(256, 224, 256) == (256 + 224) * 8 * 16
    assert lib.bnn_xnor_gemm_ws_bytes(3, 5, 65) == 8 * 4 * 16
    assert lib.bnn_xnor_gemm_ws_bytes(0, 5, 65) == 0
    base = [1, 1, 1, 1, 4, 4, 64, 0, 0, 1, 4, 1, 0, 0, None, 0, None]
    for pos, bad, rc in ((4, 0, -2), (6, 1 << 24, -3), (7, 2, -4), (12, 7, -1), (13, 99, -7)):
        a = list(base)
        a[pos] = bad
        if pos == 6:
            a[1] = a[3] = 1 << 18
        assert lib.bnn_xnor_gemm_ws(*a) == rc, (pos, bad)
    a = list(base)
    a[15] = -1
    assert lib.bnn_xnor_gemm_ws(*a) == -1  # negative workspace size
    from paper_1705_09864_b200.gemm import xp_eligible
    assert xp_eligible(8192, 8192, 8192) and xp_eligible(4096, 4096, 4096)
    assert not xp_eligible(256, 1024, 4096) and not xp_eligible(4096, 4096, 1024)


def test_conv_and_pack_validation(lib):
    # tensor.conv_output_hw (tensor.py:15-27): kernel must fit, stride >= 1
    rc = lib.bnn_bconv2d(1, 1, 1, 3, 3, 1, 1, 5, 5, 1, 1, 0, 0, 1, 0, None, None, 0, None)
    assert rc == -6 and b"does not fit" in lib.bnn_last_error()
    rc = lib.bnn_bconv2d(1, 1, 1, 3, 3, 1, 1, 2, 2, 0, 1, 0, 0, 1, 0, None, None, 0, None)
    assert rc == -6
    assert lib.bnn_pack_rows_f32(1, 1, 4, 4, 1, 1, 2, 0, None, None, None) == -4
    assert lib.bnn_pack_rows_f32(1, 1, 130, 130, 1, 2, 0, 0, None, None, None) == -5
    assert lib.bnn_pack_cols_f32(1, 4, 4, 4, 1, 4, 0, 5, None, None) == -1
    assert lib.bnn_conv_channel_words(64) == 1 and lib.bnn_conv_channel_words(65) == 2
    assert lib.bnn_audit_padding(1, 1, 70, 1, 1, 3, 1, None) == -4
    # split-K combine: sizes, stride, domain and GemmDims' K bound, checked before any launch
    assert lib.bnn_sum_partials_f32(1, 0, 4, 4, 0, 64, 1, None) == -1
    assert lib.bnn_sum_partials_f32(1, 2, 8, 4, 0, 64, 1, None) == -5  # stride < count
    assert lib.bnn_sum_partials_f32(1, 2, 4, 4, 5, 64, 1, None) == -1
    assert lib.bnn_sum_partials_f32(1, 2, 4, 4, 1, 1 << 24, 1, None) == -3
    assert lib.bnn_sum_partials_f32(None, 2, 4, 4, 0, 64, None, None) == -1
    assert lib.bnn_sum_partials_f32(None, 2, 0, 0, 0, 64, None, None) == 0  # empty: no launch


def test_host_split_k_ranges():
    """DensePlan's opt-in host split-K ranges: word-aligned, whole 256-bit superstages,
    contiguous, covering [0, K) with the tail in the last range only."""
    from types import SimpleNamespace
    from paper_1705_09864_b200.plan import DensePlan
    assert DensePlan._k_chunks(SimpleNamespace(k=4096), None) == [(0, 4096)]  # off by default
    for splits, k in [(8, 4096), (3, 4096), (2, 1000), (5, 2047), (16, 8192), (4, 200), (7, 64)]:
        ch = DensePlan._k_chunks(SimpleNamespace(k=k), splits)
        assert ch[0][0] == 0 and ch[-1][1] == k
        assert all(a1 == b0 for (_, a1), (b0, _) in zip(ch[:-1], ch[1:]))
        assert all(k0 % 256 == 0 and k1 > k0 for k0, k1 in ch)
        assert all((k1 - k0) % 256 == 0 for k0, k1 in ch[:-1])
        assert 1 <= len(ch) <= splits
    assert DensePlan._k_chunks(SimpleNamespace(k=4096), 8) == [(512 * i, 512 * (i + 1)) for i in range(8)]


def test_host_gemm_dims_and_workers(monkeypatch):
    from paper_1705_09864_b200 import gemm
    d = gemm.GemmDims(2, 3, 65)
    assert d.words_per_k == 2 and d.binary_ops == 2 * 2 * 3 * 65
    for bad in ((0, 1, 1), (1, 0, 1), (1, 1, 0), (-1, 2, 2)):
        with pytest.raises(ValueError):
            gemm.GemmDims(*bad)
    with pytest.raises(ValueError):
        gemm.GemmDims(1, 1, 1 << 24)
    # resolve_workers precedence (test_gemm.py:62-75)
    monkeypatch.delenv(gemm.THREADS_ENV_VAR, raising=False)
    assert gemm.resolve_workers(3) == 3
    monkeypatch.setenv(gemm.THREADS_ENV_VAR, "5")
    assert gemm.resolve_workers() == 5 and gemm.resolve_workers(2) == 2
    monkeypatch.setenv(gemm.THREADS_ENV_VAR, "junk")
    with pytest.raises(ValueError):
        gemm.resolve_workers()
    monkeypatch.setenv(gemm.THREADS_ENV_VAR, "0")
    with pytest.raises(ValueError):
        gemm.resolve_workers()


def test_host_bitmatrix_validation():
    from paper_1705_09864_b200.bitpack import BitMatrix, words_per_bits
    words = np.zeros((2, 1), dtype=np.uint64)
    with pytest.raises(ValueError):
        BitMatrix(words, vectors=2, n_bits=10, layout="c", pad_fill=0)
    with pytest.raises(ValueError):
        BitMatrix(words, vectors=2, n_bits=10, layout="a", pad_fill=2)
    with pytest.raises(ValueError):
        BitMatrix(words, vectors=3, n_bits=10, layout="a", pad_fill=0)
    with pytest.raises(ValueError):
        BitMatrix(words.astype(np.int64), vectors=2, n_bits=10, layout="a", pad_fill=0)
    with pytest.raises(ValueError):
        BitMatrix(words, vectors=2, n_bits=80, layout="b", pad_fill=1)
    assert [words_per_bits(n) for n in (0, 1, 63, 64, 65, 128, 129)] == [0, 1, 1, 1, 2, 2, 3]


def test_host_csv_schema_and_checksum():
    from paper_1705_09864_b200 import gemm
    rec = gemm.BenchRecord("xnor_base", 2, 3, 4, 5, 1000, 10, 99, 1)
    assert gemm.CSV_HEADER == "kernel,M,N,K,repeats,median_ns,pack_ns,checksum,seed"
    assert rec.to_csv_row() == "xnor_base,2,3,4,5,1000,10,99,1"
    text = gemm.records_to_csv([rec, rec])
    assert text.splitlines()[0] == gemm.CSV_HEADER and text.endswith("\n")
    dims = gemm.GemmDims(3, 4, 129)
    a, b = gemm.make_operands(dims, seed=3)
    dot = a.astype(np.float64) @ b.astype(np.float64)
    p = (dot + 129) / 2
    assert gemm.checksum_popcount(p, "xnor_base", dims) == int(p.sum())
    assert gemm.checksum_popcount(dot, "naive_f32", dims) == int(p.sum())


def test_host_layer_constructors():
    from paper_1705_09864_b200 import layers
    with pytest.raises(ValueError):
        layers.QConv2d(3, 4, (3, 3), pad=(1, 1))  # layers.py:178-180
    q = layers.QConvolution(3, 4, (3, 3), pad=(1, 1))  # BMXNet name accepts pad (G2)
    assert q.k_reduce == 27 and q.act_bit == q.weight_bit == 1
    with pytest.raises(ValueError):
        layers.QDense(4, 5, bits=0)
    with pytest.raises(ValueError):
        layers.QFullyConnected(4, 5, act_bit=1, weight_bit=2)
    rng = np.random.default_rng(0)
    d = layers.QDense(100, 50, rng=rng)
    assert np.abs(d.weight).max() <= np.sqrt(6.0 / 150)
    qd = layers.QDense(8, 3, bits=2)
    with pytest.raises(layers.ModeError):
        qd.pack()
    with pytest.raises(ValueError):
        layers.QActivation(1).forward(np.zeros(3), "bogus")
    with pytest.raises(layers.ModeError):
        layers.QActivation(1).forward(np.zeros(3), layers.TRAIN_FLOAT)


def test_sign_pack_and_stem_validation(lib):
    """Argument checks of the fused sign-pack epilogue and the float stem entry
    points (no CUDA call is made before validation fails)."""
    import ctypes
    from paper_1705_09864_b200 import _lib as L
    e = L.Epilogue()
    e.domain = 1
    e.pack_out, e.pack_ld = 16, 1
    rc = lib.bnn_xnor_gemm_ex(16, 2, 16, 2, 70, 8, 128, 0, 0, 16, 8, 1, ctypes.byref(e), 1, None)
    assert rc == -7 and b"tcgen05" in lib.bnn_last_error()  # CUDA-core engines: no sign-pack
    rc = lib.bnn_xnor_gemm_ex(16, 2, 16, 2, 70, 8, 128, 0, 0, 16, 8, 1, ctypes.byref(e), 0, None)
    assert rc == -5 and b"pack_ld" in lib.bnn_last_error()  # ceil(70/64) = 2 words needed
    e2 = L.Epilogue()
    e2.domain = 1
    rc = lib.bnn_xnor_gemm_ex(16, 2, 16, 2, 70, 8, 128, 0, 0, None, 8, 1, ctypes.byref(e2), 0, None)
    assert rc == -1  # a null f32 output needs a packed output
    rc = lib.bnn_bconv2d_ex(16, 1, 64, 8, 8, 16, 64, 3, 3, 1, 1, 1, 1, None, ctypes.byref(e2), 0,
                            None)
    assert rc == -1
    # float stem conv: geometry, pointers, supported shapes
    assert lib.bnn_conv2d_f32_tc(16, 1, 3, 4, 4, 16, None, 64, 7, 7, 2, 2, 0, 0, 16, None) == -6
    assert lib.bnn_conv2d_f32_tc(None, 1, 3, 8, 8, 16, None, 64, 7, 7, 2, 2, 3, 3, 16, None) == -1
    assert lib.bnn_conv2d_f32_tc(16, 1, 3, 8, 8, 16, None, 32, 7, 7, 2, 2, 3, 3, 16, None) == -7
    assert lib.bnn_conv2d_f32_tc(16, 1, 9, 8, 8, 16, None, 64, 7, 7, 2, 2, 3, 3, 16, None) == -7
    args = [16, 1, 3, 16, 16, 16, 64, 7, 7, 2, 2, 3, 3, 16, 16, 16, 16, 1, 16, None]
    args[6] = 48  # F != 64
    assert lib.bnn_conv_bn_relu_maxpool_f32_tc(*args) == -7
    args[6], args[4] = 64, 18  # W % 4 != 0
    assert lib.bnn_conv_bn_relu_maxpool_f32_tc(*args) == -7
    args[4], args[13] = 16, None
    assert lib.bnn_conv_bn_relu_maxpool_f32_tc(*args) == -1


def test_lenet_stem_and_packed_pool_validation(lib):
    assert lib.bnn_maxpool_packed(16, 1, 1, 4, 1, 2, 2, 16, None) == -6  # window taller than H
    assert lib.bnn_maxpool_packed(16, 1, 4, 4, 1, 2, 0, 16, None) == -6  # stride 0
    assert lib.bnn_maxpool_packed(None, 1, 4, 4, 1, 2, 2, 16, None) == -1
    args = [16, 1, 1, 28, 28, 16, None, 64, 5, 5, 1, 1, 2, 2, 0, 16, None]
    assert lib.bnn_conv_tanh_maxpool2_f32_tc(*args[:5], None, *args[6:]) == -1
    args[7] = 32  # F != 64
    assert lib.bnn_conv_tanh_maxpool2_f32_tc(*args) == -7


def test_network_launch_counter():
    """plan._count_lib_launches counts the library's compute calls of a step (the
    bench's gpu_launches for the network workloads), not its queries / setters."""
    from paper_1705_09864_b200 import _lib, plan

    def step():
        _lib.call("bnn_debug_set", _lib.DEBUG_FP4_BN, 0)  # setter: not a launch
        for _ in range(3):
            try:  # rejected in validation before any CUDA call, but counted as a launch
                _lib.call("bnn_maxpool_packed", None, 1, 4, 4, 1, 2, 2, None, None)
            except ValueError:
                pass
        _lib.call_status("bnn_conv2d_f32_tc", None, 1, 3, 8, 8, None, None, 64, 7, 7, 2, 2, 3,
                         3, None, None)

    assert plan._count_lib_launches(step) == 4
    assert _lib.call.__name__ == "call"  # restored
