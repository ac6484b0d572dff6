"""The reference-side binding of INTEGRATION.md section 2 (integration/bitnn/gemm_b200.py),
executed as a ``bitnn`` maintainer would: imported inside a ``bitnn`` package whose
``gemm._check_operands`` is the reference's validation (here its restatement in this
package, gemm.py:212-223) and fed the reference-packed words of the 40-shape test_gemm
sweep (tests/golden/gemm40.npz, produced by the unmodified reference)."""

import importlib.util
import os
import sys
import types
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STUB = os.path.join(ROOT, "integration", "bitnn", "gemm_b200.py")


def _load_stub(monkeypatch):
    from paper_1705_09864_b200 import _lib, gemm
    monkeypatch.setenv("BITNN_B200_LIB", _lib.LIB_PATH)
    pkg = types.ModuleType("bitnn")
    pkg.__path__ = [os.path.dirname(STUB)]
    monkeypatch.setitem(sys.modules, "bitnn", pkg)
    monkeypatch.setitem(sys.modules, "bitnn.gemm", gemm)
    spec = importlib.util.spec_from_file_location("bitnn.gemm_b200", STUB)
    mod = importlib.util.module_from_spec(spec)
    monkeypatch.setitem(sys.modules, "bitnn.gemm_b200", mod)
    spec.loader.exec_module(mod)
    return mod


def _bm(words, vectors, n_bits, layout, pad):
    return SimpleNamespace(words=words, vectors=vectors, n_bits=n_bits, layout=layout,
                           pad_fill=pad)


def test_stub_validates_like_the_reference(monkeypatch):
    """No GPU needed: bad operands raise the reference's ValueError before any call."""
    stub = _load_stub(monkeypatch)
    a = _bm(np.zeros((2, 1), np.uint64), 2, 10, "a", 0)
    with pytest.raises(ValueError, match="layouts"):
        stub.xnor_gemm_b200(a, _bm(np.zeros((1, 3), np.uint64), 3, 10, "a", 1))
    with pytest.raises(ValueError, match="complementary"):
        stub.xnor_gemm_b200(a, _bm(np.zeros((1, 3), np.uint64), 3, 10, "b", 0))
    with pytest.raises(ValueError, match="reduction lengths"):
        stub.xnor_gemm_b200(a, _bm(np.zeros((1, 3), np.uint64), 3, 11, "b", 1))


@pytest.mark.gpu
def test_stub_matches_reference_gemm40(monkeypatch, golden_dir):
    stub = _load_stub(monkeypatch)
    g = np.load(os.path.join(golden_dir, "gemm40.npz"))
    i = 0
    while f"a{i}" in g:
        m, n, k = (int(v) for v in g[f"dims{i}"])
        a = _bm(g[f"a{i}"], m, k, "a", 0)
        b = _bm(g[f"b{i}"], n, k, "b", 1)
        c = stub.xnor_gemm_b200(a, b)
        assert c.dtype == np.float32 and c.shape == (m, n)
        assert np.array_equal(c, g[f"c{i}"]), (m, n, k)
        i += 1
    assert i == 40
