"""Pin the CPU oracle to the reference's own golden vectors (CPU only).

The vectors were produced by the unmodified reference (``bitnn``) via
``tests/golden/gen_golden_vectors.py``; the frozen literals below are the
known answers of the reference's tests (cited per test).
"""

import hashlib
import json
import os

import numpy as np
import pytest

import workloads as wl
from oracle import oracle as orc


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_frozen_words():
    # test_bitpack.py:24-31: [+1,-1,+1,+1] -> 13; one-filled tail -> 0xFFFFFFFFFFFFFFF0 | 13
    v = np.array([[1.0, -1.0, 1.0, 1.0]], np.float32)
    assert orc.pack_rows(v, 0).tolist() == [[13]]
    assert orc.pack_rows(v, 1).tolist() == [[0xFFFFFFFFFFFFFFF0 | 13]]
    assert orc.pack_cols(v.T, 1).tolist() == [[0xFFFFFFFFFFFFFFF0 | 13]]


def test_binarize_convention():
    # test_bitpack.py:34-43
    x = np.array([-0.5, 0.0, -0.0, 2.0, -3.0], np.float32)
    assert orc.binarize(x).tolist() == [-1.0, 1.0, 1.0, 1.0, -1.0]
    for bad in (np.nan, np.inf, -np.inf):
        with pytest.raises(ValueError):
            orc.binarize(np.array([1.0, bad], np.float32))
        with pytest.raises(ValueError):
            orc.binarize_pack_rows(np.array([[1.0, bad]], np.float32))


def test_pack_rejects_non_sign_values():
    # test_bitpack.py:46-56
    with pytest.raises(ValueError):
        orc.pack_rows(np.array([[1.0, 0.0]], np.float32))
    with pytest.raises(ValueError):
        orc.pack_cols(np.zeros((3, 3), np.float32))


def test_eq2_frozen_example():
    # test_qmath.py:96-106: a=[+1,-1,+1], b=[+1,+1,-1] -> dot -1, p = 1
    a = np.array([[1.0, -1.0, 1.0]], np.float32)
    b = np.array([[1.0], [1.0], [-1.0]], np.float32)
    p = orc.xnor_gemm(orc.pack_rows(a, 0), orc.pack_cols(b, 1))
    assert p.tolist() == [[1]]
    assert orc.map_xnor_to_dot(p, 3).tolist() == [[-1.0]]
    assert orc.map_dot_to_xnor(-1.0, 3) == 1.0


def test_pack_cases_match_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "pack_cases.npz"))
    i = 0
    while f"x{i}" in g:
        x = g[f"x{i}"]
        assert np.array_equal(orc.binarize(x), g[f"signs{i}"])
        assert np.array_equal(orc.pack_rows(g[f"signs{i}"], 0), g[f"a{i}"])
        assert np.array_equal(orc.binarize_pack_rows(x, 0), g[f"a{i}"])
        assert np.array_equal(orc.pack_cols(np.ascontiguousarray(g[f"signs{i}"].T), 1), g[f"b{i}"])
        # layout 'b' words transposed == layout 'a' of the transpose,
        # except the tail fill
        k = x.shape[1]
        a1 = orc.pack_rows(g[f"signs{i}"], 1)
        assert np.array_equal(a1.T, g[f"b{i}"])
        orc.audit_padding(g[f"a{i}"], k, "a", 0)
        orc.audit_padding(g[f"b{i}"], k, "b", 1)
        i += 1
    assert i >= 5


def test_gemm40_matches_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "gemm40.npz"))
    for i, (m, n, k, seed) in enumerate(wl.gemm40_cases()):
        a, b = wl.make_operands(m, n, k, seed)
        aw, bw = orc.pack_rows(a, 0), orc.pack_cols(b, 1)
        assert np.array_equal(aw, g[f"a{i}"]) and np.array_equal(bw, g[f"b{i}"])
        for threads in (1, 3):
            c = orc.xnor_gemm(aw, bw, threads).astype(np.float32)
            assert np.array_equal(c, g[f"c{i}"]), (m, n, k)
        # row-row identity with both tails 0: P = K - sum popc(a ^ b)
        x = orc.xor_popc_rowrow(aw, orc.pack_rows(np.ascontiguousarray(b.T), 0))
        assert np.array_equal((k - x).astype(np.float32), g[f"c{i}"])


def test_sweep504_matches_reference(golden_dir):
    rows = json.load(open(os.path.join(golden_dir, "sweep504.json")))
    got = []
    for m, n, k, a, b in wl.sweep504():
        c = orc.xnor_gemm(orc.pack_rows(a, 0), orc.pack_cols(b, 1)).astype(np.float32)
        got.append([m, n, k, _sha(c), int(c.astype(np.int64).sum())])
    assert got == rows


def test_conv_cases_match_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "conv_cases.npz"))
    for i, case in enumerate(wl.CONV_CASES):
        x, w = wl.conv_case_inputs(case)
        y = orc.qconv_packed(x, w, case[7], case[8])
        assert np.array_equal(y, g[f"y{i}"]), case


def test_layers_match_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "layers.npz"))
    y = orc.qdense_packed(g["qdense_x"], g["qdense_w"])
    assert np.array_equal(y, g["qdense_y_packed"])
    assert np.array_equal(y, g["qdense_y_float"])
    assert np.array_equal(orc.binarize_pack_rows(g["qdense_w"], 0), g["qdense_words"])
    y = orc.qconv_packed(g["qconv_x"], g["qconv_w"])
    assert np.array_equal(y, g["qconv_y_packed"])
    assert np.array_equal(orc.quantize_signed(g["qact_x"], 1), g["qact_y1"])
    assert np.array_equal(orc.quantize_signed(g["qact_x"], 2), g["qact_y2"])


def test_qmath_matches_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "qmath.npz"))
    assert np.array_equal(orc.quantize(g["x"], 2), g["q2"])
    assert np.array_equal(orc.quantize_signed(g["xs"], 2), g["qs2"])
    assert np.array_equal(orc.quantize_signed(g["xs"], 1), g["qs1"])
    ca = orc.quantize_codes(g["x"], 2)
    cw = orc.quantize_codes(g["w"], 2)
    assert np.array_equal(ca.astype(np.float32) / np.float32(3), g["q2"])
    # exact-grid decode vs the reference's f32 grid values: 1/3 is rounded to
    # f32 there (rel 3e-8), far inside the 1e-5 multi-bit tolerance
    dot = (ca @ cw.T) / 9.0
    assert np.all(np.abs(dot - g["dot2"]) <= 1e-6 * np.maximum(1.0, np.abs(g["dot2"])))


def test_config1_config2_match_reference(golden_dir):
    cfg = json.load(open(os.path.join(golden_dir, "configs.json")))
    a, w = wl.config1_inputs()
    y = orc.qfc_dot(a, w)
    assert _sha(y) == cfg["c1"]["sha256"]
    x, wt = wl.config2_inputs()
    c = wl.C2
    y = orc.qconv_packed(x, wt, c["stride"], c["pad"])
    assert list(y.shape) == cfg["c2"]["shape"]
    assert _sha(y) == cfg["c2"]["sha256"]
