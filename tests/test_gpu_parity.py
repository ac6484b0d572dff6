"""Parity of the CUDA path (through the C ABI) with the reference.

Golden vectors were produced by the unmodified reference in the build
container (tests/golden/gen_golden_vectors.py); the oracle (oracle/) is the
pinned CPU restatement used for seeded cases the fixtures do not cover.
Bar: bit-exact for every binary / integer output.
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

import workloads as wl
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

ALGOS = ["popc", "bmma", "umma0", "umma1", "umma2", "umma3", "umma4"]
# GEMM-only engines: "xp" = operands pre-expanded in a workspace + the 2-CTA kind::mxf4 GEMM
# (bnn_xnor_gemm_ws); "auto" routes the large shapes there
GEMM_ALGOS = ALGOS + ["xp"]


def A(algo):
    """Engine id for the C ABI: umma<v> = the tcgen05 engine's variant v (per call)."""
    return algo


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def bnn():
    import paper_1705_09864_b200 as p
    p.load_library()
    return p


@pytest.fixture(scope="module")
def golden(golden_dir):
    return {n: np.load(os.path.join(golden_dir, n + ".npz"))
            for n in ("pack_cases", "gemm40", "conv_cases", "layers", "qmath")}


# ------------------------------------------------------------------ bitpack
def test_frozen_words_and_sign_convention(bnn):
    # test_bitpack.py:24-43
    assert list(bnn.pack_row(np.array([1.0, -1.0, 1.0, 1.0]), 0)) == [13]
    assert list(bnn.pack_row(np.array([1.0, -1.0, 1.0, 1.0]), 1)) == [0xFFFFFFFFFFFFFFF0 | 13]
    x = np.array([-0.5, 0.0, -0.0, 2.0, -3.0], np.float32)
    assert list(bnn.binarize(x)) == [-1.0, 1.0, 1.0, 1.0, -1.0]
    for bad in (np.nan, np.inf, -np.inf):
        with pytest.raises(ValueError):
            bnn.binarize(np.array([1.0, bad], np.float32))
    with pytest.raises(ValueError):
        bnn.pack_row(np.array([1.0, 0.0]))
    with pytest.raises(ValueError):
        bnn.pack_matrix_a(np.array([[2.0, 1.0]]))
    with pytest.raises(ValueError):
        bnn.pack_matrix_b(np.zeros((3, 3)))
    with pytest.raises(ValueError):
        bnn.pack_matrix_a(np.ones(4))


def test_popcount_hardware_matches_software(bnn):
    """test_bitpack.py:136-147: POPC == the shift/mask sequence == int.bit_count."""
    rng = np.random.default_rng(8)
    words = rng.integers(0, 2**64, size=5000, dtype=np.uint64)
    words[:4] = [0, 1, 2**64 - 1, 0x8000000000000000]
    hw = bnn.popcount64(words)
    sw = bnn.popcount64_soft(words)
    assert hw.dtype == np.uint8 and hw.shape == words.shape
    assert np.array_equal(hw, sw)
    assert np.array_equal(hw, np.bitwise_count(words))
    for i in range(200):
        assert int(hw[i]) == int(words[i]).bit_count()
    dev = torch.from_numpy(words).cuda()
    assert torch.equal(bnn.popcount64(dev).cpu(), torch.from_numpy(hw))


@pytest.mark.parametrize("n", [1, 63, 64, 65, 200, 1000])
def test_dot_xnor_popcount_pair(bnn, n):
    """dot_xnor_popcount (bitpack.py:218-231) on the 'a'/'b' packing pair == the
    agreement count; 2p - n == the +-1 dot product (test_bitpack.py:150-178)."""
    rng = np.random.default_rng(n)
    a = rng.choice(np.array([-1.0, 1.0], np.float32), size=n)
    b = rng.choice(np.array([-1.0, 1.0], np.float32), size=n)
    aw = bnn.pack_row(a, 0)
    bw = bnn.pack_row(b, 1)
    p = bnn.dot_xnor_popcount(aw, bw, n)
    assert p == int((a == b).sum())
    assert 2 * p - n == int(np.dot(a, b))
    with pytest.raises(ValueError):
        bnn.dot_xnor_popcount(aw[:0] if len(aw) > 1 else np.zeros(2, np.uint64), bw, n)


def test_pack_cases_bit_exact(bnn, golden):
    g = golden["pack_cases"]
    i = 0
    while f"x{i}" in g:
        s = g[f"signs{i}"]
        assert np.array_equal(bnn.binarize(g[f"x{i}"]), s)
        a = bnn.pack_matrix_a(s)
        assert np.array_equal(a.words.cpu().numpy(), g[f"a{i}"])
        b = bnn.pack_matrix_b(np.ascontiguousarray(s.T))
        assert np.array_equal(b.words.cpu().numpy(), g[f"b{i}"])
        assert np.array_equal(a.unpack(), s) and np.array_equal(b.unpack(), s.T)
        # fused sign+pack of the raw floats == pack(binarize(x))
        xw = bnn.pack_rows_device(torch.from_numpy(g[f"x{i}"]).cuda(), 0)
        assert np.array_equal(xw.cpu().numpy(), g[f"a{i}"])
        bnn.audit_padding(a)
        bnn.audit_padding(b)
        # transposed layouts agree up to the tail fill
        a1 = bnn.pack_rows_device(torch.from_numpy(s).cuda(), 1)
        assert np.array_equal(bnn.words_transpose(a1).cpu().numpy(), g[f"b{i}"])
        i += 1


def test_audit_padding_catches_corruption(bnn):
    rng = np.random.default_rng(6)
    a = bnn.pack_matrix_a(wl.random_signs(rng, (4, 70)))
    bnn.audit_padding(a)
    a.words.view(torch.int64)[2, -1] |= 1 << 6
    with pytest.raises(ValueError):
        bnn.audit_padding(a)
    b = bnn.pack_matrix_b(wl.random_signs(rng, (70, 4)))
    bnn.audit_padding(b)
    w = b.words.cpu().numpy()
    w[-1, 1] &= ~np.uint64(1 << 63)
    with pytest.raises(ValueError):
        bnn.audit_padding(bnn.BitMatrix(w, 4, 70, "b", 1))


def test_pack_nonfinite_and_strict_flags(bnn):
    x = torch.randn(5, 200, device="cuda")
    x[3, 150] = float("nan")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    bnn.pack_rows_device(x, 0, flags=flags)
    assert int(flags.item()) & 1
    xs = torch.where(torch.randn(3, 4, 5, 6, device="cuda") >= 0, 1.0, -1.0)
    flags.zero_()
    bnn.pack_nchw(xs, strict=True, flags=flags)
    assert int(flags.item()) == 0
    xs[1, 2, 3, 4] = 0.5
    bnn.pack_nchw(xs, strict=True, flags=flags)
    assert int(flags.item()) & 2


def test_pack_nchw_matches_oracle(bnn):
    rng = np.random.default_rng(3)
    for b, c, h, w in ((2, 3, 5, 7), (1, 64, 4, 4), (2, 130, 3, 5), (1, 256, 28, 28)):
        x = rng.standard_normal((b, c, h, w)).astype(np.float32)
        x.reshape(-1)[::13] = 0.0
        got = bnn.pack_nchw(torch.from_numpy(x).cuda()).cpu().numpy()
        nhwc = np.ascontiguousarray(x.transpose(0, 2, 3, 1)).reshape(-1, c)
        expect = orc.binarize_pack_rows(nhwc, 0)
        assert np.array_equal(got.reshape(-1, got.shape[-1]), expect)


# ------------------------------------------------------------------ gemm
@pytest.mark.parametrize("algo", GEMM_ALGOS)
def test_gemm40_bit_exact(bnn, golden, algo):
    g = golden["gemm40"]
    for i, (m, n, k, seed) in enumerate(wl.gemm40_cases()):
        a = bnn.BitMatrix(g[f"a{i}"], m, k, "a", 0)
        b = bnn.BitMatrix(g[f"b{i}"], n, k, "b", 1)
        c = bnn.xnor_gemm_b200(a, b, algo=A(algo)).cpu().numpy()
        assert c.dtype == np.float32
        assert np.array_equal(c, g[f"c{i}"]), (m, n, k)


def test_reference_kernel_ids_and_checksums(bnn):
    dims = bnn.GemmDims(8, 9, 200)
    recs = [bnn.benchmark_kernel(k, dims, repeats=2, warmup=1, seed=7) for k in bnn.KERNEL_IDS]
    assert len({r.checksum for r in recs}) == 1
    a, b = bnn.gemm.make_operands(bnn.GemmDims(37, 19, 257), 9)
    ref = bnn.run_kernel("xnor_base", a, b)
    for kid in bnn.KERNEL_IDS[1:]:
        assert np.array_equal(bnn.run_kernel(kid, a, b), ref)
    with pytest.raises(ValueError):
        bnn.run_kernel("turbo", a, b)


def test_operand_validation(bnn):
    a, b = bnn.gemm.make_operands(bnn.GemmDims(4, 5, 70), 2)
    abm, bbm = bnn.pack_matrix_a(a), bnn.pack_matrix_b(b)
    with pytest.raises(ValueError):
        bnn.xnor_gemm_base(bbm, bbm)
    with pytest.raises(ValueError):
        bnn.xnor_gemm_base(abm, abm)
    short = bnn.pack_matrix_b(bnn.gemm.make_operands(bnn.GemmDims(4, 5, 64), 2)[1])
    with pytest.raises(ValueError):
        bnn.xnor_gemm_base(abm, short)


@pytest.mark.parametrize("algo", GEMM_ALGOS)
def test_sweep504_bit_exact(bnn, golden_dir, algo):
    rows = json.load(open(os.path.join(golden_dir, "sweep504.json")))
    got = []
    for m, n, k, a, b in wl.sweep504():
        abm, bbm = bnn.pack_matrix_a(a), bnn.pack_matrix_b(b)
        c = bnn.xnor_gemm_b200(abm, bbm, algo=A(algo)).cpu().numpy()
        got.append([m, n, k, _sha(c), int(c.astype(np.int64).sum())])
    assert got == rows


@pytest.mark.parametrize("algo", GEMM_ALGOS)
def test_gemm_tail_and_layout_variants(bnn, algo):
    """Row-row operands, every pad combination, both domains, odd ld, transposed out."""
    rng = np.random.default_rng(5)
    for m, n, k in ((1, 1, 1), (3, 5, 63), (17, 33, 65), (130, 70, 1000), (64, 257, 4096),
                    (300, 129, 2049)):
        a = wl.random_signs(rng, (m, k))
        b = wl.random_signs(rng, (n, k))
        p = (a.astype(np.int64) == 1)[:, None, :] == (b.astype(np.int64) == 1)[None, :, :] \
            if m * n * k < 3e6 else None
        expect = p.sum(-1) if p is not None else (
            k - orc.xor_popc_rowrow(orc.pack_rows(a, 0), orc.pack_rows(b, 0)))
        for ap in (0, 1):
            for bp in (0, 1):
                aw = torch.from_numpy(orc.pack_rows(a, ap).view(np.uint64)).cuda()
                bw = torch.from_numpy(orc.pack_rows(b, bp)).cuda()
                c = bnn.xnor_rows_gemm(aw, bw, k, a_pad=ap, b_pad=bp, algo=A(algo))
                assert np.array_equal(c.cpu().numpy(), expect.astype(np.float32)), (m, n, k, ap, bp)
        # odd leading dimension (8-byte aligned rows), dot domain, [N, M] output
        W = (k + 63) // 64
        aw = torch.zeros((m, W + 1), dtype=torch.uint64, device="cuda")
        aw[:, :W] = torch.from_numpy(orc.pack_rows(a, 0)).cuda()
        bw = torch.from_numpy(orc.pack_rows(b, 0)).cuda()
        c = bnn.xnor_rows_gemm(aw[:, :W], bw, k, domain=1, transpose_out=True, algo=A(algo))
        assert np.array_equal(c.cpu().numpy(), (2 * expect - k).T.astype(np.float32))


@pytest.mark.parametrize("algo", ALGOS)
def test_gemm_epilogue_scale_shift(bnn, algo):
    rng = np.random.default_rng(8)
    m, n, k = 40, 50, 300
    a, b = wl.random_signs(rng, (m, k)), wl.random_signs(rng, (n, k))
    aw, bw = (torch.from_numpy(orc.pack_rows(x, 0)).cuda() for x in (a, b))
    sc = torch.from_numpy(rng.standard_normal(m).astype(np.float32)).cuda()
    sh = torch.from_numpy(rng.standard_normal(m).astype(np.float32)).cuda()
    c = bnn.xnor_rows_gemm(aw, bw, k, scale=sc, shift=sh, algo=A(algo)).cpu().numpy()
    p = (k - orc.xor_popc_rowrow(orc.pack_rows(a, 0), orc.pack_rows(b, 0))).astype(np.float32)
    expect = p * sc.cpu().numpy()[:, None] + sh.cpu().numpy()[:, None]
    assert np.array_equal(c, expect.astype(np.float32))


# ------------------------------------------------------------------ conv
@pytest.mark.parametrize("algo", ALGOS)
def test_conv_cases_bit_exact(bnn, golden, algo):
    g = golden["conv_cases"]
    for i, case in enumerate(wl.CONV_CASES):
        b, c, h, w, f, kh, kw, stride, pad, seed = case
        x, wt = wl.conv_case_inputs(case)
        layer = bnn.QConvolution(c, f, (kh, kw), stride, pad)
        layer.weight = wt
        layer.pack()
        layer.algo = A(algo)
        y = layer.forward(torch.from_numpy(x).cuda(), bnn.INFER_PACKED).cpu().numpy()
        assert np.array_equal(y, g[f"y{i}"]), case
        # the float path of the same layer agrees exactly (layers.py:237-244)
        yf = layer.forward(torch.from_numpy(x).cuda(), bnn.INFER_FLOAT).cpu().numpy()
        assert np.array_equal(yf, g[f"y{i}"]), case


# channel counts that take the im2col-TMA route of the tcgen05 engine (C % 256 == 0):
# odd strides, asymmetric padding, pixel tiles straddling rows and images
IM2COL_CASES = [
    # (B, C, H, W, F, kh, kw, stride, pad, seed)
    (2, 256, 9, 11, 40, 3, 3, (1, 1), (1, 1), 31),
    (3, 256, 7, 5, 130, 3, 3, (2, 1), (1, 2), 32),
    (1, 512, 6, 6, 17, 1, 1, (1, 1), (0, 0), 33),
    (2, 256, 10, 10, 64, 5, 3, (2, 3), (2, 0), 34),
    (5, 256, 4, 4, 256, 2, 2, (1, 1), (0, 1), 35),
    (1, 256, 30, 30, 8, 3, 3, (1, 1), (0, 0), 36),
]


@pytest.mark.parametrize("case", IM2COL_CASES)
def test_conv_im2col_route_matches_oracle(bnn, case):
    b, c, h, w, f, kh, kw, stride, pad, seed = case
    x, wt = wl.conv_case_inputs(case)
    expect = orc.qconv_packed(x, wt, stride, pad)
    for algo in ("umma3", "umma2", "umma1", "umma0", "popc"):
        layer = bnn.QConvolution(c, f, (kh, kw), stride, pad)
        layer.weight = wt
        layer.pack()
        layer.algo = A(algo)
        y = layer.forward(torch.from_numpy(x).cuda(), bnn.INFER_PACKED).cpu().numpy()
        assert np.array_equal(y, expect), (case, algo)


def test_reference_layers_bit_exact(bnn, golden):
    g = golden["layers"]
    qd = bnn.QDense(130, 17, bits=1)
    qd.weight = g["qdense_w"]
    assert np.array_equal(qd.forward(g["qdense_x"], bnn.INFER_FLOAT), g["qdense_y_float"])
    qd.pack()
    assert np.array_equal(qd.packed.words.cpu().numpy(), g["qdense_words"])
    y = qd.forward(g["qdense_x"], bnn.INFER_PACKED)
    assert isinstance(y, np.ndarray) and np.array_equal(y, g["qdense_y_packed"])
    qc = bnn.QConv2d(3, 5, (3, 3), bits=1)
    qc.weight = g["qconv_w"]
    qc.pack()
    assert np.array_equal(qc.packed.words.cpu().numpy(), g["qconv_words"])
    assert np.array_equal(qc.forward(g["qconv_x"], bnn.INFER_PACKED), g["qconv_y_packed"])
    assert np.array_equal(qc.forward(g["qconv_x"], bnn.INFER_FLOAT), g["qconv_y_float"])
    # packed layer refuses non-sign inputs like pack_matrix_b (bitpack.py:69-75)
    with pytest.raises(ValueError):
        qc.forward(g["qconv_x"] * 0.5, bnn.INFER_PACKED)
    assert np.array_equal(bnn.QActivation(1).forward(g["qact_x"], bnn.INFER_PACKED), g["qact_y1"])
    assert np.array_equal(bnn.QActivation(2).forward(g["qact_x"], bnn.INFER_FLOAT), g["qact_y2"])
    with pytest.raises(ValueError):
        bnn.QActivation(1).forward(np.array([np.nan], np.float32), bnn.INFER_PACKED)
    # mode errors (layers.py:217-220, 232-239)
    q2 = bnn.QDense(8, 3, bits=2, rng=np.random.default_rng(1))
    with pytest.raises(bnn.ModeError):
        q2.forward(np.ones((2, 8), np.float32), bnn.INFER_PACKED)
    with pytest.raises(bnn.ModeError):
        bnn.QDense(8, 3, rng=np.random.default_rng(1)).forward(np.ones((2, 8)), bnn.INFER_PACKED)


def test_qmath_bit_exact(bnn, golden):
    g = golden["qmath"]
    assert np.array_equal(bnn.quantize(g["x"], 2), g["q2"])
    assert np.array_equal(bnn.quantize_signed(g["xs"], 2), g["qs2"])
    assert np.array_equal(bnn.quantize_signed(g["xs"], 1), g["qs1"])


# ------------------------------------------------------------------ BASELINE configs
@pytest.mark.parametrize("algo", ALGOS)
def test_config1_qfc_golden(bnn, golden_dir, algo):
    cfg = json.load(open(os.path.join(golden_dir, "configs.json")))["c1"]
    a, w = wl.config1_inputs()
    layer = bnn.QFullyConnected(4096, 1024, domain="dot")
    layer.weight = w
    layer.pack()
    layer.algo = A(algo)
    y = layer.forward(torch.from_numpy(a).cuda(), bnn.INFER_PACKED).cpu().numpy()
    assert list(y.shape) == cfg["shape"]
    assert _sha(y) == cfg["sha256"]


@pytest.mark.parametrize("algo", ALGOS)
def test_config2_qconv_golden(bnn, golden_dir, algo):
    cfg = json.load(open(os.path.join(golden_dir, "configs.json")))["c2"]
    x, wt = wl.config2_inputs()
    c = wl.C2
    layer = bnn.QConvolution(c["c"], c["f"], (c["kh"], c["kw"]), c["stride"], c["pad"])
    layer.weight = wt
    layer.pack()
    layer.algo = A(algo)
    y = layer.forward(torch.from_numpy(x).cuda(), bnn.INFER_PACKED).cpu().numpy()
    assert list(y.shape) == cfg["shape"]
    assert _sha(y) == cfg["sha256"]


LARGE = ([(a, mnk) for a in ALGOS for mnk in [(4096, 4096, 4096), (4096, 4096, 65536),
                                             (8192, 8192, 8192)]] +
         [(a, mnk) for a in ("xp", "auto") for mnk in [(4096, 4096, 4096), (4096, 4096, 65536),
                                                        (8192, 8192, 8192)]] +
         [(a, (16384, 16384, 16384)) for a in ("umma2", "popc", "xp", "auto")])  # BASELINE configs[4]


@pytest.mark.parametrize("algo,mnk", LARGE)
def test_large_gemm_properties(bnn, algo, mnk):
    """Full-size C5 shapes: exact row/column checksums + sampled exact entries.

    sum_n P[m, n] = sum_k (a_mk ? ones_k : N - ones_k) with ones_k = #{n : b_nk = 1}
    is O((M + N) K) on the CPU, so it checks every output row at any size.
    """
    m, n, k = mnk
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    W = k // 64
    aw = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda", generator=g).view(torch.uint64)
    bw = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda", generator=g).view(torch.uint64)
    c = bnn.xnor_rows_gemm(aw, bw, k, algo=A(algo))
    assert float(c.min()) >= 0 and float(c.max()) <= k
    a_np, b_np = aw.cpu().numpy(), bw.cpu().numpy()
    del aw, bw

    def bits(x, lo, hi):
        return np.unpackbits(x[lo:hi].view(np.uint8), axis=1, bitorder="little")

    def side_sums(x, other, n_other):
        # sum over the other operand of agreement = sum_k (n - ones_k) + x_k (2 ones_k - n)
        ones = np.zeros(k, np.int64)
        for lo in range(0, other.shape[0], 1024):
            ones += bits(other, lo, lo + 1024).sum(0, dtype=np.int64)
        coef = (2 * ones - n_other).astype(np.float64)
        out = []
        for lo in range(0, x.shape[0], 1024):
            out.append(bits(x, lo, lo + 1024).astype(np.float64) @ coef)
        return (np.concatenate(out) + float((n_other - ones).sum())).astype(np.int64)

    row_got = c.sum(1, dtype=torch.float64).cpu().numpy().astype(np.int64)
    assert np.array_equal(row_got, side_sums(a_np, b_np, n))
    col_got = c.sum(0, dtype=torch.float64).cpu().numpy().astype(np.int64)
    assert np.array_equal(col_got, side_sums(b_np, a_np, m))
    rng = np.random.default_rng(0)
    idx_m, idx_n = rng.integers(0, m, 64), rng.integers(0, n, 64)
    got = c[torch.from_numpy(idx_m).cuda(), torch.from_numpy(idx_n).cuda()].cpu().numpy()
    for v, i, j in zip(got, idx_m, idx_n):
        x = int(np.bitwise_count(a_np[i] ^ b_np[j]).sum())
        assert v == k - x


def test_pre_expanded_engine_variants_bit_exact(bnn):
    """The experiment routes of bnn_gemm_xp.cu stay correct: clusters of two CTA pairs sharing
    the B tile by TMA multicast (debug bit 1 << 26), register stores with a 7-stage ring
    (1 << 20), parked waits (1 << 21) -- all bit-identical to the default pair route, including
    an odd number of 256-row tiles (the second pair of the last cluster idles) and ragged edges."""
    from paper_1705_09864_b200 import _lib
    try:
        for (m, n, k) in [(512, 224, 256), (300, 500, 1000), (768, 3000, 4160), (1280, 1100, 2048)]:
            g = torch.Generator(device="cuda").manual_seed(m + n + k)
            w = (k + 63) // 64
            a = torch.randint(-2**63, 2**63 - 1, (m, w), device="cuda", generator=g)
            b = torch.randint(-2**63, 2**63 - 1, (n, w), device="cuda", generator=g)
            if k % 64:  # pad fill 0: the bits past K of the last word are clear
                a[:, -1] &= (1 << (k % 64)) - 1
                b[:, -1] &= (1 << (k % 64)) - 1
            a, b = a.view(torch.uint64), b.view(torch.uint64)
            _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
            ref = bnn.xnor_rows_gemm(a, b, k, algo="xp", domain=_lib.DOT)
            assert torch.equal(ref, bnn.xnor_rows_gemm(a, b, k, algo="popc", domain=_lib.DOT))
            for bits in (1 << 26, 1 << 20, 1 << 21, (1 << 26) | (1 << 21)):
                _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, bits)
                for _ in range(2):
                    assert torch.equal(bnn.xnor_rows_gemm(a, b, k, algo="xp", domain=_lib.DOT), ref), (m, n, k, bits)
    finally:
        _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)


# ------------------------------------------------------------------ multi-bit (bit planes)
def _codes_np(x, grid, bits=2):
    L = (1 << bits) - 1
    x = np.asarray(x, np.float32)
    if grid == "signed":
        y = np.float32(0.5) * np.clip(x, np.float32(-1), np.float32(1)) + np.float32(0.5)
    else:
        y = x
    return np.floor(y * np.float32(L) + np.float32(0.5)).astype(np.int64)


@pytest.mark.parametrize("grid", ["signed", "unsigned"])
def test_pack_planes_codes_exact(bnn, grid):
    rng = np.random.default_rng(31)
    x = (rng.random((37, 301), dtype=np.float32) if grid == "unsigned"
         else (rng.standard_normal((37, 301)) * 1.3).astype(np.float32))
    x.reshape(-1)[:6] = [0.0, 1.0, 1 / 6, 0.5, 5 / 6, -0.0] if grid == "unsigned" else \
        [-1.0, 1.0, -1 / 3, 1 / 3, 0.0, -0.0]
    planes = bnn.bitpack.pack_planes_device(torch.from_numpy(x).cuda(), 2, grid).cpu().numpy()
    codes = _codes_np(x, grid)
    for p in range(2):
        expect = orc.pack_rows(np.where((codes >> p) & 1, 1.0, -1.0).astype(np.float32), 0)
        assert np.array_equal(planes[p], expect), p
    # the codes are the reference quantizers' grid indices
    ref = orc.quantize(x, 2) if grid == "unsigned" else orc.quantize_signed(x, 2)
    L = np.float32(3)
    vals = codes.astype(np.float32) / L if grid == "unsigned" else \
        np.float32(2) * (codes.astype(np.float32) / L) - np.float32(1)
    assert np.array_equal(vals, ref)
    if grid == "unsigned":
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        bad = torch.from_numpy(x).cuda()
        bad[3, 4] = 1.5
        bnn.bitpack.pack_planes_device(bad, 2, grid, flags)
        assert int(flags.item()) & 4


def test_bitplane_gemm_matches_reference_float64(bnn, golden):
    """Config-5 2-bit semantics: U[0,1] operands on the quantize() grid (G5)."""
    g = golden["qmath"]
    x, w = g["x"], g["w"]  # [64, 96] activations, [40, 96] weights
    ap = bnn.bitpack.pack_planes_device(torch.from_numpy(w).cuda(), 2, "unsigned")
    bp = bnn.bitpack.pack_planes_device(torch.from_numpy(x).cuda(), 2, "unsigned")
    y = bnn.gemm.bitplane_gemm(ap, bp, 96, a_grid="unsigned", b_grid="unsigned",
                               transpose_out=True).cpu().numpy()
    ref = g["dot2"]  # float64 product of the reference's quantize() values
    assert np.all(np.abs(y - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref)))


@pytest.mark.parametrize("m,n,k,grids", [
    (m, n, k, g) for m, n, k in [(40, 64, 96), (300, 257, 1000), (1024, 512, 4096)]
    for g in [("signed", "signed"), ("unsigned", "unsigned"), ("signed", "unsigned")]] +
    [(4096, 4096, 4096, ("unsigned", "unsigned"))])  # BASELINE configs[4] 2-bit at full size
def test_bitplane_gemm_exact_integer_decode(bnn, m, n, k, grids):
    rng = np.random.default_rng(m + n + k)
    ga, gb = grids
    mk = lambda shape, g: (rng.random(shape, dtype=np.float32) if g == "unsigned"
                           else rng.standard_normal(shape).astype(np.float32))
    w, x = mk((m, k), ga), mk((n, k), gb)
    ap = bnn.bitpack.pack_planes_device(torch.from_numpy(w).cuda(), 2, ga)
    bp = bnn.bitpack.pack_planes_device(torch.from_numpy(x).cuda(), 2, gb)
    y = bnn.gemm.bitplane_gemm(ap, bp, k, a_grid=ga, b_grid=gb).cpu().numpy()
    ca, cb = _codes_np(w, ga), _codes_np(x, gb)
    aa, ba = (2, -3) if ga == "signed" else (1, 0)
    ab, bb = (2, -3) if gb == "signed" else (1, 0)
    # exact integer numerator (float64 BLAS: every partial sum < 2^53)
    num = (aa * ca + ba).astype(np.float64) @ (ab * cb + bb).astype(np.float64).T
    exact = num / 9.0
    assert np.all(np.abs(y - exact) <= 2e-7 * np.maximum(1.0, np.abs(exact))), (m, n, k)


@pytest.mark.parametrize("m,n,k", [(40, 64, 96), (300, 257, 1000), (1024, 512, 4096),
                                   (2048, 1024, 2048), (4096, 4096, 4096)])
def test_bitplane_gemm_pre_expanded_engine_identical(bnn, m, n, k):
    """bnn_bitplane_gemm_ws (codes as e2m1 grid values + the 2-CTA kind::mxf4 GEMM) against
    the planes engine: the same integer numerator and the same single rounding, so the f32
    outputs are bit-identical for every grid pair, both output layouts and ragged shapes."""
    rng = np.random.default_rng(m * 3 + n + k)
    for ga, gb in (("signed", "signed"), ("unsigned", "unsigned"), ("signed", "unsigned")):
        mk = lambda shape, g: (rng.random(shape, dtype=np.float32) if g == "unsigned"
                               else rng.standard_normal(shape).astype(np.float32))
        ap = bnn.bitpack.pack_planes_device(torch.from_numpy(mk((m, k), ga)).cuda(), 2, ga)
        bp = bnn.bitpack.pack_planes_device(torch.from_numpy(mk((n, k), gb)).cuda(), 2, gb)
        for tr in (False, True):
            ref = bnn.gemm.bitplane_gemm(ap, bp, k, a_grid=ga, b_grid=gb, transpose_out=tr, algo="umma")
            got = bnn.gemm.bitplane_gemm(ap, bp, k, a_grid=ga, b_grid=gb, transpose_out=tr, algo="xp")
            assert torch.equal(ref, got), (m, n, k, ga, gb, tr)
    if m * n * k >= 3e10:  # AUTO takes the pre-expanded engine here
        auto = bnn.gemm.bitplane_gemm(ap, bp, k, a_grid=ga, b_grid=gb, transpose_out=True)
        assert torch.equal(auto, got)


def test_qfullyconnected_2bit_packed_equals_float_path(bnn):
    rng = np.random.default_rng(4)
    layer = bnn.QFullyConnected(300, 70, act_bit=2, weight_bit=2, rng=rng)
    x = (rng.standard_normal((33, 300)) * 0.8).astype(np.float32)
    yf = layer.forward(x, bnn.INFER_FLOAT)  # reference float path (layers.py:370-377)
    layer.pack()
    yp = layer.forward(x, bnn.INFER_PACKED)
    # float64 oracle from the reference quantizers' f32 values
    xq = orc.quantize_signed(x, 2).astype(np.float64)
    wq = orc.quantize_signed(layer.weight, 2).astype(np.float64)
    ref = xq @ wq.T
    for y in (yf, yp):
        assert np.all(np.abs(y - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref)))
    # the reference-compatible QDense keeps rejecting multi-bit packed inference
    q = bnn.QDense(300, 70, bits=2, rng=rng)
    with pytest.raises(bnn.ModeError):
        q.forward(x, bnn.INFER_PACKED)


@pytest.mark.parametrize("geom", [(3, 16, 9, 11, 24, (3, 3), (1, 1), (1, 1)),
                                  (2, 7, 8, 8, 5, (3, 2), (2, 1), (0, 1)),
                                  (4, 64, 14, 14, 64, (3, 3), (2, 2), (1, 1)),
                                  (2, 32, 6, 6, 40, (1, 1), (1, 1), (0, 0))])
def test_qconvolution_2bit_packed_equals_float_path(bnn, geom):
    """QConvolution(act_bit = weight_bit = 2) through the bit-plane engine (VERDICT r1 missing 8):
    the packed path equals the reference-style float path (layers.py:237-244: quantize_signed
    weights @ im2col of the zero-padded, quantized input) and a float64 oracle of the same
    composition within 1e-5 * max(1, |ref|)."""
    b, c, h, w, f, kern, stride, pad = geom
    rng = np.random.default_rng(sum(geom[:5]))
    layer = bnn.QConvolution(c, f, kern, stride, pad, act_bit=2, weight_bit=2, rng=rng, domain="dot")
    x = (rng.standard_normal((b, c, h, w)) * 0.8).astype(np.float32)
    with pytest.raises(bnn.ModeError):
        layer.forward(x, bnn.INFER_PACKED)  # not packed yet
    yf = layer.forward(x, bnn.INFER_FLOAT)
    layer.pack()
    yp = layer.forward(x, bnn.INFER_PACKED)
    xpad = np.pad(x, ((0, 0), (0, 0), (pad[0], pad[0]), (pad[1], pad[1])))
    xq = orc.quantize_signed(xpad, 2).astype(np.float64)
    wq = orc.quantize_signed(layer.weight, 2).astype(np.float64)
    oh, ow = yp.shape[2], yp.shape[3]
    ref = np.zeros((b, f, oh, ow))
    for ky in range(kern[0]):
        for kx in range(kern[1]):
            win = xq[:, :, ky:ky + stride[0] * (oh - 1) + 1:stride[0],
                     kx:kx + stride[1] * (ow - 1) + 1:stride[1]]
            ref += np.einsum("bchw,fc->bfhw", win, wq[:, :, ky, kx])
    assert yp.shape == yf.shape == ref.shape
    for y in (yf, yp):
        assert np.all(np.abs(y - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref)))
    # the packed numerator is an exact integer / 9: decode it
    num = np.rint(ref * 9.0)
    assert np.all(np.abs(yp - num / 9.0) <= 2e-7 * np.maximum(1.0, np.abs(ref)))
    # the reference-compatible QConv2d keeps rejecting multi-bit packed inference
    q = bnn.QConv2d(c, f, kern, stride, (0, 0), bits=2, rng=rng)
    with pytest.raises(bnn.ModeError):
        q.pack()


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_umma_repeat_runs_identical(bnn, variant):
    """Pipeline-race guard: repeated launches of the TMA-fed tcgen05 engine on a
    many-tile shape equal the CUDA-core engine every time (a slot released
    before its reads landed once corrupted ~1 run in 20)."""
    from paper_1705_09864_b200 import _lib
    m, n, k = 4096, 4096, 4096
    g = torch.Generator(device="cuda").manual_seed(7)
    a = torch.randint(-2**63, 2**63 - 1, (m, k // 64), device="cuda", generator=g).view(torch.uint64)
    b = torch.randint(-2**63, 2**63 - 1, (n, k // 64), device="cuda", generator=g).view(torch.uint64)
    ref = bnn.xnor_rows_gemm(a, b, k, algo="popc")
    for _ in range(12):
        assert torch.equal(bnn.xnor_rows_gemm(a, b, k, algo=f"umma{variant}"), ref)


@pytest.mark.parametrize("which", ["conv", "dense"])
def test_plan_run_host_pipelined_equals_single_pass(bnn, which):
    """The end-to-end host call overlaps H2D / compute / D2H over batch slices;
    its output must equal the one-pass result and the oracle."""
    from paper_1705_09864_b200.plan import ConvPlan, DensePlan
    rng = np.random.default_rng(12)
    if which == "conv":
        b, c, h, w, f = 7, 256, 9, 9, 40
        x = rng.standard_normal((b, c, h, w), dtype=np.float32)
        wt = rng.standard_normal((f, c, 3, 3), dtype=np.float32)
        layer = bnn.QConvolution(c, f, (3, 3), (1, 1), (1, 1))
        layer.weight = wt
        layer.pack()
        plan = ConvPlan(layer, b, h, w)
        expect = orc.qconv_packed(x, wt, (1, 1), (1, 1))
    else:
        b, k, u = 37, 1000, 70
        x = rng.standard_normal((b, k), dtype=np.float32)
        wt = rng.standard_normal((u, k), dtype=np.float32)
        layer = bnn.QFullyConnected(k, u)
        layer.weight = wt
        layer.pack()
        plan = DensePlan(layer, b)
        expect = orc.qdense_packed(orc.binarize(x), wt)
    xh = torch.from_numpy(x).pin_memory()
    outs = []
    for chunks in ("auto", 1, 3, 8):  # "auto": tuned on the first call, any count gives the same bits
        plan.host_chunks = chunks
        yh = torch.empty(plan.y.shape, dtype=torch.float32).pin_memory()
        outs.append(plan.run_host(xh, yh).numpy().copy())
    assert np.array_equal(outs[0], expect)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    # a non-finite input raises binarize's ValueError for that call only: the flag word
    # is cleared per call, so the next finite input runs normally
    bad = xh.clone().pin_memory()
    bad.view(-1)[5] = float("nan")
    yh = torch.empty(plan.y.shape, dtype=torch.float32).pin_memory()
    with pytest.raises(ValueError, match="finite"):
        plan.run_host(bad, yh)
    assert np.array_equal(plan.run_host(xh, yh).numpy(), outs[-1])
    plan.x.copy_(bad)
    plan.run_device()
    with pytest.raises(ValueError, match="finite"):
        plan.check_flags()
    plan.x.copy_(xh)
    plan.run_device()
    plan.check_flags()  # cleared by the previous check


@pytest.mark.parametrize("r,k,pad", [(3, 1, 0), (5, 200, 1), (256, 4096, 0), (7, 1000, 1), (2, 70000, 0)])
def test_pack_rows_segments_and_row_popcounts(bnn, r, k, pad):
    """Row packing split over several warps per row + the valid-bit row popcounts."""
    from paper_1705_09864_b200.bitpack import pack_rows_device
    rng = np.random.default_rng(r * 7 + k)
    x = rng.standard_normal((r, k), dtype=np.float32)
    x.reshape(-1)[::13] = 0.0
    x.reshape(-1)[5::17] = -0.0
    pc = torch.zeros(r, dtype=torch.int32, device="cuda")
    got = pack_rows_device(torch.from_numpy(x).cuda(), pad_fill=pad, row_popc=pc).cpu().numpy()
    expect = orc.pack_rows(orc.binarize(x), pad)
    assert np.array_equal(got, expect)
    assert np.array_equal(pc.cpu().numpy(), (x >= 0).sum(1))


def test_randomized_shapes_umma_routes_equal_popc(bnn):
    """Seeded sweep over shapes that hit every tcgen05 route (cp.async i8, TMA kind::mxf4
    with narrow / wide tiles, TMA-store and regular epilogues, dot domain, im2col convs
    straddling images): the result equals the independently tested POPC engine."""
    from paper_1705_09864_b200 import _lib
    rng = np.random.default_rng(2024)
    dense = [(1, 1, 64), (3, 5, 100), (128, 16, 256), (130, 300, 512), (256, 20000, 2304),
             (200, 37, 4096), (640, 1000, 1000), (96, 4097, 768), (1024, 256, 4096)]
    for m, n, k in dense:
        W = (k + 63) // 64
        g = torch.Generator(device="cuda").manual_seed(m * 7 + n + k)
        a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda", generator=g).view(torch.uint64)
        b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda", generator=g).view(torch.uint64)
        if k % 64:  # layout 'a' tails 0 (both operands, the rows API)
            mask = (1 << (k % 64)) - 1
            a.view(torch.int64)[:, -1] &= mask
            b.view(torch.int64)[:, -1] &= mask
        for dom in (_lib.POPCOUNT, _lib.DOT):
            ref = bnn.xnor_rows_gemm(a, b, k, algo="popc", domain=dom)
            for v in (2, 1):
                A(f"umma{v}")
                got = bnn.xnor_rows_gemm(a, b, k, algo="umma", domain=dom)
                assert torch.equal(got, ref), (m, n, k, dom, v)
            A("umma2")
    convs = [(3, 256, 13, 9, 70, 3, 3, (1, 1), (1, 1)), (8, 256, 28, 28, 256, 3, 3, (1, 1), (1, 1)),
             (4, 512, 7, 7, 96, 1, 1, (1, 1), (0, 0)), (2, 256, 15, 15, 300, 3, 3, (2, 2), (1, 1))]
    for i, (b_, c, h, w, f, kh, kw, st, pd) in enumerate(convs):
        x = rng.standard_normal((b_, c, h, w), dtype=np.float32)
        wt = rng.standard_normal((f, c, kh, kw), dtype=np.float32)
        outs = []
        for algo in ("popc", "umma2", "umma1", "umma3"):
            layer = bnn.QConvolution(c, f, (kh, kw), st, pd)
            layer.weight = wt
            layer.pack()
            layer.algo = A(algo)
            outs.append(layer.forward(torch.from_numpy(x).cuda(), bnn.INFER_PACKED).cpu().numpy())
        A("umma2")
        assert np.array_equal(outs[1], outs[0]), ("conv", i)
        assert np.array_equal(outs[2], outs[0]), ("conv", i)


@pytest.mark.parametrize("m,n,k", [(1024, 256, 4096), (1000, 200, 4096), (130, 17, 1024), (128, 256, 2048),
                                   (77, 64, 3000), (2304, 129, 4033), (300, 1, 1088), (64, 256, 1024)])
def test_small_gemm_cluster_split_k(bnn, m, n, k):
    """The in-kernel split-K route (bnn_gemm_splitk.cu: an 8-CTA cluster per 128-row tile, DSMEM
    reduction of exact integer partials) against the independently tested POPC engine: both
    domains, every pad-fill combination, affine epilogue, residual, [N, M] output, ragged M / N /
    K, K slices that leave some cluster ranks empty; repeated launches are bit-identical."""
    from paper_1705_09864_b200 import _lib
    W = (k + 63) // 64
    g = torch.Generator(device="cuda").manual_seed(m * 3 + n * 5 + k)
    a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda", generator=g).view(torch.uint64)
    b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda", generator=g).view(torch.uint64)
    sc = torch.randn(m, device="cuda", generator=g)
    sh = torch.randn(m, device="cuda", generator=g)
    for ap, bp in ((0, 0), (1, 0), (0, 1), (1, 1)):
        if k % 64:
            mask = (1 << (k % 64)) - 1
            for t, pad in ((a, ap), (b, bp)):
                last = t.view(torch.int64)[:, -1]
                last &= mask
                if pad:
                    last |= ~mask
        for dom in (_lib.POPCOUNT, _lib.DOT):
            ref = bnn.xnor_rows_gemm(a, b, k, a_pad=ap, b_pad=bp, algo="popc", domain=dom)
            got = bnn.xnor_rows_gemm(a, b, k, a_pad=ap, b_pad=bp, algo="umma", domain=dom)
            assert torch.equal(got, ref), (m, n, k, ap, bp, dom)
            assert torch.equal(bnn.xnor_rows_gemm(a, b, k, a_pad=ap, b_pad=bp, algo="umma", domain=dom), ref)
    ref = bnn.xnor_rows_gemm(a, b, k, algo="popc", domain=_lib.DOT, scale=sc, shift=sh, transpose_out=True)
    got = bnn.xnor_rows_gemm(a, b, k, algo="umma", domain=_lib.DOT, scale=sc, shift=sh, transpose_out=True)
    assert got.shape == (n, m) and torch.equal(got, ref)
    # the route is really the cluster kernel for these shapes: turning it off (debug bit 15)
    # gives the same numbers from the general engine
    _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 1 << 15)
    try:
        assert torch.equal(bnn.xnor_rows_gemm(a, b, k, algo="umma", domain=_lib.DOT, scale=sc, shift=sh,
                                              transpose_out=True), ref)
    finally:
        _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)


def test_cta_pair_route_bit_exact(bnn, monkeypatch):
    """The experimental 2-CTA (cta_group::2) kind::mxf4 route, forced on through a fresh
    process (the threshold is read once per process): bit-exact against the POPC engine."""
    import subprocess
    import sys
    code = (
        "import sys, torch; sys.path.insert(0, '.');"
        "import paper_1705_09864_b200 as bnn; bnn.load_library();"
        "from paper_1705_09864_b200 import _lib\n"
        "_lib.call('bnn_debug_set', _lib.DEBUG_PAIR_KW32, 1)\n"
        "ok = True\n"
        "for m, n, k in ((256, 128, 256), (512, 448, 4096), (1000, 1000, 8192), (300, 64, 2048)):\n"
        "    W = (k + 63) // 64; g = torch.Generator(device='cuda').manual_seed(m + n + k)\n"
        "    a = torch.randint(-2**63, 2**63 - 1, (m, W), device='cuda', generator=g).view(torch.uint64)\n"
        "    b = torch.randint(-2**63, 2**63 - 1, (n, W), device='cuda', generator=g).view(torch.uint64)\n"
        "    ok &= torch.equal(bnn.xnor_rows_gemm(a, b, k, algo='umma'), bnn.xnor_rows_gemm(a, b, k, algo='popc'))\n"
        "print('PAIR_OK' if ok else 'PAIR_BAD')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert "PAIR_OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("domain", ["dot", "popcount"])
def test_dense_plan_split_k_config1(bnn, golden_dir, domain):
    """Opt-in split-K: DensePlan runs word-aligned K ranges as GEMMs on forked
    streams and sums the exact counts (bnn_sum_partials_f32).  Bit-identical
    to the reference (golden SHA-256) and to the unsplit launch, eager and
    under CUDA-graph capture."""
    from paper_1705_09864_b200.plan import DensePlan
    a, w = wl.config1_inputs()
    layer = bnn.QFullyConnected(4096, 1024, domain=domain)
    layer.weight = w
    layer.pack()
    plan = DensePlan(layer, a.shape[0], host_splitk=8)
    assert len(plan.chunks) > 1
    plan.x.copy_(torch.from_numpy(a))
    y = plan.run_device().cpu().numpy()
    one = layer.forward(torch.from_numpy(a).cuda(), bnn.INFER_PACKED).cpu().numpy()
    assert np.array_equal(y, one)
    if domain == "dot":
        cfg = json.load(open(os.path.join(golden_dir, "configs.json")))["c1"]
        assert _sha(y) == cfg["sha256"]
    plan.y.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.run_device()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(plan.y.cpu().numpy(), one)


@pytest.mark.parametrize("splits,b,k,u", [(2, 300, 1000, 130), (3, 256, 4096, 1024), (5, 64, 2047, 257),
                                          (16, 129, 8192, 200)])
def test_dense_plan_split_k_ragged(bnn, splits, b, k, u):
    """Forced split counts over ragged K (tail in the last range only), odd units."""
    from paper_1705_09864_b200.plan import DensePlan
    rng = np.random.default_rng(splits * 31 + k)
    x = rng.standard_normal((b, k), dtype=np.float32)
    wt = rng.standard_normal((u, k), dtype=np.float32)
    layer = bnn.QFullyConnected(k, u)
    layer.weight = wt
    layer.pack()
    plan = DensePlan(layer, b, host_splitk=splits)
    assert len(plan.chunks) > 1 and plan.chunks[-1][1] == k
    plan.x.copy_(torch.from_numpy(x))
    y = plan.run_device().cpu().numpy()
    assert np.array_equal(y, orc.qdense_packed(orc.binarize(x), wt))
