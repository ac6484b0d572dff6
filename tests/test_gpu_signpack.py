"""Fused sign-pack epilogue: the next layer's QActivation + pack
(layers.py:409-413 -> bitpack.binarize :30-42 -> _pack_last_axis :78-87) run in
the GEMM / conv epilogue, so activations stay 1 bit per element between binary
layers.

The packed words must equal the oracle's pack of sign(f32 output) bit for bit
(channel tail 0, sign(-0) = +1), and the f32 output must be unchanged by the
extra output.
"""

import ctypes

import numpy as np
import pytest
import torch

import workloads as wl
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bnn():
    import paper_1705_09864_b200 as p
    p.load_library()
    return p


class _BN:
    """BatchNorm parameters whose mean hits exact dot-domain integers, so some
    outputs are exactly +0 / -0 (negative gammas give -0 products)."""

    def __init__(self, f, k, seed):
        rng = np.random.default_rng(seed)
        self.mean = (2 * rng.integers(-4, 5, f) + (k % 2)).astype(np.float32)
        self.inv = (0.5 + rng.random(f)).astype(np.float32)
        self.gamma = (rng.standard_normal(f)).astype(np.float32)
        self.beta = np.where(rng.random(f) < 0.5, 0.0, -0.0).astype(np.float32)
        self.beta[::5] = rng.standard_normal(len(self.beta[::5])).astype(np.float32) * 3

    def device_params(self):
        return tuple(torch.from_numpy(a).cuda() for a in (self.mean, self.inv, self.gamma, self.beta))


def _oracle_pack_nhwc(y_nchw: np.ndarray) -> np.ndarray:
    b, f, h, w = y_nchw.shape
    rows = np.ascontiguousarray(y_nchw.transpose(0, 2, 3, 1).reshape(-1, f))
    return orc.binarize_pack_rows(rows, pad_fill=0).reshape(b, h, w, -1)


# (B, C, H, W, F, kh, kw, stride, pad, seed): cp.async route (C % 256 != 0) and the
# im2col-TMA route (C % 256 == 0); F not a multiple of 64 / 32; images of fewer
# than 32 pixels (32-column blocks straddle images)
CASES = [
    (2, 64, 9, 9, 64, 3, 3, (1, 1), (1, 1), 1),
    (3, 64, 7, 7, 96, 3, 3, (1, 1), (1, 1), 2),
    (2, 128, 8, 8, 24, 3, 3, (2, 2), (1, 1), 3),
    (2, 256, 7, 7, 160, 3, 3, (1, 1), (1, 1), 4),
    (4, 256, 5, 5, 256, 3, 3, (1, 1), (1, 1), 5),
    (1, 512, 9, 11, 200, 1, 1, (2, 2), (0, 0), 6),
    (2, 100, 12, 12, 70, 3, 3, (1, 1), (1, 1), 7),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("variant", [2, 1, 0, 4])
@pytest.mark.parametrize("with_res", [False, True])
def test_conv_sign_pack_epilogue(bnn, case, variant, with_res):
    from paper_1705_09864_b200.layers import PackedNHWC
    b, c, h, w, f, kh, kw, stride, pad, seed = case
    x, wt = wl.conv_case_inputs(case)
    layer = bnn.QConvolution(c, f, (kh, kw), stride, pad, domain="dot")
    layer.weight = wt
    layer.pack()
    layer.algo = f"umma{variant}"
    bn = _BN(f, c * kh * kw, seed)
    oh, ow = layer.output_hw(h, w)
    res = None
    if with_res:
        res = torch.from_numpy(np.random.default_rng(seed + 50).standard_normal(
            (b, f, oh, ow)).astype(np.float32)).cuda()
        res.view(-1)[::9] = 0.0
    xd = torch.from_numpy(x).cuda()
    plain = layer.forward_fused(xd, bn, residual=res)
    out = layer.forward_fused(xd, bn, residual=res, pack_out=True)
    assert isinstance(out, PackedNHWC) and out.shape == (b, f, oh, ow)
    y = plain.cpu().numpy()
    assert np.array_equal(out.f32.cpu().numpy(), y)  # f32 output unchanged
    # the unfused composition: conv -> BN -> (+ res) in the reference op order
    p = orc.qconv_packed(x, wt, stride, pad).astype(np.float32)
    ref = 2 * p - np.float32(c * kh * kw)
    sh = (1, -1, 1, 1)
    ref = bn.gamma.reshape(sh) * ((ref - bn.mean.reshape(sh)) * bn.inv.reshape(sh)) + \
        bn.beta.reshape(sh)
    if with_res:
        ref = ref + res.cpu().numpy()
    assert np.array_equal(y, ref.astype(np.float32))
    words = out.words.cpu().numpy()
    assert np.array_equal(words, _oracle_pack_nhwc(y))
    assert np.array_equal(words, bnn.pack_nchw(plain).cpu().numpy())
    # packed-only output (the f32 tensor is never written)
    only = layer.forward_fused(xd, bn, residual=res, pack_out=True, f32_out=False)
    assert only.f32 is None and np.array_equal(only.words.cpu().numpy(), words)
    # a consumer conv reading the packed words == reading the f32 tensor
    nxt = bnn.QConvolution(f, 40, (3, 3), (1, 1), (1, 1), domain="dot")
    nxt.weight = np.random.default_rng(seed + 9).standard_normal((40, f, 3, 3)).astype(np.float32)
    nxt.pack()
    assert torch.equal(nxt.forward_fused(only), nxt.forward_fused(plain))


# POPC-pipe pointwise conv (bnn_pwconv.cu, the AUTO route of 1x1 / pad 0 / C <= 256 convs with an
# f32 output): ResNet-18's three downsample shapes, ragged channels / filters, strides 1-3,
# asymmetric strides, pixel counts that straddle images inside a warp
PW_CASES = [
    (3, 64, 56, 56, 128, 1, 1, (2, 2), (0, 0), 21),
    (2, 128, 28, 28, 256, 1, 1, (2, 2), (0, 0), 22),
    (5, 256, 14, 14, 512, 1, 1, (2, 2), (0, 0), 23),
    (7, 100, 9, 11, 70, 1, 1, (1, 1), (0, 0), 24),
    (4, 200, 13, 7, 130, 1, 1, (3, 2), (0, 0), 25),
    (33, 40, 5, 5, 9, 1, 1, (1, 2), (0, 0), 26),
    (24, 64, 112, 112, 24, 1, 1, (1, 1), (0, 0), 27),  # >= 2^17 pixels: the 4-pixel kernel
    (88, 50, 112, 112, 17, 1, 1, (2, 2), (0, 0), 28),  # the same with stride 2, ragged C / F
]


@pytest.mark.parametrize("case", PW_CASES)
@pytest.mark.parametrize("domain", ["dot", "popcount"])
def test_pointwise_conv_popc_route(bnn, case, domain):
    """AUTO takes the POPC pointwise kernel here; bit-identical to the tcgen05 engine (umma2),
    to the CUDA-core engine and to the oracle's conv -> BN (-> + shortcut) composition."""
    b, c, h, w, f, kh, kw, stride, pad, seed = case
    x, wt = wl.conv_case_inputs(case)
    layer = bnn.QConvolution(c, f, (kh, kw), stride, pad, domain=domain)
    layer.weight = wt
    layer.pack()
    bn = _BN(f, c, seed)
    oh, ow = layer.output_hw(h, w)
    res = torch.from_numpy(np.random.default_rng(seed + 50).standard_normal(
        (b, f, oh, ow)).astype(np.float32)).cuda()
    xd = torch.from_numpy(x).cuda()
    p = orc.qconv_packed(x, wt, stride, pad).astype(np.float32)
    base = 2 * p - np.float32(c) if domain == "dot" else p
    sh = (1, -1, 1, 1)
    ref_bn = bn.gamma.reshape(sh) * ((base - bn.mean.reshape(sh)) * bn.inv.reshape(sh)) + \
        bn.beta.reshape(sh)
    outs = {}
    for algo in ("auto", "umma2", "popc"):
        layer.algo = algo
        outs[algo] = (layer.forward_fused(xd).cpu().numpy(),
                      layer.forward_fused(xd, bn).cpu().numpy(),
                      layer.forward_fused(xd, bn, residual=res).cpu().numpy())
    assert np.array_equal(outs["auto"][0], base)
    assert np.array_equal(outs["auto"][1], ref_bn.astype(np.float32))
    assert np.array_equal(outs["auto"][2], (ref_bn + res.cpu().numpy()).astype(np.float32))
    for algo in ("umma2", "popc"):
        for a, o in zip(outs["auto"], outs[algo]):
            assert np.array_equal(a, o), algo
    # a sign-packed output is not the pointwise kernel's: AUTO falls through, same words
    layer.algo = "auto"
    pk = layer.forward_fused(xd, bn, pack_out=True)
    assert np.array_equal(pk.f32.cpu().numpy(), outs["auto"][1])
    assert np.array_equal(pk.words.cpu().numpy(), _oracle_pack_nhwc(outs["auto"][1]))


# pre-expanded conv engine (bnn_bconv2d_ws, C % 256 == 0, F % 64 == 0): strides 1 / 2, 1x1 and
# 5x5 kernels, asymmetric geometry, image sizes that make 32-pixel lane groups straddle images,
# pixel counts below / across the 256-row pair tile, ResNet-18 layer-3 / layer-4 shapes
XP_CASES = [
    (2, 256, 7, 7, 128, 3, 3, (1, 1), (1, 1), 11),
    (4, 256, 5, 5, 256, 3, 3, (1, 1), (1, 1), 12),
    (3, 512, 9, 11, 192, 1, 1, (2, 2), (0, 0), 13),
    (2, 256, 9, 8, 64, 3, 3, (2, 2), (1, 1), 14),
    (1, 512, 6, 6, 512, 5, 5, (1, 1), (2, 2), 15),
    (5, 256, 10, 13, 320, 3, 2, (1, 2), (1, 0), 16),
    (33, 256, 14, 14, 256, 3, 3, (1, 1), (1, 1), 17),
    (20, 512, 7, 7, 512, 3, 3, (1, 1), (1, 1), 18),
]


@pytest.mark.parametrize("case", XP_CASES)
def test_conv_pre_expanded_engine(bnn, case):
    """Every epilogue form of bnn_bconv2d_ws on the pre-expanded engine: bit-identical to the
    packed tcgen05 engine, and to the oracle's conv -> BN -> (+ shortcut) composition."""
    b, c, h, w, f, kh, kw, stride, pad, seed = case
    x, wt = wl.conv_case_inputs(case)
    outs = {}
    bn = _BN(f, c * kh * kw, seed)
    for algo in ("umma2", "xp", "auto"):
        layer = bnn.QConvolution(c, f, (kh, kw), stride, pad, domain="dot")
        layer.weight = wt
        layer.pack()
        layer.algo = algo
        oh, ow = layer.output_hw(h, w)
        res = torch.from_numpy(np.random.default_rng(seed + 50).standard_normal(
            (b, f, oh, ow)).astype(np.float32)).cuda()
        res.view(-1)[::9] = 0.0
        xd = torch.from_numpy(x).cuda()
        o = {"plain": layer.forward(xd, bnn.INFER_PACKED),
             "bn": layer.forward_fused(xd, bn),
             "bn_res": layer.forward_fused(xd, bn, residual=res)}
        pk = layer.forward_fused(xd, bn, residual=res, pack_out=True)
        o["pk_f32"], o["pk_words"] = pk.f32, pk.words
        o["only_words"] = layer.forward_fused(xd, bn, pack_out=True, f32_out=False).words
        pop = bnn.QConvolution(c, f, (kh, kw), stride, pad)  # popcount domain
        pop.weight = wt
        pop.pack()
        pop.algo = algo
        o["popcount"] = pop.forward(xd, bnn.INFER_PACKED)
        outs[algo] = o
    for key, ref in outs["umma2"].items():
        for algo in ("xp", "auto"):
            assert torch.equal(outs[algo][key], ref), (algo, key)
    p = orc.qconv_packed(x, wt, stride, pad).astype(np.float32)
    assert np.array_equal(outs["xp"]["popcount"].cpu().numpy(), p)
    ref = 2 * p - np.float32(c * kh * kw)
    assert np.array_equal(outs["xp"]["plain"].cpu().numpy(), ref)
    sh = (1, -1, 1, 1)
    ref = bn.gamma.reshape(sh) * ((ref - bn.mean.reshape(sh)) * bn.inv.reshape(sh)) + bn.beta.reshape(sh)
    assert np.array_equal(outs["xp"]["bn"].cpu().numpy(), ref.astype(np.float32))
    y = outs["xp"]["bn_res"].cpu().numpy()
    assert np.array_equal(y, (ref + res.cpu().numpy()).astype(np.float32))
    assert np.array_equal(outs["xp"]["pk_words"].cpu().numpy(), _oracle_pack_nhwc(y))


def _gemm_ex(bnn, a, bw, m, n, k, c, ldc_m, ldc_n, e, algo="auto"):
    from paper_1705_09864_b200 import _lib
    _lib.call("bnn_xnor_gemm_ex", _lib.ptr(a), a.stride(0), _lib.ptr(bw), bw.stride(0), m, n, k,
              0, 0, _lib.ptr(c), ldc_m, ldc_n, ctypes.byref(e), _lib.ALGOS[algo],
              _lib.stream_ptr())


@pytest.mark.parametrize("m,n,k", [(64, 40, 300), (1000, 256, 4096), (130, 77, 64), (32, 500, 1)])
@pytest.mark.parametrize("transposed", [False, True])
def test_dense_sign_pack_epilogue(bnn, m, n, k, transposed):
    """QFullyConnected -> BN -> sign -> pack: words of the [N, M] layer output
    rows (the K-contiguous rows the next dense layer reads)."""
    from paper_1705_09864_b200.layers import make_epilogue
    rng = np.random.default_rng(m + n + k)
    w = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    x = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    wa = torch.from_numpy(orc.binarize_pack_rows(w)).cuda()
    xb = torch.from_numpy(orc.binarize_pack_rows(x)).cuda()
    bn = _BN(m, k, m)
    words = torch.full((n, (m + 63) // 64 + 1), 0x5A5A, dtype=torch.int64).cuda().view(torch.uint64)
    if transposed:  # layer output [N, M]
        c = torch.empty((n, m), dtype=torch.float32, device="cuda")
        ldc_m, ldc_n = 1, m
    else:
        c = torch.empty((m, n), dtype=torch.float32, device="cuda")
        ldc_m, ldc_n = n, 1
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    e = make_epilogue(bnn._lib.DOT, bn, pack_out=words, pack_flags=flags)
    _gemm_ex(bnn, wa, xb, m, n, k, c, ldc_m, ldc_n, e)
    y = c.cpu().numpy() if transposed else c.cpu().numpy().T  # [N, M]
    dot = np.float32(k) - 2 * orc.xor_popc_rowrow(orc.binarize_pack_rows(w),
                                                   orc.binarize_pack_rows(x)).astype(np.float32)
    ref = bn.gamma * ((dot.T - bn.mean) * bn.inv) + bn.beta
    assert np.array_equal(y, ref.astype(np.float32))
    got = words.cpu().numpy()
    wpk = (m + 63) // 64
    assert np.array_equal(got[:, :wpk], orc.binarize_pack_rows(np.ascontiguousarray(y)))
    assert np.all(got[:, wpk:] == 0x5A5A)  # past ceil(M/64): untouched
    assert int(flags.item()) == 0


def test_sign_pack_flags_nonfinite_and_validation(bnn):
    from paper_1705_09864_b200 import _lib
    from paper_1705_09864_b200.layers import make_epilogue
    m, n, k = 70, 33, 128
    rng = np.random.default_rng(0)
    wa = torch.from_numpy(orc.binarize_pack_rows(rng.uniform(-1, 1, (m, k)).astype(np.float32))).cuda()
    xb = torch.from_numpy(orc.binarize_pack_rows(rng.uniform(-1, 1, (n, k)).astype(np.float32))).cuda()
    bn = _BN(m, k, 1)
    bn.mean[5] = np.nan  # channel 5 -> NaN outputs: binarize's ValueError case
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    words = torch.empty((n, 2), dtype=torch.uint64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    e = make_epilogue(_lib.DOT, bn, pack_out=words, pack_flags=flags)
    _gemm_ex(bnn, wa, xb, m, n, k, c, n, 1, e)
    assert int(flags.item()) == 1
    # the CUDA-core engines have no fused sign-pack
    with pytest.raises(ValueError, match="tcgen05"):
        _gemm_ex(bnn, wa, xb, m, n, k, c, n, 1, e, algo="popc")
    small = torch.empty((n, 1), dtype=torch.uint64, device="cuda")
    e2 = make_epilogue(_lib.DOT, None, pack_out=small, pack_flags=flags)
    with pytest.raises(ValueError, match="pack_ld"):
        _gemm_ex(bnn, wa, xb, m, n, k, c, n, 1, e2)
    # a null f32 output is legal only with a packed output
    e3 = make_epilogue(_lib.DOT, None)
    with pytest.raises(ValueError, match="null"):
        _lib.call("bnn_xnor_gemm_ex", _lib.ptr(wa), wa.stride(0), _lib.ptr(xb), xb.stride(0), m, n,
                  k, 0, 0, None, n, 1, ctypes.byref(e3), _lib.ALGOS["auto"], _lib.stream_ptr())


@pytest.mark.parametrize("shape", [(2, 64, 9, 9), (3, 100, 5, 7), (1, 32, 4, 4)])
def test_add_pack_nchw(bnn, shape):
    """bnn_add_pack_nchw_f32: y = a + r (f32) and the packed sign words of y."""
    from paper_1705_09864_b200 import _lib
    g = torch.Generator().manual_seed(sum(shape))
    a = torch.randn(shape, generator=g).cuda()
    r = torch.randn(shape, generator=g).cuda()
    a.view(-1)[::7] = 0.0
    r.view(-1)[::7] = -0.0
    b, c, h, w = shape
    y = torch.empty_like(a)
    words = torch.empty((b, h, w, (c + 63) // 64), dtype=torch.uint64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("bnn_add_pack_nchw_f32", _lib.ptr(a), _lib.ptr(r), b, c, h, w, _lib.ptr(y),
              _lib.ptr(words), _lib.ptr(flags), _lib.stream_ptr())
    assert torch.equal(y, a + r)
    assert np.array_equal(words.cpu().numpy(), bnn.pack_nchw(a + r).cpu().numpy())
    assert int(flags.item()) == 0


# Small-channel kernel (bnn_sconv.cu: C, F in {64, 128}, pixels in TMEM, filter-stationary
# weights): every epilogue combination against the oracle composition and against the
# general engine (variant 4 -- no small-channel route) on the same inputs.  Shapes: ResNet
# layer 1/2 geometry at small batch, strided 3x3 and 1x1 downsamples, images whose tiles
# straddle images and rows, odd image widths (falls back when W * C / 64 is odd), pad 0.
SCONV_CASES = [
    (2, 64, 56, 56, 64, 3, 3, (1, 1), (1, 1), 11),
    (3, 64, 56, 56, 128, 3, 3, (2, 2), (1, 1), 12),
    (2, 128, 28, 28, 128, 3, 3, (1, 1), (1, 1), 13),
    (3, 64, 56, 56, 128, 1, 1, (2, 2), (0, 0), 14),
    (5, 64, 10, 12, 64, 3, 3, (1, 1), (1, 1), 15),
    (2, 128, 9, 6, 64, 3, 3, (1, 1), (0, 0), 16),
    (1, 64, 7, 9, 128, 3, 3, (2, 2), (1, 1), 17),
    (4, 128, 14, 14, 128, 1, 1, (1, 1), (0, 0), 18),
    (2, 64, 33, 20, 64, 3, 3, (2, 1), (1, 1), 19),
]


@pytest.fixture(params=[0, 3], ids=["grid_sms", "grid_cap3"])
def grid_cap(request):
    """0: one CTA per SM; 3: three persistent CTAs, so every CTA walks many tiles and
    every ring (bands, A chunks, accumulators, popcounts) wraps around."""
    from paper_1705_09864_b200 import _lib
    _lib.call("bnn_debug_set", _lib.DEBUG_GRID_CAP, request.param)
    yield request.param
    _lib.call("bnn_debug_set", _lib.DEBUG_GRID_CAP, 0)


@pytest.mark.parametrize("case", SCONV_CASES)
@pytest.mark.parametrize("epi", ["plain", "bn_pack", "bn_res_pack", "bn_res"])
def test_small_channel_conv_kernel(bnn, case, epi, grid_cap):
    from paper_1705_09864_b200.layers import PackedNHWC
    b, c, h, w, f, kh, kw, stride, pad, seed = case
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, c, h, w)).astype(np.float32)
    x.reshape(-1)[::17] = 0.0
    wt = rng.standard_normal((f, c, kh, kw)).astype(np.float32)
    layer = bnn.QConvolution(c, f, (kh, kw), stride, pad, domain="dot")
    layer.weight = wt
    layer.pack()
    oh, ow = layer.output_hw(h, w)
    xd = torch.from_numpy(x).cuda()
    p = orc.qconv_packed(x, wt, stride, pad).astype(np.float32)
    ref = 2 * p - np.float32(c * kh * kw)
    if epi == "plain":
        y = layer.forward_fused(xd)
        assert np.array_equal(y.cpu().numpy(), ref)
        return
    bn = _BN(f, c * kh * kw, seed)
    # constant-sign channels (zero / negative-zero gamma) and huge gammas (outputs that
    # overflow to +-inf: the packed-only path keeps the full chain and raises the flag)
    bn.gamma[:3] = [0.0, -0.0, 1e-30]
    bn.beta[:3] = [-0.0, 1.0, -1.0]
    sh = (1, -1, 1, 1)
    ref = bn.gamma.reshape(sh) * ((ref - bn.mean.reshape(sh)) * bn.inv.reshape(sh)) + \
        bn.beta.reshape(sh)
    res = None
    if "res" in epi:
        res = torch.from_numpy(rng.standard_normal((b, f, oh, ow)).astype(np.float32)).cuda()
        res.view(-1)[::9] = 0.0
        ref = ref + res.cpu().numpy()
    ref = ref.astype(np.float32)
    pack = "pack" in epi
    out = layer.forward_fused(xd, bn, residual=res, pack_out=pack)
    y = out.f32 if pack else out
    assert np.array_equal(y.cpu().numpy(), ref)
    if pack:
        assert isinstance(out, PackedNHWC)
        assert np.array_equal(out.words.cpu().numpy(), _oracle_pack_nhwc(ref))
        only = layer.forward_fused(xd, bn, residual=res, pack_out=True, f32_out=False)
        assert np.array_equal(only.words.cpu().numpy(), out.words.cpu().numpy())
    layer.algo = "umma4"  # the general engine on the same inputs
    other = layer.forward_fused(xd, bn, residual=res, pack_out=pack)
    assert torch.equal(other.f32 if pack else other, y)


# Shifted-window kernel (bnn_wconv.cu: stride 1, every pixel expanded once, taps = shifted
# no-swizzle descriptors).  Geometries beyond the ResNet ones: asymmetric / zero padding,
# non-square kernels and images, the widest padded row (Wp = 64), bands that cross images,
# one-pixel images, 64 <-> 128 channel / filter mixes, C = 256 with filter groups (C = 512
# falls through to the general engine).
WCONV_CASES = [
    (3, 64, 17, 62, 64, 3, 3, (1, 1), 31),
    (2, 128, 9, 11, 64, 3, 3, (0, 1), 32),
    (2, 64, 12, 7, 128, 3, 3, (1, 0), 33),
    (4, 64, 6, 5, 128, 1, 3, (0, 1), 34),
    (2, 128, 8, 8, 128, 3, 1, (1, 0), 35),
    (5, 64, 1, 1, 64, 3, 3, (1, 1), 36),
    (2, 64, 30, 30, 64, 2, 2, (1, 1), 37),
    (9, 128, 4, 4, 128, 3, 3, (2, 2), 38),
    (2, 256, 10, 12, 256, 3, 3, (1, 1), 39),
    (2, 512, 5, 6, 192, 3, 3, (1, 1), 40),
    (8, 256, 14, 14, 256, 3, 3, (1, 1), 41),    # C = 256 on this kernel with 3 CTAs (grid_cap3)
    (190, 256, 14, 14, 256, 3, 3, (1, 1), 42),  # ... and with every SM (>= 5 tiles per CTA)
    # kernels up to 5 x 5 (C * kh * kw <= 5120): LeNet's binary conv, non-square / asymmetric ones
    (37, 64, 14, 14, 64, 5, 5, (2, 2), 43),
    (3, 64, 9, 20, 128, 5, 3, (2, 0), 44),
    (2, 128, 11, 8, 64, 4, 5, (3, 4), 45),
    (2, 64, 7, 7, 64, 5, 5, (0, 0), 46),
    (2, 128, 6, 9, 128, 5, 5, (4, 1), 47),
]


@pytest.mark.parametrize("case", WCONV_CASES)
@pytest.mark.parametrize("epi", ["plain", "bn_pack", "bn_res_pack"])
def test_shifted_window_conv_kernel(bnn, case, epi, grid_cap):
    from paper_1705_09864_b200 import _lib
    from paper_1705_09864_b200.layers import PackedNHWC
    b, c, h, w, f, kh, kw, pad, seed = case
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, c, h, w)).astype(np.float32)
    x.reshape(-1)[::13] = 0.0
    wt = rng.standard_normal((f, c, kh, kw)).astype(np.float32)
    layer = bnn.QConvolution(c, f, (kh, kw), (1, 1), pad, domain="dot")
    layer.weight = wt
    layer.pack()
    oh, ow = layer.output_hw(h, w)
    xd = torch.from_numpy(x).cuda()
    p = orc.qconv_packed(x, wt, (1, 1), pad).astype(np.float32)
    ref = 2 * p - np.float32(c * kh * kw)
    try:
        if epi == "plain":
            assert np.array_equal(layer.forward_fused(xd).cpu().numpy(), ref)
            return
        bn = _BN(f, c * kh * kw, seed)
        bn.gamma[:3] = [0.0, -0.0, 1e-30]
        bn.beta[:3] = [-0.0, 1.0, -1.0]
        sh = (1, -1, 1, 1)
        ref = bn.gamma.reshape(sh) * ((ref - bn.mean.reshape(sh)) * bn.inv.reshape(sh)) + bn.beta.reshape(sh)
        res = None
        if "res" in epi:
            res = torch.from_numpy(rng.standard_normal((b, f, oh, ow)).astype(np.float32)).cuda()
            ref = ref + res.cpu().numpy()
        ref = ref.astype(np.float32)
        out = layer.forward_fused(xd, bn, residual=res, pack_out=True)
        assert isinstance(out, PackedNHWC)
        assert np.array_equal(out.f32.cpu().numpy(), ref)
        assert np.array_equal(out.words.cpu().numpy(), _oracle_pack_nhwc(ref))
        only = layer.forward_fused(xd, bn, residual=res, pack_out=True, f32_out=False)
        assert np.array_equal(only.words.cpu().numpy(), out.words.cpu().numpy())
        again = layer.forward_fused(xd, bn, residual=res, pack_out=True, f32_out=False)
        assert np.array_equal(again.words.cpu().numpy(), out.words.cpu().numpy())
    finally:
        _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
