"""Whole-network runners: cross-mode exactness + teacher-forced oracle.

As in the reference (test_layers.py:181-220), the packed path and the float
path must agree exactly at every binary layer; the binary conv is also
checked against the pinned CPU oracle on the GPU's own layer input
(teacher forcing), so float-op rounding differences upstream
cannot mask a kernel error.
"""

import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nets():
    import paper_1705_09864_b200 as p
    p.load_library()
    from paper_1705_09864_b200 import nets as n
    return n


def _modes(net, x, bnn):
    cap_f, cap_p = [], []
    yf = net.forward(x, bnn.INFER_FLOAT, capture=cap_f)
    yp = net.forward(x, bnn.INFER_PACKED, capture=cap_p)
    return yf, yp, cap_f, cap_p


def test_lenet_c3_cross_mode_and_oracle(nets):
    import paper_1705_09864_b200 as bnn
    net = nets.lenet_c3(seed=3)
    net.pack_for_inference()
    x = torch.rand((16, 1, 28, 28), generator=torch.Generator().manual_seed(0)).cuda()
    # fused BN epilogues (default) are bit-identical to the unfused float path
    yf, yp, cap_f, cap_p = _modes(net, x, bnn)
    for i in range(len(net.layers)):
        if cap_p[i] is not None:
            assert torch.equal(cap_f[i], cap_p[i]), f"layer {i}"
    assert torch.equal(yf, yp)
    assert yp.shape == (16, 10)
    net.fuse_bn = False
    yf, yp, cap_f, cap_p = _modes(net, x, bnn)
    for i, layer in enumerate(net.layers):
        if isinstance(layer, (bnn.QConvolution, bnn.QFullyConnected)):
            assert torch.equal(cap_f[i], cap_p[i]), f"layer {i}"
    assert torch.equal(yf, yp)
    # teacher-forced: the binary conv's GPU input through the CPU oracle
    conv = net.layers[3]
    xin = cap_p[2].cpu().numpy()
    expect = orc.qconv_packed(xin, conv.weight, conv.stride, conv.pad)
    assert np.array_equal(cap_p[3].cpu().numpy(), expect)
    fc = net.layers[7]
    xin = cap_p[6].cpu().numpy()
    expect = orc.qdense_packed(orc.binarize(xin), fc.weight)
    assert np.array_equal(cap_p[7].cpu().numpy(), expect)
    assert nets.binary_ops_per_image(net, (1, 28, 28)) == \
        2 * 64 * 14 * 14 * 64 * 25 + 2 * 1000 * 3136


def test_resnet18_c4_cross_mode(nets):
    import paper_1705_09864_b200 as bnn
    net = nets.resnet18_c4(seed=5, num_classes=1000)
    net.pack_for_inference()
    g = torch.Generator().manual_seed(1)
    x = torch.randn((4, 3, 224, 224), generator=g).cuda()
    yf, yp, cap_f, cap_p = _modes(net, x, bnn)
    assert yp.shape == (4, 1000)
    # blocks are composite: compare every block output (binary layers inside are exact)
    for i, layer in enumerate(net.layers):
        if isinstance(layer, nets.BinaryBasicBlock):
            assert torch.equal(cap_f[i], cap_p[i]), f"block {i}"
    assert torch.equal(yf, yp)
    # activations kept sign-packed between the binary convs (conv epilogues emit the
    # packed words) == a pack pass over every f32 block output
    for layer in net.layers:  # the shortcut add inside the conv2 epilogue
        if isinstance(layer, nets.BinaryBasicBlock):
            layer.split_shortcut = False
    assert torch.equal(net.forward(x, bnn.INFER_PACKED), yf)
    for layer in net.layers:
        if isinstance(layer, nets.BinaryBasicBlock):
            layer.packed_io = False
    assert torch.equal(net.forward(x, bnn.INFER_PACKED), yf)
    for layer in net.layers:  # unfused epilogues agree as well
        if isinstance(layer, nets.BinaryBasicBlock):
            layer.fused = False
    assert torch.equal(net.forward(x, bnn.INFER_PACKED), yf)
    ops = nets.binary_ops_per_image(net, (3, 224, 224))
    assert 3.3e9 < ops < 3.5e9  # 3.391e9 binary ops / image


@pytest.fixture(scope="module")
def resnet_run(nets):
    """One packed ResNet-18 (C4 topology) forward at batch 8 with per-layer capture."""
    import paper_1705_09864_b200 as bnn
    net = nets.resnet18_c4(seed=4)
    net.pack_for_inference()
    x = np.random.default_rng(4).standard_normal((8, 3, 224, 224)).astype(np.float32)
    cap = []
    y = net.forward(torch.from_numpy(x).cuda(), bnn.INFER_PACKED, capture=cap)
    return net, x, y, cap


def test_resnet18_teacher_forced_every_binary_conv(nets, resnet_run):
    """Every binary conv of ResNet-18 (16 3x3 convs + 3 strided 1x1 downsamples) against the
    pinned oracle (im2col(zero pad) -> binarize -> pack_matrix_b -> xnor GEMM, G2) on the
    GPU's own layer input (teacher forcing), and each block's output rebuilt
    from those convs == the packed network's captured block output, bit for bit."""
    import paper_1705_09864_b200 as bnn
    net, _, _, cap = resnet_run
    checked = 0
    for i, blk in enumerate(net.layers):
        if not isinstance(blk, nets.BinaryBasicBlock):
            continue
        xin = cap[i - 1]
        xin_np = xin.cpu().numpy()

        def check(conv, inp, inp_np):
            out = conv.forward(inp, bnn.INFER_PACKED)  # dot domain (BN applied separately)
            p = orc.qconv_packed(inp_np, conv.weight, conv.stride, conv.pad)
            assert np.array_equal(out.cpu().numpy(), 2 * p - np.float32(conv.k_reduce)), \
                (i, conv.in_channels, conv.filters, conv.kernel, conv.stride)
            return out

        h = blk.bn1.forward(check(blk.conv1, xin, xin_np))
        h2 = check(blk.conv2, h, h.cpu().numpy())
        sc = xin if blk.down is None else blk.bnd.forward(check(blk.down, xin, xin_np))
        checked += 2 + (blk.down is not None)
        assert torch.equal(blk.bn2.forward(h2) + sc, cap[i]), f"block {i}"
    assert checked == 19


def test_resnet18_end_to_end_vs_cpu_reference(nets, resnet_run):
    """ResNet-18 (C4) against the composed CPU reference (oracle/nets_ref: NumPy float
    layers + the pinned binary composition, G6):
    * the float stem agrees to f32 rounding (3xTF32 tensor cores vs NumPy BLAS);
    * from the GPU's stem output on, every block output is bit-identical (the binary
      layers are exact and BN / residual adds are the same f32 ops); the logits differ
      only by the average-pool / classifier summation order;
    * end to end from the raw images, sign flips of the block outputs (float rounding
      of the stem propagated through the sign activations) and top-1 agreement are
      reported, as for LeNet."""
    from oracle import nets_ref
    net, x, y, cap = resnet_run
    threads = os.cpu_count()
    stem_cpu = nets_ref.forward(nets.Sequential(net.layers[:2]), x, threads)
    stem_gpu = cap[1].cpu().numpy()
    assert np.all(np.abs(stem_gpu - stem_cpu) <= 1e-5 * np.maximum(1.0, np.abs(stem_cpu)))
    tail_cap = []
    y_tail = nets_ref.forward(nets.Sequential(net.layers[2:]), stem_gpu, threads, tail_cap)
    for j, layer in enumerate(net.layers[2:]):
        if isinstance(layer, nets.BinaryBasicBlock):
            assert np.array_equal(cap[j + 2].cpu().numpy(), tail_cap[j]), f"block {j + 2}"
    yg = y.cpu().numpy()
    assert np.all(np.abs(yg - y_tail) <= 1e-4 * np.maximum(1.0, np.abs(y_tail)))
    full_cap = []
    y_cpu = nets_ref.forward(net, x, threads, full_cap)
    flips = [float(np.mean((cap[i].cpu().numpy() >= 0) != (full_cap[i] >= 0)))
             for i, l in enumerate(net.layers) if isinstance(l, nets.BinaryBasicBlock)]
    top1 = float(np.mean(yg.argmax(1) == y_cpu.argmax(1)))
    print(f"\nResNet-18 end to end vs CPU reference: sign-flip rate per block {flips}, "
          f"top-1 agreement {top1:.3f}")
    assert max(flips) < 1e-2
    assert top1 >= 0.75


def test_lenet_c3_cross_mode_batch1024(nets):
    """BASELINE configs[2] at its benchmarked batch (1024): packed == float path at every
    binary layer and at the output."""
    import paper_1705_09864_b200 as bnn
    net = nets.lenet_c3(seed=3)
    net.pack_for_inference()
    x = torch.rand((1024, 1, 28, 28), generator=torch.Generator().manual_seed(6)).cuda()
    yf, yp, cap_f, cap_p = _modes(net, x, bnn)
    for i in range(len(net.layers)):
        if cap_p[i] is not None:
            assert torch.equal(cap_f[i], cap_p[i]), f"layer {i}"
    assert torch.equal(yf, yp) and yp.shape == (1024, 10)


def test_resnet_block_teacher_forced_oracle(nets):
    """One stride-2 block's binary convs against the oracle on the GPU's own inputs."""
    import paper_1705_09864_b200 as bnn
    rng = np.random.default_rng(9)
    blk = nets.BinaryBasicBlock(64, 128, 2, rng)
    for c in blk.binary_layers():
        c.pack()
    x = torch.randn((2, 64, 20, 20), generator=torch.Generator().manual_seed(2)).cuda()
    h1 = blk.conv1.forward(x, bnn.INFER_PACKED)
    xn = x.cpu().numpy()
    p = orc.qconv_packed(xn, blk.conv1.weight, (2, 2), (1, 1))
    assert np.array_equal(h1.cpu().numpy(), 2 * p - 64 * 9)  # dot domain
    d = blk.down.forward(x, bnn.INFER_PACKED)
    p = orc.qconv_packed(xn, blk.down.weight, (2, 2), (0, 0))
    assert np.array_equal(d.cpu().numpy(), 2 * p - 64)


def test_lenet_end_to_end_vs_cpu_reference(nets):
    """Full-network agreement with the CPU reference composition (float ops differ in
    rounding between cuDNN/torch and NumPy, so a sign can flip near 0)."""
    import paper_1705_09864_b200 as bnn
    from oracle import nets_ref
    net = nets.lenet_c3(seed=11)
    net.pack_for_inference()
    x = np.random.default_rng(3).random((32, 1, 28, 28), dtype=np.float32)
    cap = []
    y_gpu = net.forward(torch.from_numpy(x).cuda(), bnn.INFER_PACKED, capture=cap).cpu().numpy()
    y_cpu = nets_ref.forward(net, x)
    assert (y_gpu.argmax(1) == y_cpu.argmax(1)).mean() >= 0.9
    # the binary conv input differs from the CPU one only by float rounding: count sign flips
    xin_gpu = cap[2].cpu().numpy()
    flips = np.mean((xin_gpu >= 0) != (nets_ref.forward(nets.Sequential(net.layers[:3]), x) >= 0))
    assert flips < 1e-3


@pytest.mark.parametrize("shape,k,st,pd", [((2, 5, 17, 13), 3, 2, 1), ((1, 3, 8, 8), 2, 2, 0),
                                           ((3, 4, 9, 11), 3, 1, 1), ((2, 6, 40, 36), 3, 2, 1),
                                           ((1, 4, 112, 112), 3, 2, 1), ((1, 2, 7, 2000), 3, 2, 1)])
def test_stem_post_kernel_equals_torch_ops(nets, shape, k, st, pd):
    """bnn_bn_relu_maxpool_f32 is bit-identical to BatchNorm -> ReLU -> MaxPool (the
    banded kernel pools first and applies BN once: exact by monotonicity, also for
    negative and zero gammas)."""
    import paper_1705_09864_b200 as bnn
    rng = np.random.default_rng(4)
    post = nets.StemPost(shape[1], rng, k, st, pd)
    post.bn.gamma[::2] *= -1.0
    post.bn.gamma[1] = 0.0
    if shape[1] > 3:
        post.bn.gamma[3] = -0.0
    x = torch.randn(shape, generator=torch.Generator().manual_seed(3)).cuda()
    assert torch.equal(post.forward(x, bnn.INFER_PACKED), post.forward(x, bnn.INFER_FLOAT))


@pytest.mark.parametrize("case", [
    # (B, C, H, W, F, k, stride, pad, bias): ResNet-18 stem, LeNet conv1, ragged shapes
    (2, 3, 224, 224, 64, 7, 2, 3, False),
    (3, 1, 28, 28, 64, 5, 1, 2, True),
    (1, 3, 37, 29, 64, 7, 2, 3, True),
    (2, 5, 9, 13, 64, 3, 1, 1, True),
    (1, 6, 20, 20, 64, 7, 3, 0, False),
])
def test_conv2d_f32_tensor_core_accuracy(nets, case):
    """bnn_conv2d_f32_tc (3xTF32 on tcgen05) against a float64 convolution: f32-level
    error (|d| <= 1e-5 * max(1, |ref|), the tolerance of test_layers.py:68), no worse
    than cuDNN's f32 conv by more than a small factor."""
    import torch.nn.functional as F
    b, c, h, w, f, k, st, pd, bias = case
    rng = np.random.default_rng(sum(case[:8]))
    x = rng.standard_normal((b, c, h, w)).astype(np.float32)
    conv = nets.Conv2d(c, f, k, stride=st, pad=pd, bias=bias, rng=rng)
    if bias:
        conv.bias = rng.standard_normal(f).astype(np.float32)
    assert conv.tc_supported()
    xd = torch.from_numpy(x).cuda()
    y = conv.forward(xd).cpu().double()
    ref = F.conv2d(torch.from_numpy(x).double(), torch.from_numpy(conv.weight).double(),
                   torch.from_numpy(conv.bias).double() if bias else None, stride=st, padding=pd)
    err = (y - ref).abs()
    assert y.shape == ref.shape
    assert bool((err <= 1e-5 * ref.abs().clamp(min=1.0)).all()), float(err.max())
    conv.engine = "cudnn"
    y_cudnn = conv.forward(xd).cpu().double()
    assert float(err.max()) <= 4 * float((y_cudnn - ref).abs().max()) + 1e-6


@pytest.mark.parametrize("shape", [(2, 3, 224, 224), (3, 3, 36, 36), (2, 3, 30, 44), (1, 5, 20, 16)])
def test_fused_stem_conv_pool_bit_identical(nets, shape):
    """bnn_conv_bn_relu_maxpool_f32_tc == bnn_conv2d_f32_tc followed by BatchNorm ->
    ReLU -> MaxPool 3x3/2/1 bit for bit (pool-before-BN by monotonicity, negative and
    zero gammas included); the first case is ResNet-18's stem."""
    import paper_1705_09864_b200 as bnn
    rng = np.random.default_rng(shape[2])
    conv = nets.Conv2d(shape[1], 64, 7, stride=2, pad=3, bias=False, rng=rng)
    post = nets.StemPost(64, rng, 3, 2, 1)
    post.bn.gamma[::3] *= -1.0
    post.bn.gamma[1] = 0.0
    post.bn.gamma[4] = -0.0
    assert post.fusable(conv)
    x = torch.randn(shape, generator=torch.Generator().manual_seed(shape[3])).cuda()
    fused = post.forward_fused_conv(conv, x)
    conv_out = conv.forward(x)
    assert torch.equal(fused, post.forward(conv_out, bnn.INFER_PACKED))
    assert torch.equal(fused, post.forward(conv_out, bnn.INFER_FLOAT))


def test_lenet_fused_stem_bit_identical(nets):
    """bnn_conv_tanh_maxpool2_f32_tc == tensor-core conv -> torch.tanh -> max_pool2d."""
    import torch.nn.functional as F
    rng = np.random.default_rng(21)
    conv = nets.Conv2d(1, 64, 5, pad=2, rng=rng)
    conv.bias = rng.standard_normal(64).astype(np.float32) * 0.1
    x = torch.rand((5, 1, 28, 28), generator=torch.Generator().manual_seed(1)).cuda()
    ref = F.max_pool2d(torch.tanh(conv.forward(x)), 2)
    monotone = nets.tanh_is_monotone()
    for pool_first in ([False, True] if monotone else [False]):  # tanh per element / pool first
        fused = nets._lenet_stem_forward(conv, x, pool_first=pool_first)
        assert fused.shape == ref.shape and torch.equal(fused, ref), pool_first
        # the same kernel also writing the next binary conv's packed input (sign + pack fused),
        # with and without the f32 tensor
        import paper_1705_09864_b200 as bnn
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        expect = bnn.pack_nchw(ref).cpu().numpy()
        both = nets._lenet_stem_forward(conv, x, pool_first=pool_first, pack=True, flags=flags)
        assert both.shape == tuple(ref.shape) and torch.equal(both.f32, ref)
        assert np.array_equal(both.words.cpu().numpy(), expect)
        only = nets._lenet_stem_forward(conv, x, pool_first=pool_first, pack=True, f32_out=False,
                                        flags=flags)
        assert only.f32 is None and np.array_equal(only.words.cpu().numpy(), expect)
        assert int(flags.item()) == 0
    # a non-finite input raises the NONFINITE flag through the fused pack
    xb = x.clone()
    xb[2, 0, 5, 5] = float("nan")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    nets._lenet_stem_forward(conv, xb, pack=True, f32_out=False, flags=flags)
    assert int(flags.item()) != 0


@pytest.mark.parametrize("shape,k", [((3, 14, 14, 1), 2), ((2, 9, 7, 3), 3), ((1, 6, 10, 2), 2)])
def test_maxpool_packed_is_pack_of_maxpool(nets, shape, k):
    """OR-pooling sign-packed words == packing the max-pooled floats (sign(-0) = +1)."""
    import paper_1705_09864_b200 as bnn
    import torch.nn.functional as F
    from paper_1705_09864_b200 import _lib
    b, h, w, cw = shape
    c = 64 * cw
    x = torch.randn((b, c, h, w), generator=torch.Generator().manual_seed(h * w)).cuda()
    x.view(-1)[::7] = 0.0
    x.view(-1)[3::11] = -0.0
    words = bnn.pack_nchw(x)
    oh, ow = (h - k) // k + 1, (w - k) // k + 1
    out = torch.empty((b, oh, ow, cw), dtype=torch.uint64, device="cuda")
    _lib.call("bnn_maxpool_packed", _lib.ptr(words), b, h, w, cw, k, k, _lib.ptr(out),
              _lib.stream_ptr())
    expect = bnn.pack_nchw(F.max_pool2d(x, k)).cpu().numpy()
    assert np.array_equal(out.cpu().numpy(), expect)
    # the strided form (one padded row per image, what a following QFullyConnected reads)
    rw = oh * ow * cw
    pitch = rw + 3
    rows = torch.full((b, pitch), 0x5A5A, dtype=torch.int64, device="cuda").view(torch.uint64)
    _lib.call("bnn_maxpool_packed_ld", _lib.ptr(words), b, h, w, cw, k, k, _lib.ptr(rows), pitch,
              _lib.stream_ptr())
    got = rows.cpu().numpy()
    assert np.array_equal(got[:, :rw], expect.reshape(b, rw))
    assert np.all(got[:, rw:] == 0x5A5A)  # the pad words are not touched
    with pytest.raises(Exception):
        _lib.call("bnn_maxpool_packed_ld", _lib.ptr(words), b, h, w, cw, k, k, _lib.ptr(rows), rw - 1,
                  _lib.stream_ptr())


def test_lenet_packed_tail_equals_float_path(nets):
    """QConv -> BN -> maxpool -> flatten -> QFC -> BN with 1-bit activations between the
    binary layers == the same layers on f32 tensors (infer_float), bit for bit."""
    import paper_1705_09864_b200 as bnn
    net = nets.lenet_c3(seed=8)
    net.pack_for_inference()
    tail = nets.Sequential(net.layers[3:9])
    assert nets._binary_pool_fc(tail.layers)
    x = torch.randn((6, 64, 14, 14), generator=torch.Generator().manual_seed(5)).cuda()
    x.view(-1)[::13] = 0.0
    assert torch.equal(tail.forward(x, bnn.INFER_PACKED), tail.forward(x, bnn.INFER_FLOAT))


def test_fused_stem_sign_pack(nets):
    """The stem kernel's packed output == packing its f32 output (the first block's input)."""
    import paper_1705_09864_b200 as bnn
    rng = np.random.default_rng(17)
    conv = nets.Conv2d(3, 64, 7, stride=2, pad=3, bias=False, rng=rng)
    post = nets.StemPost(64, rng, 3, 2, 1)
    post.bn.gamma[::3] *= -1.0
    x = torch.randn((2, 3, 64, 64), generator=torch.Generator().manual_seed(3)).cuda()
    out = post.forward_fused_conv(conv, x, pack=True)
    assert isinstance(out, nets.PackedNHWC)
    assert torch.equal(out.f32, post.forward_fused_conv(conv, x))
    assert np.array_equal(out.words.cpu().numpy(), bnn.pack_nchw(out.f32).cpu().numpy())


@pytest.mark.parametrize("shape", [(2, 3, 224, 224), (1, 3, 37, 224), (3, 3, 8, 224), (2, 3, 1, 224),
                                   (1, 3, 225, 224), (5, 3, 58, 224)])
def test_stride2_stem_kernel(nets, shape):
    """The gather-free stride-2 stem kernel (bnn_stem_s2.cu; W = 224, conv7x7/2 pad 3, 64
    filters): its raw conv output (with a bias) is f32-accurate against a float64
    convolution, and its fused BN -> ReLU -> maxpool output and sign-packed words equal the
    post-op applied to its own raw output bit for bit -- for odd heights, single-row
    images, several bands per image and repeated launches."""
    import torch.nn.functional as F
    import paper_1705_09864_b200 as bnn
    rng = np.random.default_rng(shape[0] * 1000 + shape[2])
    conv = nets.Conv2d(3, 64, 7, stride=2, pad=3, bias=True, rng=rng)
    conv.bias = rng.standard_normal(64).astype(np.float32)
    x = torch.randn(shape, generator=torch.Generator().manual_seed(shape[2])).cuda()
    y = conv.forward(x)
    ref = F.conv2d(x.cpu().double(), torch.from_numpy(conv.weight).double(),
                   torch.from_numpy(conv.bias).double(), stride=2, padding=3)
    err = (y.cpu().double() - ref).abs()
    assert y.shape == ref.shape
    assert bool((err <= 1e-5 * ref.abs().clamp(min=1.0)).all()), float(err.max())
    conv.bias = None
    conv.__dict__.pop("_dev_cache", None)  # (device copies are cached per attribute)
    post = nets.StemPost(64, rng, 3, 2, 1)
    post.bn.gamma[::3] *= -1.0
    post.bn.gamma[1] = 0.0
    raw = conv.forward(x)
    fused = post.forward_fused_conv(conv, x, pack=True)
    assert isinstance(fused, nets.PackedNHWC)
    assert torch.equal(fused.f32, post.forward(raw, bnn.INFER_FLOAT))
    assert torch.equal(fused.f32, post.forward_fused_conv(conv, x))
    assert np.array_equal(fused.words.cpu().numpy(), bnn.pack_nchw(fused.f32).cpu().numpy())
    # repeated launches (ring / accumulator phases restart cleanly) are bit-identical
    assert torch.equal(post.forward_fused_conv(conv, x), fused.f32)


def test_classifier_head_is_batch_independent(nets):
    """bnn_avgpool_fc_f32 (GlobalAvgPool -> Dense): f32-accurate against float64 and each
    image's logits bit-identical in any batch / shard (what multi-GPU batch sharding
    relies on); both network modes use it."""
    rng = np.random.default_rng(3)
    dense = nets.Dense(512, 1000, rng=rng)
    dense.bias = rng.standard_normal(1000).astype(np.float32)
    x = torch.randn((37, 512, 7, 7), generator=torch.Generator().manual_seed(2)).cuda()
    y = nets.avgpool_dense(x, dense)
    ref = x.double().mean(dim=(2, 3)) @ torch.from_numpy(dense.weight).double().cuda().T + \
        torch.from_numpy(dense.bias).double().cuda()
    assert torch.allclose(y.double(), ref, rtol=1e-5, atol=1e-5)
    for lo, hi in ((0, 1), (3, 11), (11, 37), (5, 6)):
        assert torch.equal(nets.avgpool_dense(x[lo:hi], dense), y[lo:hi]), (lo, hi)
