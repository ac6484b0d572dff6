"""Pointwise (1x1 stride-2) downsample convs of ResNet-18 at batch 256: the POPC-pipe kernel
(bnn_pwconv.cu, AUTO) against the tensor-core engines (debug bit 1 << 29), CUDA-graph timed."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets, _lib  # noqa: E402
from paper_1705_09864_b200.layers import PackedNHWC  # noqa: E402

bnn.load_library()
rng = np.random.default_rng(0)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    g.replay()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n * 1e3


for b, c, h, w, f in [(256, 64, 56, 56, 128), (256, 128, 28, 28, 256), (256, 256, 14, 14, 512),
                      (32, 64, 56, 56, 128), (32, 256, 14, 14, 512)]:
    conv = bnn.QConvolution(c, f, (1, 1), (2, 2), (0, 0), rng=rng, domain="dot")
    conv.pack()
    conv.sync_checks = False
    bn = nets.BatchNorm(f, rng)
    xp = PackedNHWC.from_f32(torch.randn((b, c, h, w), device="cuda"))
    oh, ow = conv.output_hw(h, w)
    out = torch.empty((b, f, oh, ow), device="cuda")
    run = lambda: conv.forward_fused(xp, bn, out=out)  # noqa: E731
    mb = out.numel() * 4 / 1e6
    for bits in (0, 1 << 29):
        _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, bits)
        us = t(run)
        print(f"B={b} C={c} {h}x{w} F={f} {'tensor-core' if bits else 'popc pointwise'}: "
              f"{us:.1f} us ({mb:.0f} MB out, {mb / us:.2f} GB/ms)", flush=True)
    _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
