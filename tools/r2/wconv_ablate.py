"""Shifted-window conv (bnn_wconv.cu) timing per ablation (debug bits 21..23 of BNN_DEBUG_UMMA_BITS:
1 no MMAs, 2 no epilogue work, 4 no band loads); bit 19 = the previous kernel (bnn_sconv.cu)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets, _lib  # noqa: E402
from paper_1705_09864_b200.layers import PackedNHWC  # noqa: E402

SHAPES = [(256, 64, 56, 56, 64, 3, 1, 1, "pack"), (256, 64, 56, 56, 64, 3, 1, 1, "res"),
          (256, 128, 28, 28, 128, 3, 1, 1, "pack"), (256, 128, 28, 28, 128, 3, 1, 1, "res"),
          (1, 64, 56, 56, 64, 3, 1, 1, "pack"), (6, 64, 56, 56, 64, 3, 1, 1, "pack"),
          (32, 256, 28, 28, 256, 3, 1, 1, "plain"), (256, 256, 14, 14, 256, 3, 1, 1, "pack"),
          (256, 256, 14, 14, 256, 3, 1, 1, "bnf32"), (256, 512, 7, 7, 512, 3, 1, 1, "pack"),
          (256, 512, 7, 7, 512, 3, 1, 1, "bnf32"), (256, 256, 14, 14, 256, 3, 1, 1, "res"),
          (256, 256, 14, 14, 256, 3, 1, 1, "respk"), (1024, 64, 14, 14, 64, 5, 1, 2, "pack")]
bnn.load_library()
import os
BIG = (1 << 17) if os.environ.get("WCONV_NOBIG") else 0  # C >= 256 back on the general engine
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


idx = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 2, 3]
bits = [int(a) for a in sys.argv[2:]] or [0, 1, 2, 4, 3, 6, 7]
for i in idx:
    b, c, h, w, f, k, s, p, kind = SHAPES[i]
    conv = bnn.QConvolution(c, f, (k, k), (s, s), (p, p), rng=rng, domain="dot")
    conv.pack()
    conv.sync_checks = False
    bn = nets.BatchNorm(f, rng)
    xp = PackedNHWC.from_f32(torch.randn((b, c, h, w), device="cuda"))
    oh, ow = conv.output_hw(h, w)
    res = torch.randn((b, f, oh, ow), device="cuda")
    if kind == "pack":
        run = lambda: conv.forward_fused(xp, bn, pack_out=True, f32_out=False)  # noqa: E731
    elif kind == "plain":
        run = lambda: conv.forward_fused(xp)  # noqa: E731
    elif kind == "bnf32":
        run = lambda: conv.forward_fused(xp, bn)  # noqa: E731
    elif kind == "respk":
        run = lambda: conv.forward_fused(xp, bn, residual=res, pack_out=True, f32_out=False)  # noqa: E731
    else:
        run = lambda: conv.forward_fused(xp, bn, residual=res, pack_out=True)  # noqa: E731
    for d in bits:
        v = (1 << 19) if d < 0 else ((d << 21) | BIG)
        _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, v)
        print(f"shape {i} {kind} dbg={d}: {t(run):.1f} us", flush=True)
    _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
