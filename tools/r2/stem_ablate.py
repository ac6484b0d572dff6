"""Stride-2 stem ablation (BNN_DEBUG_STEM_BITS: 1 no input loads, 2 no MMAs, 4 no epilogue work)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets, _lib  # noqa: E402

bnn.load_library()
rng = np.random.default_rng(0)
conv = nets.Conv2d(3, 64, 7, stride=2, pad=3, bias=False, rng=rng)
post = nets.StemPost(64, rng, 3, 2, 1)
x = torch.randn(256, 3, 224, 224, device="cuda")


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n


for bits in [int(a) for a in sys.argv[1:]] or (0, 1, 2, 4, 3, 5, 6, 7):
    _lib.call("bnn_debug_set", 4, bits)
    print(f"dbg={bits} fused {t(lambda: post.forward_fused_conv(conv, x)):.4f} ms  raw {t(lambda: conv.forward(x)):.4f} ms")
_lib.call("bnn_debug_set", 4, 0)
