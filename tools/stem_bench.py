"""Stem timing (ResNet-18 conv7x7/2 3->64 + BN + ReLU + maxpool, batch 256): the fused
tensor-core kernel, the unfused tensor-core conv + StemPost, and cuDNN f32 (TF32 off)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets  # noqa: E402


def t(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n


bnn.load_library()
import os
from paper_1705_09864_b200 import _lib
if os.environ.get("BNN_STEM_OLD"):
    _lib.call("bnn_debug_set", 4, 16)  # BNN_DEBUG_STEM_BITS bit 4: the gather kernel (bnn_stem.cu)
b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
rng = np.random.default_rng(0)
conv = nets.Conv2d(3, 64, 7, stride=2, pad=3, bias=False, rng=rng)
post = nets.StemPost(64, rng, 3, 2, 1)
x = torch.randn(b, 3, 224, 224, device="cuda")
print("fused ms", t(lambda: post.forward_fused_conv(conv, x)))
print("tc conv ms", t(lambda: conv.forward(x)))
y = conv.forward(x)
print("stempost ms", t(lambda: post.forward(y, bnn.INFER_PACKED)))
conv.engine = "cudnn"
print("cudnn conv ms", t(lambda: conv.forward(x)))
