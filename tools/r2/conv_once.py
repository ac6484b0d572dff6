"""Run ResNet-18 binary conv layers once each (for ncu): conv_once.py [algo] [shape idx ...]
shapes: 0 layer1 3x3 C64 F64 (packed out), 1 layer1 conv2 (f32 + residual + packed),
2 layer2 C128 F128 3x3, 3 layer2 conv1 C64->F128 stride 2."""
import sys

import torch

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets  # noqa: E402
from paper_1705_09864_b200.layers import PackedNHWC  # noqa: E402

SHAPES = [(256, 64, 56, 56, 64, 3, 1, 1, "pack"), (256, 64, 56, 56, 64, 3, 1, 1, "res"),
          (256, 128, 28, 28, 128, 3, 1, 1, "pack"), (256, 64, 56, 56, 128, 3, 2, 1, "pack")]
algo = sys.argv[1] if len(sys.argv) > 1 else "auto"
idx = [int(a) for a in sys.argv[2:] if not a.startswith("dbg=")] or [0, 1]
dbg = [int(a[4:]) for a in sys.argv[2:] if a.startswith("dbg=")]
bnn.load_library()
if dbg:
    from paper_1705_09864_b200 import _lib
    _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, dbg[0])
rng = np.random.default_rng(0)
runs = []
for i in idx:
    b, c, h, w, f, k, s, p, kind = SHAPES[i]
    conv = bnn.QConvolution(c, f, (k, k), (s, s), (p, p), rng=rng, domain="dot")
    conv.pack()
    conv.algo = algo
    conv.sync_checks = False
    bn = nets.BatchNorm(f, rng)
    xp = PackedNHWC.from_f32(torch.randn((b, c, h, w), device="cuda"))
    oh, ow = conv.output_hw(h, w)
    res = torch.randn((b, f, oh, ow), device="cuda")
    if kind == "pack":
        runs.append(lambda conv=conv, bn=bn, xp=xp: conv.forward_fused(xp, bn, pack_out=True,
                                                                       f32_out=False))
    else:
        runs.append(lambda conv=conv, bn=bn, xp=xp, res=res: conv.forward_fused(
            xp, bn, residual=res, pack_out=True))
for r in runs:  # warm-up
    r()
torch.cuda.synchronize()
for r in runs:
    r()
torch.cuda.synchronize()
print("ok")
