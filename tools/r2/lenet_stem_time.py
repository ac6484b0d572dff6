"""LeNet's fused float stem (conv5x5 + tanh + maxpool, + sign-pack): tanh per element vs pool first."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets  # noqa: E402

bnn.load_library()
rng = np.random.default_rng(0)
conv = nets.Conv2d(1, 64, 5, pad=2, rng=rng)
x = torch.rand((1024, 1, 28, 28), device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")


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


for pf in (False, True):
    for pack, f32 in ((False, True), (True, False)):
        us = t(lambda: nets._lenet_stem_forward(conv, x, pool_first=pf, pack=pack, f32_out=f32, flags=flags))
        print(f"pool_first={pf} pack={pack} f32_out={f32}: {us:.1f} us", flush=True)

from paper_1705_09864_b200 import _lib  # noqa: E402
for bits in (0, 1, 2, 4, 8, 6, 14):
    _lib.call("bnn_debug_set", 4, bits)  # BNN_DEBUG_STEM_BITS: role ablations (wrong results)
    us = t(lambda: nets._lenet_stem_forward(conv, x, pack=True, f32_out=False, flags=flags))
    print(f"stem_bits={bits}: {us:.1f} us", flush=True)
_lib.call("bnn_debug_set", 4, 0)
for bits in (0, 4, 14):
    _lib.call("bnn_debug_set", 4, bits)
    us = t(lambda: nets._lenet_stem_forward(conv, x, pool_first=True, pack=True, f32_out=False, flags=flags))
    print(f"pool_first stem_bits={bits}: {us:.1f} us", flush=True)
_lib.call("bnn_debug_set", 4, 0)
