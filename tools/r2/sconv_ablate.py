"""Ablations of the small-channel conv kernel (debug bits, wrong results): time per variant."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import _lib, nets  # noqa: E402
from paper_1705_09864_b200.layers import PackedNHWC  # noqa: E402

SHAPES = [(256, 64, 56, 56, 64, 3, 1, 1), (256, 128, 28, 28, 128, 3, 1, 1)]
bnn.load_library()
for (b, c, h, w, f, k, s, p) in SHAPES:
    rng = np.random.default_rng(0)
    conv = bnn.QConvolution(c, f, (k, k), (s, s), (p, p), rng=rng, domain="dot")
    conv.pack()
    conv.sync_checks = False
    bn = nets.BatchNorm(f, rng)
    xp = PackedNHWC.from_f32(torch.randn((b, c, h, w), device="cuda"))
    run = lambda: conv.forward_fused(xp, bn, pack_out=True, f32_out=False)
    for name, bits in [("full", 0), ("no MMA", 1 << 21), ("no epilogue", 2 << 21),
                       ("no TMEM st", 4 << 21), ("no MMA+epi", 3 << 21), ("none", 7 << 21),
                       ("full, try_wait", 1 << 20)]:
        _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, bits)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                run()
        g.replay()
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(True), torch.cuda.Event(True)
        st.record()
        g.replay()
        en.record()
        en.synchronize()
        print(f"C{c} F{f} {h}x{w}: {name:16s} {st.elapsed_time(en) / 10 * 1e3:8.1f} us", flush=True)
    _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
