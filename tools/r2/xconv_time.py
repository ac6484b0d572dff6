"""Time the pre-expanded conv engine on C2 / ResNet-18 layer shapes (kernel only, CUDA events)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import _lib  # noqa: E402

bnn.load_library()
bits = int(sys.argv[1]) if len(sys.argv) > 1 else 0
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, bits)
shapes = {"c2": (32, 256, 28, 28, 256), "l3": (256, 256, 14, 14, 256), "l4": (256, 512, 7, 7, 512)}
for name, (b, c, h, w, f) in shapes.items():
    rng = np.random.default_rng(1)
    layer = bnn.QConvolution(c, f, (3, 3), (1, 1), (1, 1), domain="dot")
    layer.weight = rng.standard_normal((f, c, 3, 3)).astype(np.float32)
    layer.pack()
    x = torch.randn((b, c, h, w), device="cuda")
    xw = bnn.pack_nchw(x)
    out = torch.empty((b, f, h, w), device="cuda")
    for algo in ("umma2", "xp"):
        layer.algo = algo
        for _ in range(3):
            layer.forward_packed_words(xw, b, h, w, out=out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()  # (kernel time, not the host's launch / tensor-map cost)
        with torch.cuda.graph(g):
            for _ in range(10):
                layer.forward_packed_words(xw, b, h, w, out=out)
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        g.replay()
        e.record()
        e.synchronize()
        print(f"bits={bits} {name} {algo}: {s.elapsed_time(e) / 10 * 1e3:.1f} us", flush=True)
