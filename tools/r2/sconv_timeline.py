"""Per-tile pipeline timeline of CTA 0 of the small-channel conv kernel (debug trace):
sconv_timeline.py [shape idx] (conv_once.py shapes)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools/r2")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import _lib, nets  # noqa: E402
from paper_1705_09864_b200.layers import PackedNHWC  # noqa: E402

SHAPES = [(256, 64, 56, 56, 64, 3, 1, 1, "pack"), (256, 64, 56, 56, 64, 3, 1, 1, "res"),
          (256, 128, 28, 28, 128, 3, 1, 1, "pack"), (256, 64, 56, 56, 128, 3, 2, 1, "pack")]
i = int(sys.argv[1]) if len(sys.argv) > 1 else 0
lib = bnn.load_library()
b, c, h, w, f, k, s, p, kind = SHAPES[i]
rng = np.random.default_rng(0)
conv = bnn.QConvolution(c, f, (k, k), (s, s), (p, p), rng=rng, domain="dot")
conv.pack()
conv.sync_checks = False
bn = nets.BatchNorm(f, rng)
xp = PackedNHWC.from_f32(torch.randn((b, c, h, w), device="cuda"))
oh, ow = conv.output_hw(h, w)
res = torch.randn((b, f, oh, ow), device="cuda")
run = (lambda: conv.forward_fused(xp, bn, pack_out=True, f32_out=False)) if kind == "pack" else \
    (lambda: conv.forward_fused(xp, bn, residual=res, pack_out=True))
for _ in range(3):
    run()
torch.cuda.synchronize()
tr = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 16 | extra)
lib.bnn_umma_trace(tr.data_ptr())
st = torch.zeros(2, dtype=torch.int64, device="cuda")
g = torch.cuda.CUDAGraph()  # one graph (stamp, conv, stamp): no host gaps
with torch.cuda.graph(g):
    _lib.call("bnn_debug_stamp", st.data_ptr(), _lib.stream_ptr())
    run()
    _lib.call("bnn_debug_stamp", st.data_ptr() + 8, _lib.stream_ptr())
g.replay()
torch.cuda.synchronize()
lib.bnn_umma_trace(None)
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
t = tr.view(16, 64).cpu().numpy().astype(np.int64)
t0 = int(st[0].item())
names = ["band issue", "exp band ok", "exp done", "mma start", "mma commit", "epi start", "epi end",
         "mma top", "mma tempty", "mma issued", "mma commit0", "exp loaded", "exp stored", "exp arrived"]
print(f"shape {SHAPES[i]}: kernel span {(int(st[1].item()) - t0) / 1e3:.1f} us")
print("tile " + " ".join(f"{n:>11s}" for n in names) + "   (us after the launch stamp)")
for it in range(64):
    if t[0, it] == 0:
        break
    print(f"{it:4d} " + " ".join(f"{(t[e, it] - t0) / 1e3:11.2f}" if t[e, it] else " " * 11
                                 for e in range(14)))
