"""Per-row pipeline timeline of CTA 0 of the stride-2 stem kernel (clock64 cycles)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets, _lib  # noqa: E402

lib = bnn.load_library()
rng = np.random.default_rng(0)
conv = nets.Conv2d(3, 64, 7, stride=2, pad=3, bias=False, rng=rng)
post = nets.StemPost(64, rng, 3, 2, 1)
x = torch.randn(256, 3, 224, 224, device="cuda")
extra = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for _ in range(3):
    post.forward_fused_conv(conv, x)
torch.cuda.synchronize()
tr = torch.zeros(8 * 64, dtype=torch.int64, device="cuda")
lib.bnn_umma_trace(tr.data_ptr())
_lib.call("bnn_debug_set", 4, 8 | extra)
post.forward_fused_conv(conv, x)
torch.cuda.synchronize()
_lib.call("bnn_debug_set", 4, 0)
lib.bnn_umma_trace(None)
t = tr.view(8, 64).cpu().numpy()
t0 = t[t > 0].min()
names = ["ld empty ok", "ld arrived", "mma waits ok", "mma issued", "epi tfull", "epi ld done", "epi row end"]
print("idx  " + " ".join(f"{n:>13s}" for n in names) + "   (cycles after the first event; loader idx = pair, others = conv row)")
for i in range(64):
    print(f"{i:3d}  " + " ".join(f"{int(t[e, i] - t0):13d}" if t[e, i] else " " * 13 for e in range(7)))
print("kernel entry", int(t[7, 0] - t0), "exit", int(t[7, 1] - t0))
print("tfull of rows 64, 72, ...:", [int(v - t0) for v in t[7, 2:] if v])
