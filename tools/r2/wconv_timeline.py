"""Per-tile pipeline timeline of CTA 0 of the shifted-window conv kernel (clock64 cycles):
wconv_timeline.py [shape idx] [extra debug bits << 21]."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets, _lib  # noqa: E402
from paper_1705_09864_b200.layers import PackedNHWC  # noqa: E402

SHAPES = [(256, 64, 56, 56, 64, 3, 1, 1, "pack"), (256, 64, 56, 56, 64, 3, 1, 1, "res"), (32, 256, 28, 28, 256, 3, 1, 1, "plain"),
          (256, 128, 28, 28, 128, 3, 1, 1, "pack"), (256, 128, 28, 28, 128, 3, 1, 1, "res")]
i = int(sys.argv[1]) if len(sys.argv) > 1 else 0
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw_bits = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # e.g. 262144: bit 18, C >= 256 on this kernel
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
    (lambda: conv.forward_fused(xp)) if kind == "plain" else \
    (lambda: conv.forward_fused(xp, bn, residual=res, pack_out=True))
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, raw_bits)
for _ in range(3):
    run()
torch.cuda.synchronize()
tr = torch.zeros(8 * 64, dtype=torch.int64, device="cuda")
lib.bnn_umma_trace(tr.data_ptr())
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 16 | (extra << 21) | raw_bits)
run()
torch.cuda.synchronize()
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
lib.bnn_umma_trace(None)
t = tr.view(8, 64).cpu().numpy()
t0 = int(t[7, 0])
print("prologue stamps (after alloc+pdl wait, after weights, after params/sf):", [int(t[7, k]) - t0 for k in (3, 6, 4, 5)], '(2nd = after the expansion loop)')
print(f"shape {SHAPES[i]}: entry 0, prologue done {int(t[7, 1]) - t0}, exit {int(t[7, 2]) - t0} cycles")
names = ["ld bempty ok", "ld arrived", "mma tempty ok", "mma committed", "epi coords", "epi tfull", "epi end"]
print("idx  " + " ".join(f"{n:>13s}" for n in names) + "   (loader idx = item, others = tile; epilogue = warp 0 / 4 by parity)")
for j in range(64):
    if not any(t[e, j] for e in range(7)):
        break
    print(f"{j:3d}  " + " ".join(f"{int(t[e, j]) - t0:13d}" if t[e, j] else " " * 13 for e in range(7)))
