"""Per-layer timing of the binary conv epilogue variants (CUDA events, warm L2).

python tools/layer_bench.py [B C H W F k stride pad] ...
Variants: f32 (BN), f32+res, pack-only (BN, sign-pack), pack+f32+res.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets  # noqa: E402
from paper_1705_09864_b200.layers import PackedNHWC  # noqa: E402

SHAPES = [(256, 64, 56, 56, 64, 3, 1, 1), (256, 64, 56, 56, 128, 3, 2, 1),
          (256, 64, 56, 56, 128, 1, 2, 0),
          (256, 128, 28, 28, 128, 3, 1, 1), (256, 128, 28, 28, 256, 3, 2, 1),
          (256, 256, 14, 14, 256, 3, 1, 1), (256, 512, 7, 7, 512, 3, 1, 1),
          (32, 256, 28, 28, 256, 3, 1, 1)]


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    bnn.load_library()
    shapes = SHAPES
    if len(sys.argv) > 1:
        v = [int(a) for a in sys.argv[1:]]
        shapes = [tuple(v[i:i + 8]) for i in range(0, len(v), 8)]
    rng = np.random.default_rng(0)
    for (b, c, h, w, f, k, s, p) in shapes:
        conv = bnn.QConvolution(c, f, (k, k), (s, s), (p, p), rng=rng, domain="dot")
        conv.pack()
        conv.sync_checks = False
        bn = nets.BatchNorm(f, rng)
        x = torch.randn((b, c, h, w), device="cuda")
        xp = PackedNHWC.from_f32(x)
        oh, ow = conv.output_hw(h, w)
        res = torch.randn((b, f, oh, ow), device="cuda")
        out = torch.empty_like(res)
        for algo in ("auto", "umma4"):
            conv.algo = algo
            t = {
                "f32": timeit(lambda: conv.forward_fused(xp, bn, out=out)),
                "f32+res": timeit(lambda: conv.forward_fused(xp, bn, residual=res, out=out)),
                "pack": timeit(lambda: conv.forward_fused(xp, bn, pack_out=True, f32_out=False)),
                "pack+f32+res": timeit(lambda: conv.forward_fused(xp, bn, residual=res, out=out,
                                                                  pack_out=True)),
            }
            ops = 2 * f * b * oh * ow * c * k * k
            print(f"B{b} C{c} {h}x{w} F{f} k{k} s{s} [{algo}]: " +
                  "  ".join(f"{n} {us:7.1f}us ({ops / us / 1e6:6.0f} TOPS)" for n, us in t.items()),
                  flush=True)


if __name__ == "__main__":
    main()
