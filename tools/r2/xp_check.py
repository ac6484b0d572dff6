"""Pre-expanded 2-CTA engine (bnn_xnor_gemm_ws, algo "xp") against the packed tcgen05 engine:
bit-exact comparison on small / ragged / large shapes, then timings (CUDA events)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import _lib  # noqa: E402

bnn.load_library()
mode = sys.argv[1] if len(sys.argv) > 1 else "check"


def words(rows, k, seed, pad):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = (k + 63) // 64
    t = torch.randint(-2**63, 2**63 - 1, (rows, w), device="cuda", generator=g)
    if k % 64:
        mask = (1 << (k % 64)) - 1
        if pad:
            t[:, -1] |= ~mask  # pad fill 1 past K
        else:
            t[:, -1] &= mask
    return t.view(torch.uint64)


if mode == "check":
    shapes = [(256, 224, 256), (128, 96, 64), (300, 500, 1000), (257, 225, 257), (1024, 1024, 1024),
              (512, 3000, 4160), (2048, 2048, 8192), (4096, 4096, 4096)]
    bad = 0
    for (m, n, k) in shapes:
        for dom in (_lib.POPCOUNT, _lib.DOT):
            for tr in (False, True):
                a, b = words(m, k, 1, 0), words(n, k, 2, 1)
                ref = bnn.xnor_rows_gemm(a, b, k, a_pad=0, b_pad=1, domain=dom, algo="umma", transpose_out=tr)
                got = bnn.xnor_rows_gemm(a, b, k, a_pad=0, b_pad=1, domain=dom, algo="xp", transpose_out=tr)
                torch.cuda.synchronize()
                ok = torch.equal(ref, got)
                bad += not ok
                print(f"{m}x{n}x{k} dom={dom} tr={tr}: {'ok' if ok else 'MISMATCH ' + str(int((ref != got).sum()))}",
                      flush=True)
                if not ok:
                    d = (ref != got).nonzero()[:5]
                    print(d.tolist(), ref[ref != got][:5].tolist(), got[ref != got][:5].tolist())
    sys.exit(1 if bad else 0)

if mode == "bn":  # tile-N sweep of the pre-expanded engine (debug knob)
    m = n = k = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    a, b = words(m, k, 1, 0), words(n, k, 2, 0)
    out = torch.empty((m, n), device="cuda")
    bits = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, bits)
    print("debug bits", bits)
    for bn in (128, 160, 192, 224):
        _lib.call("bnn_debug_set", _lib.DEBUG_FP4_BN, bn)
        for _ in range(3):
            bnn.xnor_rows_gemm(a, b, k, algo="xp", out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(10):
            bnn.xnor_rows_gemm(a, b, k, algo="xp", out=out)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / 10
        print(f"{m}^3 BN={bn}: {ms:.4f} ms {2 * m * n * k / ms / 1e9:.0f} TOPS", flush=True)
    _lib.call("bnn_debug_set", _lib.DEBUG_FP4_BN, 0)
    _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
    sys.exit(0)

sizes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[2:]] or [(8192, 8192, 8192)]
for (m, n, k) in sizes:
    a, b = words(m, k, 1, 0), words(n, k, 2, 0)
    out = torch.empty((m, n), device="cuda")
    ref = None
    for algo in ("umma", "xp"):
        run = lambda: bnn.xnor_rows_gemm(a, b, k, algo=algo, out=out)  # noqa: E731
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(10):
            run()
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / 10
        chk = float(out.double().sum().item())
        if ref is None:
            ref = chk
        print(f"{m}x{n}x{k} {algo}: {ms:.4f} ms  {2 * m * n * k / ms / 1e9:.0f} TOPS  checksum equal {chk == ref}",
              flush=True)
