"""Large binary GEMM: single-CTA kind::mxf4 route vs the 2-CTA pair route (BNN_DEBUG_PAIR_KW32)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import _lib  # noqa: E402

bnn.load_library()
sizes = [int(a) for a in sys.argv[1:]] or [8192]
for n in sizes:
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randint(-2**63, 2**63 - 1, (n, n // 64), device="cuda", generator=g).view(torch.uint64)
    b = torch.randint(-2**63, 2**63 - 1, (n, n // 64), device="cuda", generator=g).view(torch.uint64)
    out = torch.empty((n, n), device="cuda")
    ref = None
    for pair, wide in ((0, 0), (0, 1), (1, 0), (1, 1)):
        _lib.call("bnn_debug_set", _lib.DEBUG_PAIR_KW32, 1 if pair else 0)
        _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 16384 if wide else 0)
        run = lambda: bnn.xnor_rows_gemm(a, b, n, algo="umma", out=out)  # noqa: E731
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(5):
            run()
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / 5
        chk = float(out.double().sum().item())
        if ref is None:
            ref = chk
        print(f"{n}^3 pair={pair} wide={wide}: {ms:.4f} ms  {2 * n**3 / ms / 1e9:.0f} TOPS  checksum equal {chk == ref}", flush=True)
    _lib.call("bnn_debug_set", _lib.DEBUG_PAIR_KW32, 0)
    _lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
