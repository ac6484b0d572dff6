"""Phase timeline (clock64 of CTA 0) of the cluster split-K GEMM kernel on config 1."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import _lib  # noqa: E402

lib = bnn.load_library()
m, n, k = 1024, 256, 4096
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randint(-2**63, 2**63 - 1, (m, k // 64), device="cuda", generator=g).view(torch.uint64)
b = torch.randint(-2**63, 2**63 - 1, (n, k // 64), device="cuda", generator=g).view(torch.uint64)
out = torch.empty((n, m), device="cuda")
run = lambda: bnn.xnor_rows_gemm(a, b, k, algo="umma", domain=_lib.DOT, out=out, transpose_out=True)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
tr = torch.zeros(16, dtype=torch.int64, device="cuda")
lib.bnn_umma_trace(tr.data_ptr())
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 16)
run()
torch.cuda.synchronize()
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 0)
lib.bnn_umma_trace(None)
t = tr.cpu().numpy()
names = ["entry", "setup done", "operands expanded", "MMAs done", "partials in SMEM", "cluster sync",
         "reduced + stored", "exit sync"]
for i, nm in enumerate(names):
    print(f"{nm:>20s} {int(t[i] - t[0]):8d} cycles")
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    for _ in range(20):
        run()
gr.replay()
torch.cuda.synchronize()
s.record()
gr.replay()
e.record()
e.synchronize()
print(f"graph-timed (warm L2): {s.elapsed_time(e) / 20 * 1e3:.2f} us per launch")
