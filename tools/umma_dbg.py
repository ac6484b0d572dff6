"""Per-stage cost with parts of the pipeline disabled (BNN_UMMA_DEBUG bits; wrong outputs).
usage: umma_dbg.py [M N K]  (default 128 x 192*148 x 36864); timed as a CUDA graph."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
bnn.load_library()
m, n, k = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (128, 192 * 148, 36864)
W = k // 64
a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda").view(torch.uint64)
b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda").view(torch.uint64)
out = torch.empty((m, n), device="cuda")
side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(10):
        bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
g.replay(); torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); g.replay(); e.record(); e.synchronize()
t = s.elapsed_time(e) / 10
print(f"{m}x{n}x{k} dbg={os.environ.get('BNN_UMMA_DEBUG', '0')}: {t*1e3:.1f} us  {2*m*n*k/t/1e9:.0f} TOPS")
