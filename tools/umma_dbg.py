"""Per-stage cost with parts of the pipeline disabled (BNN_UMMA_DEBUG bits; wrong outputs)."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
bnn.load_library()
m, n, k = 128, 192 * 148, 36864
W = k // 64
a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda").view(torch.uint64)
b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda").view(torch.uint64)
out = torch.empty((m, n), device="cuda")
for _ in range(2):
    bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(5):
    bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
e.record(); e.synchronize()
t = s.elapsed_time(e) / 5
print(f"dbg={os.environ.get('BNN_UMMA_DEBUG', '0')}: {t*1e3:.1f} us  {t*1e-3*1.9e9/(k/128):.0f} cyc/stage")
