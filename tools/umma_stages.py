"""Per-stage pipeline timeline of CTA 0 (debug; BNN_UMMA_DEBUG=16): umma_stages.py M N K"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn

lib = bnn.load_library()
m, n, k = map(int, sys.argv[1:4])
W = (k + 63) // 64
a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda").view(torch.uint64)
b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda").view(torch.uint64)
out = torch.empty((m, n), device="cuda")
for _ in range(3):
    bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
lib.bnn_umma_trace(tr.data_ptr())
torch.cuda.synchronize()
bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
torch.cuda.synchronize()
lib.bnn_umma_trace(None)
t = tr[4096:].view(16, 256).cpu().numpy().astype(np.int64)
names = ["tma_issue", "A_empty_ok", "A_done", "A_data", "B_empty_ok", "B_done", "B_data", "mma_full", "mma_commit"]
t0 = t[7, 0]
ns = (k + 127) // 128
print("stage " + " ".join(f"{x:>10s}" for x in names))
for g in list(range(0, min(ns, 40))) + list(range(100, min(ns, 120))):
    print(f"{g:5d} " + " ".join(f"{(t[e, g] - t0) if t[e, g] else -1:10d}" for e in range(len(names))))
d = np.diff(t[7, 20:min(ns, 250)])
print("mma_full cadence (cycles): median", np.median(d), "mean", d.mean())
