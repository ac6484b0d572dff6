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
tr = torch.zeros(4096 + 2 * 4096, dtype=torch.int64, device="cuda")
lib.bnn_umma_trace(tr.data_ptr())
torch.cuda.synchronize()
bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
torch.cuda.synchronize()
lib.bnn_umma_trace(None)
t_all = tr[4096:].view(2, 16, 256).cpu().numpy().astype(np.int64)
t = t_all[0]
names = ["tma_issue", "A_empty_ok", "A_done", "A_data", "B_empty_ok", "B_done", "B_data", "mma_full", "mma_commit"]
t0 = t[7, 0]
ns = (k + 127) // 128
print("stage " + " ".join(f"{x:>10s}" for x in names))
for g in list(range(0, min(ns, 40))) + list(range(100, min(ns, 120))):
    print(f"{g:5d} " + " ".join(f"{(t[e, g] - t0) if t[e, g] else -1:10d}" for e in range(len(names))))
t0b = t[7, 0]
print("block 1 (peer) rows, same origin (ns):")
for g in range(0, 12):
    print(f"{g:5d} " + " ".join(f"{(t_all[1][ev, g] - t0b) if t_all[1][ev, g] else -1:10d}" for ev in range(len(names))))
d = np.diff(t[7, 20:min(ns, 250)])
print("mma_full cadence (cycles): median", np.median(d), "mean", d.mean())
