"""Per-CTA timeline of one tcgen05 launch (debug): umma_trace.py M N K"""
import sys
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
tr = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
lib.bnn_umma_trace(tr.data_ptr())
torch.cuda.synchronize()
bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
torch.cuda.synchronize()
lib.bnn_umma_trace(None)
t = tr.view(148, 16).cpu().numpy().astype(np.float64)
t0 = t[:, 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us
names = ["start", "setup", "first_stage", "t0_mma", "t0_epi_s", "t0_epi_e", "t1_mma", "t1_epi_s",
         "t1_epi_e", "t2_mma", "t2_epi_s", "t2_epi_e", "exit"]
s_, e_ = torch.cuda.Event(True), torch.cuda.Event(True)
s_.record(); bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out); e_.record(); e_.synchronize()
print(f"{m}x{n}x{k} mode={sys.argv[4] if len(sys.argv) > 4 else 0}: {s_.elapsed_time(e_)*1e3:.1f} us")
for i, nm in enumerate(names):
    col = rel[:, i]
    if np.all(np.isnan(col)): continue
    print(f"{nm:12s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f} us")
