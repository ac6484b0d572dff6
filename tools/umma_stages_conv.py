"""Per-superstage pipeline timeline of CTA 0 for the c2 conv (debug; BNN_UMMA_DEBUG=16)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import bench
import paper_1705_09864_b200 as bnn

lib = bnn.load_library()
plan, host_x = bench.build_plan("c2", "umma")
plan.pack()
for _ in range(3):
    plan.kernel()
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(10):
    plan.kernel()
e.record(); e.synchronize()
print(f"c2 conv kernel: {s.elapsed_time(e) / 10 * 1e3:.1f} us")
tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
lib.bnn_umma_trace(tr.data_ptr())
torch.cuda.synchronize()
plan.kernel()
torch.cuda.synchronize()
lib.bnn_umma_trace(None)
t = tr[4096:].view(16, 256).cpu().numpy().astype(np.int64)
names = ["B_fetched", "A_empty_ok", "A_done", "A_data", "B_empty_ok", "B_done", "B_data", "mma_full", "mma_commit"]
t0 = t[7, 0]
print("super " + " ".join(f"{x:>10s}" for x in names))
for g in range(0, 24):
    print(f"{g:5d} " + " ".join(f"{(t[ev, g] - t0) if t[ev, g] else -1:10d}" for ev in range(len(names))))
c = tr[:148 * 16].view(148, 16).cpu().numpy().astype(np.float64)
c0 = c[:, 0].min()
print("per-CTA exit (us after first start): max %.1f median %.1f" % (((c[:, 12] - c0) / 1e3).max(), np.median((c[:, 12] - c0) / 1e3)))
print("per-CTA first mma (us): median %.2f" % np.median((c[:, 2] - c0) / 1e3))
