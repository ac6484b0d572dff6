"""Per-superstage pipeline timeline of CTA 0 of one bench workload's tcgen05 kernel
(default c2; `python tools/umma_stages_conv.py c1`; debug trace buffer)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import bench
import paper_1705_09864_b200 as bnn

lib = bnn.load_library()
from paper_1705_09864_b200 import _lib  # noqa: E402
_lib.call("bnn_debug_set", _lib.DEBUG_UMMA_BITS, 16)  # per-superstage stamps of CTAs 0, 1
WL = sys.argv[1] if len(sys.argv) > 1 else "c2"
plan, host_x = bench.build_plan(WL, "umma")
plan.pack()
for _ in range(3):
    plan.kernel()
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(10):
    plan.kernel()
e.record(); e.synchronize()
print(f"{WL} kernel (eager launches): {s.elapsed_time(e) / 10 * 1e3:.1f} us")
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    plan.kernel()
torch.cuda.synchronize()
with torch.cuda.graph(g):
    for _ in range(10):
        plan.kernel()
g.replay(); torch.cuda.synchronize()
s.record(); g.replay(); e.record(); e.synchronize()
print(f"{WL} kernel (graph, back to back): {s.elapsed_time(e) / 10 * 1e3:.1f} us")
tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
lib.bnn_umma_trace(tr.data_ptr())
torch.cuda.synchronize()
plan.kernel()
torch.cuda.synchronize()
lib.bnn_umma_trace(None)
t = tr[4096:].view(16, 256).cpu().numpy().astype(np.int64)
names = ["tma_issue", "A_empty_ok", "A_done", "A_data", "B_empty_ok", "B_done", "B_data", "mma_full", "mma_commit"] + [f"w{i}_done" for i in range(1, 8)]
t0 = t[7, 0]
print("super " + " ".join(f"{x:>10s}" for x in names))
for g in range(0, int(sys.argv[2]) if len(sys.argv) > 2 else 24):
    print(f"{g:5d} " + " ".join(f"{(t[ev, g] - t0) if t[ev, g] else -1:10d}" for ev in range(len(names))))
c = tr[:148 * 16].view(148, 16).cpu().numpy().astype(np.float64)
c = c[c[:, 0] > 0]  # CTAs of the launch (grid may be < 148)
c0 = c[:, 0].min()
print("per-CTA exit (us after first start): max %.1f median %.1f" % (((c[:, 12] - c0) / 1e3).max(), np.median((c[:, 12] - c0) / 1e3)))
print("per-CTA first mma (us): median %.2f" % np.median((c[:, 2] - c0) / 1e3))
print("tile 0: MMA done median %.2f, epilogue start median %.2f, epilogue end median %.2f (us)" % tuple(np.median((c[:, j] - c0) / 1e3) for j in (3, 4, 5)))
st = (c[:, 0] - c0) / 1e3
print("CTA start (us): min %.2f median %.2f max %.2f; setup done median %.2f" % (st.min(), np.median(st), st.max(), np.median((c[:, 1] - c0) / 1e3)))

# launch / teardown gaps: stamp -> conv -> stamp in one graph
st = torch.zeros(4, dtype=torch.int64, device="cuda")
from paper_1705_09864_b200 import _lib
tr.zero_()
lib.bnn_umma_trace(tr.data_ptr())
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    _lib.call("bnn_debug_stamp", st.data_ptr(), _lib.stream_ptr())
    plan.kernel()
    _lib.call("bnn_debug_stamp", st.data_ptr() + 8, _lib.stream_ptr())
lib.bnn_umma_trace(None)
g2.replay(); torch.cuda.synchronize()
c = tr[:148 * 16].view(148, 16).cpu().numpy().astype(np.int64)
c = c[c[:, 0] > 0]
s0, s1 = [int(v) for v in st[:2].cpu()]
print("stamp0 -> first CTA start %.2f us, -> last CTA start %.2f, last CTA exit -> stamp1 %.2f us, total %.2f us"
      % ((c[:, 0].min() - s0) / 1e3, (c[:, 0].max() - s0) / 1e3, (s1 - c[:, 12].max()) / 1e3, (s1 - s0) / 1e3))
d = (c[:, 13] - c[:, 12]) / 1e3
print("per-CTA trace12 -> dealloc done: min %.2f median %.2f max %.2f us; last dealloc -> stamp1 %.2f us"
      % (d.min(), np.median(d), d.max(), (s1 - c[:, 13].max()) / 1e3))
print("last trace12 %.2f, last dealloc %.2f (us after first start)" % ((c[:, 12].max() - c[:, 0].min()) / 1e3, (c[:, 13].max() - c[:, 0].min()) / 1e3))
