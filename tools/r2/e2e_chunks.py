"""End-to-end (pinned host buffers) step time per batch-slice count of the pipelined
run_host: e2e_chunks.py c2|resnet18|c1 [chunks ...]."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import bench  # noqa: E402

name = sys.argv[1]
# an integer = equal slices; a comma list = taper weights
chunks = sys.argv[2:] or ["1", "2", "4", "8"]
plan, host_x = bench.build_plan(name, "auto")
y_host = torch.empty(plan.y.shape, dtype=plan.y.dtype).pin_memory()
for c in chunks:
    if "," in c:
        plan.host_taper = [int(v) for v in c.split(",")]
    else:
        plan.host_taper, plan.host_chunks = None, int(c)
    for _ in range(3):
        plan.run_host(host_x, y_host)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(10):
        plan.run_host(host_x, y_host)
    e.record()
    e.synchronize()
    print(f"{name} chunks {c:>20s}: {s.elapsed_time(e) / 10:.3f} ms per e2e step", flush=True)
