"""End-to-end (pinned host in/out) time of the c2 plan vs host_chunks."""
import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import bench
plan, host_x = bench.build_plan("c2", "auto")
y_host = torch.empty(plan.y.shape, dtype=plan.y.dtype).pin_memory()
for chunks in (1, 2, 4, 8, 16):
    plan.host_chunks = chunks
    for _ in range(3):
        plan.run_host(host_x, y_host)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10):
        plan.run_host(host_x, y_host)
    e1.record(); torch.cuda.synchronize()
    print(f"chunks={chunks}: {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
