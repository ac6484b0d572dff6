"""Kernel-time breakdown of one network step (torch.profiler / CUPTI)."""
import sys
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import bench

name = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
plan, _ = bench.build_plan(name, "auto")
for _ in range(3):
    plan.run_device()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    plan.run_device()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
