"""Run N network steps (for an ncu launch list of one step): net_steps.py lenet|resnet18 N."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
plan, _ = bench.build_plan(name, "auto")
for _ in range(n):
    plan.run_device()
torch.cuda.synchronize()
print("ok")
