"""Run n steps of the ResNet-18 shard a rank executes at world size w (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import bench  # noqa: E402
w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
plan, _ = bench.build_plan("resnet18", "auto", world=w, rank=0)
for _ in range(n):
    plan.run_device()
torch.cuda.synchronize()
print("ok", plan.b)
