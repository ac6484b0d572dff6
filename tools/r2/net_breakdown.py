"""Per-launch device time of one ResNet-18 (or LeNet) step (NetPlan.kernel_breakdown)."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
plan, _ = bench.build_plan(name, "auto")
plan.kernel_breakdown()
tot = 0.0
for n, ms, ops in plan.kernel_breakdown():
    tot += ms
    print(f"{n:42s} {ms * 1e3:9.1f} us  {ops / (ms * 1e-3) / 1e12 if ops else 0:8.0f} TOPS")
print(f"total {tot * 1e3:.1f} us")
