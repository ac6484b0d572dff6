"""One-GPU projection of the strong-scaling runs: the step a single rank executes at N = 1, 2, 4, 8
(ResNet-18: 256 / N images; 8192^3 GEMM: N / 8192 columns of B), device-timed by CUDA-graph replay.
No collective is included (networks have none; the GEMM's all-gather is timed by bench.py --gpus N)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import bench  # noqa: E402
from paper_1705_09864_b200.plan import GemmPlan  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


base = None
for world in (1, 2, 4, 8):
    plan, _ = bench.build_plan("resnet18", "auto", world=world, rank=0)
    ms = timed(plan.run_device)
    base = base or ms
    print(f"resnet18 N={world}: {plan.b} images per GPU, {ms:.4f} ms per step -> {256 / ms:.0f}k images/s "
          f"whole job, efficiency {base / (ms * world):.2f}", flush=True)
    del plan
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randint(-2**63, 2**63 - 1, (8192, 128), device="cuda", generator=g).view(torch.uint64)
b = torch.randint(-2**63, 2**63 - 1, (8192, 128), device="cuda", generator=g).view(torch.uint64)
base = None
for world in (1, 2, 4, 8):
    n = 8192 // world
    plan = GemmPlan(a, b[:n].contiguous(), 8192)
    ms = timed(plan.run_device)
    base = base or ms
    print(f"gemm8192 N={world}: shard {n} columns, {ms:.4f} ms -> {2 * 8192**3 / ms / 1e9:.0f} TOPS whole job "
          f"(before the all-gather), efficiency {base / (ms * world):.2f}", flush=True)
