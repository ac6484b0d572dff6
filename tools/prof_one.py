"""Run one hot-path kernel a few times (for ncu): prof_one.py conv|gemm M N K [variant]."""
import sys
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import paper_1705_09864_b200 as bnn

lib = bnn.load_library()
what = sys.argv[1]
variant = int(sys.argv[5]) if len(sys.argv) > 5 else 1
if what == "conv":
    import bench
    plan, _ = bench.build_plan("c2", "auto")
    for _ in range(3):
        plan.run_device()
else:
    m, n, k = map(int, sys.argv[2:5])
    W = (k + 63) // 64
    a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda").view(torch.uint64)
    b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda").view(torch.uint64)
    for _ in range(3):
        bnn.xnor_rows_gemm(a, b, k, algo=f"umma{variant}")
torch.cuda.synchronize()
print("ok")
