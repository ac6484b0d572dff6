"""Run the CUDA-core engines once each on one shape (for ncu pipe counters):
engine_once.py M N K [algo ...]  (default algos: popc bmma)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402

m, n, k = map(int, sys.argv[1:4])
algos = sys.argv[4:] or ["popc", "bmma"]
bnn.load_library()
W = (k + 63) // 64
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda", generator=g).view(torch.uint64)
b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda", generator=g).view(torch.uint64)
ref = None
for algo in algos:
    c = bnn.xnor_rows_gemm(a, b, k, algo=algo)
    ref = c if ref is None else ref
    assert torch.equal(c, ref), algo
torch.cuda.synchronize()
print("ok", algos)
