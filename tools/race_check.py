"""Repeat large GEMMs on the tcgen05 engine and compare with the CUDA-core engine (race hunt)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
from paper_1705_09864_b200 import _lib
bnn.load_library()
shapes = [(8192, 8192, 8192), (4096, 4096, 4096), (256, 25088, 2304), (4096, 4096, 65536)]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for m, n, k in shapes:
    W = k // 64
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda", generator=g).view(torch.uint64)
    b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda", generator=g).view(torch.uint64)
    ref = bnn.xnor_rows_gemm(a, b, k, algo="popc")
    for v in (0, 1, 2):
        _lib.call("bnn_set_umma_variant", v)
        bad = 0
        for r in range(reps):
            c = bnn.xnor_rows_gemm(a, b, k, algo="umma")
            nb = int((c != ref).sum())
            if nb:
                bad += 1
                idx = (c != ref).nonzero()[:4].tolist()
                print(f"  {m}x{n}x{k} v{v} rep {r}: {nb} bad, first {idx}", flush=True)
        print(f"{m}x{n}x{k} v{v}: {bad}/{reps} bad runs", flush=True)
