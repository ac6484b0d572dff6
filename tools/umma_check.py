"""Quick umma-vs-popc cross-check + timing on a few shapes (debug helper)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn

bnn.load_library()
torch.manual_seed(0)
shapes = [(128, 256, 128), (128, 256, 4096), (200, 300, 1000), (1, 1, 1), (256, 25088, 2304),
          (1024, 256, 4096), (4096, 4096, 4096)]
for m, n, k in shapes:
    W = (k + 63) // 64
    a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda").view(torch.uint64)
    b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda").view(torch.uint64)
    if k % 64:
        mask = (1 << (k % 64)) - 1
        a.view(torch.int64)[:, -1] &= mask
        b.view(torch.int64)[:, -1] &= mask
    cp = bnn.xnor_rows_gemm(a, b, k, algo="popc")
    cu = bnn.xnor_rows_gemm(a, b, k, algo="umma")
    torch.cuda.synchronize()
    ok = torch.equal(cp, cu)
    bad = int((cp != cu).sum())
    ts = {}
    for algo in ("popc", "umma"):
        for _ in range(3):
            bnn.xnor_rows_gemm(a, b, k, algo=algo)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(10):
            bnn.xnor_rows_gemm(a, b, k, algo=algo)
        e.record(); e.synchronize()
        ts[algo] = s.elapsed_time(e) / 10
    tops = {a_: 2 * m * n * k / (t * 1e-3) / 1e12 for a_, t in ts.items()}
    print(f"{m}x{n}x{k}: equal={ok} bad={bad} popc {ts['popc']*1e3:.1f}us {tops['popc']:.0f}T  "
          f"umma {ts['umma']*1e3:.1f}us {tops['umma']:.0f}T", flush=True)
    if not ok:
        print(cp[:2, :8]); print(cu[:2, :8])
