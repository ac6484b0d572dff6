"""Quick umma-vs-popc cross-check + timing on a few shapes (debug helper)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn

lib = bnn.load_library()
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
    out = [f"{m}x{n}x{k}:"]
    cb = bnn.xnor_rows_gemm(a, b, k, algo="bmma")
    torch.cuda.synchronize()
    for _ in range(2):
        bnn.xnor_rows_gemm(a, b, k, algo="bmma")
    s0, e0 = torch.cuda.Event(True), torch.cuda.Event(True)
    s0.record()
    for _ in range(5):
        bnn.xnor_rows_gemm(a, b, k, algo="bmma")
    e0.record(); e0.synchronize()
    tb = s0.elapsed_time(e0) / 5
    for _ in range(2):
        bnn.xnor_rows_gemm(a, b, k, algo="popc")
    s0.record()
    for _ in range(5):
        bnn.xnor_rows_gemm(a, b, k, algo="popc")
    e0.record(); e0.synchronize()
    tp = s0.elapsed_time(e0) / 5
    out.append(f"popc {tp*1e3:.1f}us {2*m*n*k/(tp*1e-3)/1e12:.0f}T bmma equal={torch.equal(cp, cb)} "
               f"{tb*1e3:.1f}us {2*m*n*k/(tb*1e-3)/1e12:.0f}T |")
    for variant in (0, 1):
        lib.bnn_set_umma_variant(variant)
        cu = bnn.xnor_rows_gemm(a, b, k, algo="umma")
        torch.cuda.synchronize()
        ok = torch.equal(cp, cu)
        bad = int((cp != cu).sum())
        for _ in range(3):
            bnn.xnor_rows_gemm(a, b, k, algo="umma")
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(10):
            bnn.xnor_rows_gemm(a, b, k, algo="umma")
        e.record(); e.synchronize()
        t = s.elapsed_time(e) / 10
        out.append(f"v{variant} equal={ok} bad={bad} {t*1e3:.1f}us {2*m*n*k/(t*1e-3)/1e12:.0f}T")
        if not ok:
            out.append(str(cp[:2, :8].tolist()) + " vs " + str(cu[:2, :8].tolist()))
    print("  ".join(out), flush=True)
