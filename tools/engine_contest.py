"""Engine contest (north star: LOP3/POPC vs b1 mma.sync vs tcgen05): bit-exactness against
the POPC engine and graph-timed TOPS (2MNK/s) per shape.  Prints a markdown table."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn

lib = bnn.load_library()
shapes = [(1024, 256, 4096), (256, 25088, 2304), (4096, 4096, 4096), (8192, 8192, 8192),
          (4096, 4096, 65536)]
engines = [("popc", "popc", None), ("bmma (b1 mma.sync)", "bmma", None),
           ("tcgen05 i8, SMEM A (v0)", "umma", 0), ("tcgen05 i8, TMEM A (v1)", "umma", 1),
           ("tcgen05 mxf4 (v2)", "umma", 2), ("tcgen05 mxf4, TMEM A (v3)", "umma", 3)]


def timed(fn, reps):
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.replay(); e.record(); e.synchronize()
    return s.elapsed_time(e) / reps


print("| shape (M x N x K) | " + " | ".join(n for n, _, _ in engines) + " |")
print("|---" * (len(engines) + 1) + "|")
for m, n, k in shapes:
    W = (k + 63) // 64
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda", generator=g).view(torch.uint64)
    b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda", generator=g).view(torch.uint64)
    out = torch.empty((m, n), device="cuda")
    ref = bnn.xnor_rows_gemm(a, b, k, algo="popc")
    cells = []
    for name, algo, var in engines:
        if var is not None:
            algo = f"umma{var}"
        big = 2 * m * n * k
        if algo != "umma" and big > 3e12:
            cells.append("—")
            continue
        c = bnn.xnor_rows_gemm(a, b, k, algo=algo)
        ok = torch.equal(c, ref)
        reps = max(1, min(20, int(2e13 / big)))
        t = timed(lambda: bnn.xnor_rows_gemm(a, b, k, algo=algo, out=out), reps)
        cells.append(f"{big / (t * 1e-3) / 1e12:.0f}{'' if ok else ' (MISMATCH)'}")
    print(f"| {m} x {n} x {k} | " + " | ".join(cells) + " |", flush=True)
