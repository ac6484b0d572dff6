"""Fixed per-launch cost of the engines inside a CUDA graph (back-to-back replays)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
bnn.load_library()

def timed(fn, n=20):
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); g.replay(); e.record(); e.synchronize()
    return s.elapsed_time(e) / n * 1e3

for m, n, k in [(128, 128, 256), (128, 176, 2304), (256, 25088, 2304), (128, 28416, 2304)]:
    W = k // 64
    a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda").view(torch.uint64)
    b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda").view(torch.uint64)
    out = torch.empty((m, n), device="cuda")
    for algo in ("umma", "popc"):
        t = timed(lambda: bnn.xnor_rows_gemm(a, b, k, algo=algo, out=out))
        print(f"{m}x{n}x{k} {algo}: {t:.2f} us  {2*m*n*k/t/1e6:.0f} TOPS")
x = torch.empty(1 << 20, device="cuda")
print(f"empty torch fill 4MB: {timed(lambda: x.fill_(1.0)):.2f} us")
