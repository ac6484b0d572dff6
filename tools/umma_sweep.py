"""Timing sweep of the tcgen05 engine over K and N (fixed-cost vs per-stage cost)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn

lib = bnn.load_library()
shapes = [(256, 25088, k) for k in (128, 512, 1152, 2304, 4608, 9216)] + \
         [(256, n, 2304) for n in (192 * 74, 192 * 148, 192 * 296, 192 * 592)] + \
         [(128, 192 * 148, k) for k in (512, 2304, 9216, 36864)]
for v in (0, 1):
    lib.bnn_set_umma_variant(v)
    for m, n, k in shapes:
        W = (k + 63) // 64
        a = torch.randint(-2**63, 2**63 - 1, (m, W), device="cuda").view(torch.uint64)
        b = torch.randint(-2**63, 2**63 - 1, (n, W), device="cuda").view(torch.uint64)
        out = torch.empty((m, n), device="cuda")
        for _ in range(3):
            bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                bnn.xnor_rows_gemm(a, b, k, algo="umma", out=out)
        g.replay(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); g.replay(); e.record(); e.synchronize()
        t = s.elapsed_time(e) / 10
        bn = 256 if v == 0 else 192
        tiles = ((m + 127) // 128) * ((n + bn - 1) // bn)
        stages = (k + 127) // 128
        print(f"v{v} {m}x{n}x{k}: {t*1e3:8.1f} us  {2*m*n*k/(t*1e-3)/1e12:7.0f} TOPS  tiles={tiles} "
              f"stages/tile={stages} cyc/stage~{t*1e-3*1.9e9/(stages*((tiles+147)//148)):.0f}", flush=True)
