"""LeNet's QFullyConnected (3136 -> 1000, batch 1024) with a 49-word row pitch (odd: cp.async
kind::i8 route) against a 50-word pitch (16-byte aligned rows: TMA kind::mxf4 route)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402

bnn.load_library()
m, n, k = 1000, 1024, 3136
g = torch.Generator(device="cuda").manual_seed(3)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    gr.replay()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps * 1e3


outs = []
for pitch in (49, 50):
    a = torch.zeros((m, pitch), dtype=torch.int64, device="cuda")
    b = torch.zeros((n, pitch), dtype=torch.int64, device="cuda")
    ga = torch.Generator(device="cuda").manual_seed(1)
    a[:, :49] = torch.randint(-2**63, 2**63 - 1, (m, 49), device="cuda", generator=ga)
    b[:, :49] = torch.randint(-2**63, 2**63 - 1, (n, 49), device="cuda", generator=ga)
    av, bv = a.view(torch.uint64)[:, :49], b.view(torch.uint64)[:, :49]
    out = torch.empty((n, m), device="cuda")
    run = lambda: bnn.xnor_rows_gemm(av, bv, k, out=out, transpose_out=True)  # noqa: E731
    print(f"pitch {pitch}: {t(run):.1f} us", flush=True)
    outs.append(out.clone())
print("identical:", torch.equal(outs[0], outs[1]))
