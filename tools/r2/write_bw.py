"""Pure HBM write / copy bandwidth at the sizes of the ResNet-18 f32 activation tensors
(cudaMemsetAsync and a device copy, CUDA-graph timed, L2-cold between sizes is not attempted:
tensors below 126 MB partly stay in L2)."""
import torch


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    g.replay()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n * 1e3


for mb in (26, 51, 103, 205, 410, 1024):
    n = mb * 1000 * 1000 // 4
    a = torch.empty(n, device="cuda")
    b = torch.empty(n, device="cuda")
    us_w = t(lambda: a.zero_())
    us_f = t(lambda: a.fill_(1.5))
    us_c = t(lambda: b.copy_(a))
    print(f"{mb} MB: memset {us_w:.1f} us ({mb / us_w:.2f} TB/s), fill {us_f:.1f} us ({mb / us_f:.2f} TB/s), "
          f"copy {us_c:.1f} us ({2 * mb / us_c:.2f} TB/s r+w)", flush=True)
