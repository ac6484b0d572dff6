"""Time the NCHW sign+pack kernel on the C2 input vs torch reductions (CUDA graphs, no CPU gaps)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
from paper_1705_09864_b200 import _lib

lib = bnn.load_library()
x = torch.randn(32, 256, 28, 28, device="cuda")
out = torch.empty(32, 28, 28, 4, dtype=torch.uint64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
y = torch.empty_like(x)
flush = torch.empty(64 * 1024 * 1024, device="cuda")

def pack():
    lib.bnn_pack_nchw_f32(x.data_ptr(), 32, 256, 28, 28, out.data_ptr(), 0, flags.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)

def graph_time(fn, reps=20, fl=False):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    tot = 0.0
    for _ in range(reps):
        if fl: flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); g.replay(); b.record(); b.synchronize(); tot += a.elapsed_time(b)
    return tot / reps * 1e3

for fl in (False, True):
    tp = graph_time(pack, fl=fl)
    tc = graph_time(lambda: y.copy_(x), fl=fl)
    ts = graph_time(lambda: torch.sum(x, dim=1, out=None), fl=fl)
    print(f"flush={fl}: pack {tp:.1f} us ({x.numel()*4/tp/1e3:.0f} GB/s read)  copy {tc:.1f} us "
          f"({2*x.numel()*4/tc/1e3:.0f} GB/s)  sum(dim1) {ts:.1f} us ({x.numel()*4/ts/1e3:.0f} GB/s)")
