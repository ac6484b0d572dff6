"""pack_nchw alone: warm (L2-resident input) and cold (input flushed) timings, graph-launched."""
import sys, torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
lib = bnn.load_library()
x = torch.randn(32, 256, 28, 28, device="cuda")
out = torch.empty(32, 28, 28, 4, dtype=torch.uint64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
fl = torch.empty(64 * 1024 * 1024, device="cuda"); fr = torch.zeros(64 * 1024 * 1024, device="cuda")
sink = torch.empty((), device="cuda")
ref_out = torch.empty((), device="cuda")
y = torch.empty_like(x)
def ref_sum(s):
    torch.amax(x.view(-1), dim=0, out=ref_out)
def ref_copy(s):
    y.copy_(x)
def pack(s):
    lib.bnn_pack_nchw_f32(x.data_ptr(), 32, 256, 28, 28, out.data_ptr(), 0, flags.data_ptr(), s)
import statistics
for name, fn in (("pack", pack), ("torch.sum", ref_sum), ("torch.copy", ref_copy)):
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn(side.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn(torch.cuda.current_stream().cuda_stream)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    ts = []
    for i in range(20):
        cold = i % 2 == 0
        if cold:
            fl.zero_(); torch.amax(fr, dim=0, out=sink)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); g.replay(); e.record(); e.synchronize()
        ts.append((cold, s.elapsed_time(e) * 1e3))
    print(f"{name}: cold us: {statistics.median(t for c, t in ts if c):.2f}  warm us: {statistics.median(t for c, t in ts if not c):.2f}")
