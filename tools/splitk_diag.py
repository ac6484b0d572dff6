"""Diagnose split-K concurrency for config 1 (CUDA-event timings, eager)."""
import os, sys
_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [_R, os.path.join(_R, "tests", "golden")]
import torch
import workloads as wl
import paper_1705_09864_b200 as bnn
from paper_1705_09864_b200 import _lib
from paper_1705_09864_b200.plan import DensePlan

os.environ["BNN_DENSE_SPLITK"] = "8"
a, w = wl.config1_inputs()
layer = bnn.QFullyConnected(4096, 1024, domain="dot")
layer.weight = w
layer.pack()
plan = DensePlan(layer, 256)
plan.x.copy_(torch.from_numpy(a))
plan.pack()
lib = plan.lib


def gemm(k0, k1, st, out):
    w0 = k0 // 64
    _lib.check(lib.bnn_xnor_gemm(plan.wa.data_ptr() + 8 * w0, plan.wa.shape[1], plan.xw.data_ptr() + 8 * w0,
                                 plan.xw.shape[1], plan.m, plan.n, k1 - k0, 0, 0, out.data_ptr(), 1, plan.m,
                                 0, None, None, 0, st), "g")


def timeit(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def graph_time(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return timeit(g.replay)


cur = lambda: torch.cuda.current_stream().cuda_stream
if "--ncu" in sys.argv:  # launch list only: one unsplit GEMM, then one split step
    gemm(0, 4096, cur(), plan.y)
    plan._kernel_split()
    torch.cuda.synchronize()
    sys.exit(0)
print("full K=4096 eager us", timeit(lambda: gemm(0, 4096, cur(), plan.y)))
print("one chunk K=512 eager us", timeit(lambda: gemm(0, 512, cur(), plan.part[0])))
print("one chunk K=512 graph us", graph_time(lambda: gemm(0, 512, cur(), plan.part[0])))
print("8 chunks one stream graph us", graph_time(lambda: [gemm(k0, k1, cur(), plan.part[i]) for i, (k0, k1) in enumerate(plan.chunks)]))
print("split kernel() graph us", graph_time(plan._kernel_split))
print("split kernel() eager us", timeit(plan._kernel_split))
print("sum only us", timeit(lambda: lib.bnn_sum_partials_f32(plan.part.data_ptr(), 8, plan.y.numel(), plan.y.numel(), 1, 4096, plan.y.data_ptr(), cur())))
for v in range(5):
    try:
        lib.bnn_set_umma_variant(v)
        print("variant", v, "K=512 graph us", graph_time(lambda: gemm(0, 512, cur(), plan.part[0])),
              "full", graph_time(lambda: gemm(0, 4096, cur(), plan.y)))
    except Exception as e:
        print("variant", v, e)
