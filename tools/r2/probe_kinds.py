"""Dense tcgen05.mma issue rates per operand form / N (bnn_probe_pipe_peak pipes 1-5)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import _lib  # noqa: E402

lib = bnn.load_library()
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
names = {1: "i8 SS 128x256", 2: "mxf4 SS 128x256", 3: "mxf4 TS 128x64", 4: "mxf4 SS 128x64",
         5: "mxf4 TS 128x256", 6: "mxf4 SS 128x64, 9/commit", 7: "... + wait per commit",
         8: "sconv pattern 9/commit", 9: "sconv pattern + wait", 10: "9 + 13 spinning warps",
         11: "9 + 13 warps nanosleep"}
for pipe in (1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11):
    r = ctypes.c_double(0)
    _lib.check(lib.bnn_probe_pipe_peak(pipe, 4096, sink.data_ptr(), ctypes.byref(r),
                                       _lib.stream_ptr()), "probe")
    print(f"{names[pipe]:18s} {r.value / 148 / 1.965e9:8.0f} MAC/clk/SM  ({2 * r.value / 1e12:7.0f} binary TOPS)")
