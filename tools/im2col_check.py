"""im2col TMA route vs oracle over a set of conv shapes (debug)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "tests/golden")
import workloads as wl
from oracle import oracle as orc
import paper_1705_09864_b200 as bnn
from test_gpu_parity import IM2COL_CASES
bnn.load_library()
extra = [(1, 256, 14, 14, 8, 3, 3, (2, 2), (1, 1), 41), (1, 256, 14, 14, 8, 1, 1, (2, 2), (0, 0), 42),
         (1, 256, 7, 7, 8, 3, 3, (1, 1), (1, 1), 43), (1, 256, 5, 9, 8, 1, 1, (1, 1), (0, 0), 44),
         (1, 256, 5, 9, 8, 3, 1, (1, 1), (0, 0), 45), (1, 256, 5, 9, 8, 1, 3, (1, 1), (0, 0), 46)]
for case in IM2COL_CASES + extra:
    x, wt = wl.conv_case_inputs(case)
    expect = orc.qconv_packed(x, wt, case[7], case[8])
    layer = bnn.QConvolution(case[1], case[4], (case[5], case[6]), case[7], case[8])
    layer.weight = wt; layer.pack(); layer.algo = "umma"
    y = layer.forward(torch.from_numpy(x).cuda(), bnn.INFER_PACKED).cpu().numpy()
    bad = np.argwhere(y != expect)
    print(os.environ.get("BNN_UMMA_DEBUG", "0"), case, "OK" if len(bad) == 0 else f"BAD {len(bad)}/{y.size} first {bad[:3].tolist()}")

for case in [(1, 256, 7, 7, 8, 3, 3, (1, 1), (1, 1), 43), (1, 256, 5, 6, 8, 3, 3, (1, 1), (1, 1), 47),
             (1, 256, 5, 6, 8, 3, 3, (1, 1), (1, 0), 48), (1, 256, 5, 6, 8, 3, 3, (1, 1), (0, 1), 49)]:
    x, wt = wl.conv_case_inputs(case)
    expect = orc.qconv_packed(x, wt, case[7], case[8])
    layer = bnn.QConvolution(case[1], case[4], (case[5], case[6]), case[7], case[8])
    layer.weight = wt; layer.pack(); layer.algo = "umma"
    y = layer.forward(torch.from_numpy(x).cuda(), bnn.INFER_PACKED).cpu().numpy()
    print(case)
    print((y - expect)[0, 0].astype(int))
    # what the output would be with zero (i.e. -1) padding instead of +1
    xp = np.pad(x, ((0, 0), (0, 0), (case[8][0],) * 2, (case[8][1],) * 2), constant_values=-1.0)
    e2 = orc.qconv_packed(xp, wt, case[7], (0, 0))
    print("vs -1 padding:", np.array_equal(y, e2))
