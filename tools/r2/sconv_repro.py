"""Minimal reproducer: one small-channel conv (layer-1 geometry, batch 2), synchronised."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402

bnn.load_library()
rng = np.random.default_rng(11)
b, c, h, w, f = 2, 64, 56, 56, 64
x = torch.from_numpy(rng.standard_normal((b, c, h, w)).astype(np.float32)).cuda()
layer = bnn.QConvolution(c, f, (3, 3), (1, 1), (1, 1), domain="dot")
layer.weight = rng.standard_normal((f, c, 3, 3)).astype(np.float32)
layer.pack()
torch.cuda.synchronize()
print("packed", flush=True)
y = layer.forward_fused(x)
torch.cuda.synchronize()
print("ok", float(y.abs().sum()))
