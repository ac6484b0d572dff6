"""One LeNet fused-stem call (batch 1024) after a warm-up, for ncu."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn  # noqa: E402
from paper_1705_09864_b200 import nets  # noqa: E402

bnn.load_library()
conv = nets.Conv2d(1, 64, 5, pad=2, rng=np.random.default_rng(0))
x = torch.rand(1024, 1, 28, 28, device="cuda")
for _ in range(3):
    nets._lenet_stem_forward(conv, x)
torch.cuda.synchronize()
print("ok")
