import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
from paper_1705_09864_b200 import nets
bnn.load_library()
rng = np.random.default_rng(0)
d = nets.Dense(512, 1000, rng=rng)
x = torch.randn((256, 512, 7, 7), device="cuda")
for _ in range(3):
    nets.avgpool_dense(x, d)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20):
        nets.avgpool_dense(x, d)
g.replay(); torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); g.replay(); e.record(); e.synchronize()
print("avgpool_fc us", s.elapsed_time(e) / 20 * 1e3)
