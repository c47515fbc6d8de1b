"""Dev: three Gcn2 128-256-40 training steps (adaptive + caching) on the Arxiv
shape for ncu launch lists."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_12093_b200 import device as d

n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
X = d.random_uniform(n, 128, 12)
m = d.Model("gcn2", 128, 256, 40, scheme="adaptive", caching=True, seed=14)
t = d.random_uniform(n, 40, 13)
for _ in range(3):
    m.train_step(A, X, t)
torch.cuda.synchronize()
