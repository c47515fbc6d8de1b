"""Dev: three bench GCN steps (Arxiv 128->256, fg, adaptive + caching) for ncu
launch lists: python scripts/dev/gcn_step.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_12093_b200 import device as d  # noqa: E402

n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
X = d.random_uniform(n, 128, 12)
G = d.random_uniform(n, 256, 13)
th, b = d.gcn_params(128, 256, 14)
s = d.resolve_scheme("adaptive", 128, 256, True, True)
for _ in range(3):
    out, c = d.gcn_forward(A, X, th, b, s)
    d.gcn_backward(A, G, th, c, True)
torch.cuda.synchronize()
