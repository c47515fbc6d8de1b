"""Dev: three GAT layer fwd+bwd steps (level full, fg) on the Arxiv shape for
ncu launch lists.  python scripts/dev/gat_layer.py H K [M_IN=128]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_12093_b200 import device as d

h, k = int(sys.argv[1]), int(sys.argv[2])
m = int(sys.argv[3]) if len(sys.argv) > 3 else 128
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
P = d.Pattern.gat_pattern(n, src, dst)
X = d.random_uniform(n, m, 12)
th, a_s, a_d, b = d.gat_params(m, h, k, 14)
G = d.random_uniform(n, h * k, 13)
for _ in range(3):
    o, c = d.gat_forward(P, X, th, a_s, a_d, b, h, 0.2, "full")
    d.gat_backward(P, G, th, a_s, a_d, c, True)
torch.cuda.synchronize()
