"""Dev: three Gat2 training steps on the Arxiv shape (for ncu launch lists).
python scripts/dev/gat2_step.py [hidden_per_head=32]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_12093_b200 import device as d

hid = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
P = d.Pattern.gat_pattern(n, src, dst)
X = d.random_uniform(n, 128, 12)
m = d.Model("gat2", 128, hid, 40, heads=8, gat_level="full", seed=14)
t = d.random_uniform(n, 320, 13)
for _ in range(3):
    m.train_step(P, X, t)
torch.cuda.synchronize()
