import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2308_12093_b200 import device as d
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
P = d.Pattern.gat_pattern(n, src, dst)
X = d.random_uniform(n, 128, 12)
m = d.Model("gat2", 128, 32, 40, heads=8, gat_level="full", seed=14)
t = d.random_uniform(n, 320, 13)
for _ in range(3): m.train_step(P, X, t)
torch.cuda.synchronize()
