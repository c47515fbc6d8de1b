"""One Gat2 128-(8xHID)-(8x40) step on the Arxiv shape (for ncu launch lists)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2308_12093_b200 import device as d
hid = int(os.environ.get("HID", "256"))
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
P = d.Pattern.gat_pattern(n, src, dst)
X = d.random_uniform(n, 128, 12)
m = d.Model("gat2", 128, hid, 40, heads=8, gat_level=os.environ.get("LEVEL", "full"), seed=14)
t = d.random_uniform(n, 8 * 40, 13)
for _ in range(3):
    m.train_step(P, X, t)
torch.cuda.synchronize()
