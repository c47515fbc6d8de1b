import sys, os, statistics, torch
sys.path.insert(0, os.getcwd())
from paper_2308_12093_b200 import device as d
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
P = d.Pattern.gat_pattern(n, src, dst)
X = d.random_uniform(n, 128, 12)
for hid, out in ((256, 40), (128, 40), (32, 40)):
    m = d.Model("gat2", 128, hid, out, heads=8, gat_level="full", seed=14)
    t = d.random_uniform(n, 8 * out, 13)
    for _ in range(2): m.train_step(P, X, t)
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); m.train_step(P, X, t); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    print(f"gat2 128-(8x{hid})-(8x{out}): {statistics.median(ms):.2f} ms", flush=True)
    del m
