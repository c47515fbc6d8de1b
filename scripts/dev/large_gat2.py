import os, sys, torch
sys.path.insert(0, os.getcwd())
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29556")
import torch.distributed as dist
from paper_2308_12093_b200 import device as d, dist as pd
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
ctx = d.Context.default(0)
n, E = 2449029, 61859140
src, dst = d.powerlaw_graph(n, E / n, 2.5, 1, ctx)
P = d.Pattern.gat_pattern(n, src, dst, ctx)
pa = P.arrays()
l1 = pd.DistGatLayer(n, pa["rowptr"], pa["cols"], 8, 32, "cuda:0")
l2 = pd.DistGatLayer(n, pa["rowptr"], pa["cols"], 8, 8, "cuda:0")
model = pd.DistGat2(l1, l2, 100, 32, 8, 8, 14)
X = d.random_uniform(n, 100, 12)
tgt = d.random_uniform(n, 64, 13)
for _ in range(3):
    model.train_step(X, tgt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); model.train_step(X, tgt); e1.record(); torch.cuda.synchronize()
print("gat2 step ms", e0.elapsed_time(e1))
dist.destroy_process_group()
