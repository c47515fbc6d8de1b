import os, sys, torch
sys.path.insert(0, os.getcwd())
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
import torch.distributed as dist
from paper_2308_12093_b200 import device as d, dist as pd
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
ctx = d.Context.default(0)
n, E = 2449029, 61859140
src, dst = d.powerlaw_graph(n, E / n, 2.5, 1, ctx)
ones = torch.ones(src.numel(), dtype=torch.float32, device="cuda")
r, c, v = d.canonicalize(n, n, src, dst, ones, ctx)
r, c, v = d.gcn_normalize(n, r, c, v, ctx)
gl = pd.DistGcnLayer(n, r, c, v, pd.DeviceOps("cuda:0"), torch.float32)
model = pd.DistGcn2(gl, 100, 256, 47, 14, caching=True)
X = d.random_uniform(n, 100, 12)
tgt = d.random_uniform(n, 47, 13)
for _ in range(3):
    model.train_step(X, tgt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); model.train_step(X, tgt); e1.record(); torch.cuda.synchronize()
print("gcn2 step ms", e0.elapsed_time(e1))
dist.destroy_process_group()
