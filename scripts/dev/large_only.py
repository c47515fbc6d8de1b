import os, sys, argparse, json
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2308_12093_b200 import device as d
torch.cuda.set_device(0)
ctx = d.Context.default(0)
print(json.dumps(bench.large_graph_steps(None, ctx, 1, 5)))
