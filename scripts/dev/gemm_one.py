"""One GCN layer step on the Arxiv shape (GEMM profiling target)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2308_12093_b200 import device as d
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
X = d.random_uniform(n, 128, 11)
th, b = d.gcn_params(128, 256, 13)
G = d.random_uniform(n, 256, 12)
s = d.resolve_scheme("adaptive", 128, 256, True, True)
for _ in range(3):
    out, c = d.gcn_forward(A, X, th, b, s)
    d.gcn_backward(A, G, th, c, True)
torch.cuda.synchronize()
