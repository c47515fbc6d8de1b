import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2308_12093_b200 import device as d
n, m = 169343, 128
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
X = d.random_uniform(n, m, 12)
k = int(os.environ.get("K", "8")); fg = os.environ.get("FG", "0") == "1"
th, b = d.gcn_params(m, k, 14)
G = d.random_uniform(n, k, 13)
sch = d.resolve_scheme("adaptive", m, k, fg, True)
print(sch)
for _ in range(3):
    out, c = d.gcn_forward(A, X, th, b, sch); d.gcn_backward(A, G, th, c, fg)
torch.cuda.synchronize()
